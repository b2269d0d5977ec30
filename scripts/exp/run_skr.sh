for v in libsnapmla libsnapmla_skr; do
export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/$v.so
echo "== $v"
timeout 100 python scripts/stress_decode.py 4x64x16384 2>&1 | tail -1
for w in dsr1 longcat dsr1_tp8; do timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:30], d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
done
