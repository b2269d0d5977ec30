export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_hc.so
timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in libsnapmla_v13 libsnapmla; do
export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/$v.so
echo "== $v"
for w in dsr1 longcat dsr1_tp8; do timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:30], d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
done
export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_trace.so
timeout 200 python scripts/trace_decode.py 128 64 16384 > gpurun_out/trace_v15b_lc.txt 2>&1
