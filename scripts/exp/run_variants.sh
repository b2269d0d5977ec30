set -x
for v in 0 20 100 1000; do
  export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_sus$v.so
  echo "== suspend $v"
  for w in dsr1 longcat dsr1_tp8; do timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:30], d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
done
unset SNAPMLA_LIB
timeout 400 ncu --set full --clock-control none --import-source on -k regex:mla_decode_kernel -s 3 -c 1 -o gpurun_out/v5b_decode_longcat python bench.py --workload longcat --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out
