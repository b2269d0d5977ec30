# NEXT-2: FP8 vs BF16 on the three workloads (bench lines to gpurun_out)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in dsr1 longcat dsr1_tp8; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 30 > gpurun_out/r1_bench_fp8_$w.json 2>/dev/null
  timeout 300 python bench.py --workload $w --bf16 --steps 30 > gpurun_out/r1_bench_bf16_$w.json 2>/dev/null
  for v in fp8 bf16; do python -c "import json; d=json.loads(open('gpurun_out/r1_bench_${v}_$w.json').read().strip().splitlines()[-1]); print('$v $w', d['value'], d['ms_per_step'], d['roofline']['decode_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_decode_ -s 3 -c 1 -o gpurun_out/r1bf16b_decode_dsr1 python bench.py --bf16 --quick --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1bf16b_launches_dsr1.csv python bench.py --bf16 --quick --steps 2 --warmup 1 > /dev/null 2>&1
