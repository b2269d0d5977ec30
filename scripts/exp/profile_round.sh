# usage: bash scripts/exp/profile_round.sh <tag>
# bench lines (default dsr1 with cpu baseline, others quick) + launch lists + one ncu --set full per workload
TAG=$1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py > gpurun_out/${TAG}_bench_dsr1.json 2> gpurun_out/${TAG}_bench_dsr1.err
python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_dsr1.json 2>/dev/null
for w in longcat dsr1_tp8; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2>/dev/null; done
for w in dsr1 longcat dsr1_tp8; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_$w.csv python bench.py --workload $w --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_decode_ -s 3 -c 1 -o gpurun_out/${TAG}_decode_$w python bench.py --workload $w --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
done
ls -la gpurun_out | tail -20
