python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final2.log 2>&1; tail -2 gpurun_out/pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/exp/profile_round.sh r1final2
timeout 300 python bench.py --workload longcat --mtp 2 --no-cpu-baseline > gpurun_out/r1final2_bench_longcat_mtp2.json 2>/dev/null
timeout 300 python bench.py --workload dsr1 --mtp 2 --no-cpu-baseline > gpurun_out/r1final2_bench_dsr1_mtp2.json 2>/dev/null
