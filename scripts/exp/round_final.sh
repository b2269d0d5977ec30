# round-end evidence: gpu tests, smoke, bench lines (ours + reference arm + BF16 baseline), ncu launch lists + full captures
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; tail -2 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/exp/profile_round.sh r1final
