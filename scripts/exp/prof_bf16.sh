python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1bf16_launches_dsr1.csv python bench.py --bf16 --quick --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_decode_kernel -s 3 -c 1 -o gpurun_out/r1bf16_decode_dsr1 python bench.py --bf16 --quick --steps 2 --warmup 3 > /dev/null 2>&1
ls -la gpurun_out | tail -3
