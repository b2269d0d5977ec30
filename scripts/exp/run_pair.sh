# pair kernel bring-up: hang-check build first (stop on failure), then the product build, then A/B bench
export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_hc.so
timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mtp.py -x -q 2>&1 | grep -v "^HANG" | tail -8
timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mtp.py -x -q > /dev/null 2>&1 || exit 1
unset SNAPMLA_LIB
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for np in 0 1; do SNAPMLA_PAIR=$np timeout 200 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_pair=$np', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"; done
