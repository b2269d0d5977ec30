export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_hc.so
timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mtp.py -x -q 2>&1 | grep -v "^HANG" | tail -3
timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_mtp.py -x -q > /dev/null 2>&1 || exit 1
unset SNAPMLA_LIB
TIME_ONLY=1 timeout 200 python scripts/trace_pair.py 2>&1 | tail -1
SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_trace.so timeout 200 python scripts/trace_pair.py > gpurun_out/trace_pair.txt 2>&1; tail -2 gpurun_out/trace_pair.txt
