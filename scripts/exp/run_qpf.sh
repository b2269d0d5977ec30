for lib in libsnapmla_base libsnapmla libsnapmla_base libsnapmla; do
  export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/$lib.so
  for a in "--batch 1 --context 32768" "--batch 8 --context 32768" "--batch 64 --context 4096" "--workload dsr1" "--workload longcat"; do
    for v in 0 2; do
      SNAPMLA_PAIR=$v timeout 300 python bench.py $a --no-cpu-baseline --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib pair=$v', '$a', d['ms_per_step'], d['roofline']['decode_ms'], d['clocks']['sm_mhz'])"
    done
  done
done
V=2 SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_trace.so timeout 200 python scripts/trace_2sm.py 8 128 32768 2>&1 | tail -7 | head -3
V=0 SNAPMLA_LIB=$PWD/paper_2602_10718_b200/libsnapmla_trace.so timeout 200 python scripts/trace_2sm.py 8 128 32768 2>&1 | tail -7 | head -3
