for lib in libsnapmla_nopf libsnapmla libsnapmla_nopf libsnapmla; do
  export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/$lib.so
  for a in "--workload dsr1" "--workload longcat" "--workload dsr1_tp8" "--workload dsr1 --bf16" "--workload longcat --bf16"; do
    timeout 300 python bench.py $a --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$a', d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
