for lib in libsnapmla libsnapmla_sus200 libsnapmla_sus2000 libsnapmla libsnapmla_sus200 libsnapmla_sus2000; do
  export SNAPMLA_LIB=$PWD/paper_2602_10718_b200/$lib.so
  for a in "--workload dsr1" "--workload longcat" "--workload dsr1_tp8"; do
    timeout 300 python bench.py $a --no-cpu-baseline --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$a', d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
