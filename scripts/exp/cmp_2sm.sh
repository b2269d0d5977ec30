python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for bc in "1 32768" "8 32768" "8 131072" "64 4096" "512 4096" "64 32768" "32 16384"; do
  set -- $bc
  for v in 0 2; do
    SNAPMLA_PAIR=$v timeout 300 python bench.py --batch $1 --context $2 --no-cpu-baseline --steps 40 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$1 L=$2 pair=$v', d['ms_per_step'], d['roofline']['decode_ms'], d['clocks']['sm_mhz'])"
  done
done
