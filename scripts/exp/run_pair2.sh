for g in 0 72 70 66 60; do SNAPMLA_PAIR_GROUPS=$g timeout 200 python bench.py --no-cpu-baseline --quick --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('groups=$g', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))"; done
python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
sys.argv = ["bench.py", "--no-cpu-baseline", "--steps", "3", "--warmup", "3", "--quick"]
import bench
from paper_2602_10718_b200 import ops
try:
    bench.main()
except SystemExit:
    pass
print("max active clusters:", ops.lib().mla_debug_set_pair_groups(0))
PY
