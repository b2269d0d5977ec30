# usage: bash scripts/gpu_round.sh <tag> [quick|full]
# build, the -m gpu suite, smoke, the default bench line (+ reference arm); with "full": the
# LongCat / TP8 / MTP-2 / MX / BF16 lines, the sweep, launch lists and one ncu --set full per workload.
TAG=$1; MODE=${2:-quick}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail -20 gpurun_out/${TAG}_build.log; exit 1; }
git rev-parse --short HEAD > gpurun_out/${TAG}_commit.txt 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/${TAG}_bench_dsr1.json 2> gpurun_out/${TAG}_bench_dsr1.err; tail -c 300 gpurun_out/${TAG}_bench_dsr1.err
python - <<PY
import json
d = json.load(open("gpurun_out/${TAG}_bench_dsr1.json"))
r = d["roofline"]
print("value", d["value"], "ms", d["ms_per_step"], "decode_ms", r["decode_ms"], "bound", r["bound"], "frac", r["frac"],
      "hbm", r["roofs"]["hbm"]["frac"], "tc", r["roofs"]["tensor"]["frac"], "e2e", d["e2e"]["value"], "clk", d["clocks"], d.get("peaks_measured"))
PY
if [ "$MODE" = full ]; then
  timeout 300 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_dsr1.json 2>/dev/null
  for w in longcat dsr1_tp8; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2>/dev/null; done
  timeout 600 python bench.py --mtp 2 --workload longcat --no-cpu-baseline > gpurun_out/${TAG}_bench_longcat_mtp2.json 2>/dev/null
  timeout 600 python bench.py --mx --no-cpu-baseline > gpurun_out/${TAG}_bench_dsr1_mx.json 2>/dev/null
  timeout 600 python bench.py --bf16 --no-cpu-baseline > gpurun_out/${TAG}_bench_dsr1_bf16.json 2>/dev/null
  timeout 900 python bench.py --sweep --steps 10 > gpurun_out/${TAG}_sweep_dsr1_shape.json 2>/dev/null
  for w in dsr1 longcat dsr1_tp8; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_$w.csv python bench.py --workload $w --no-cpu-baseline --no-peaks --quick --steps 2 --warmup 1 > /dev/null 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:mla_decode_ -s 3 -c 1 -o gpurun_out/${TAG}_decode_$w python bench.py --workload $w --no-cpu-baseline --no-peaks --quick --steps 2 --warmup 3 > /dev/null 2>&1
  done
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:mla_decode_ -s 3 -c 1 -o gpurun_out/${TAG}mx_decode_dsr1 python bench.py --mx --no-cpu-baseline --no-peaks --quick --steps 2 --warmup 3 > /dev/null 2>&1
fi
ls gpurun_out | grep "^${TAG}" | head -40
