"""Summarise ncu captures (run here, on the CPU box) into profiles/.

  python scripts/ncu_summary.py <round-tag> <workload> [<workload> ...]

reads gpurun_out/<tag>_decode_<w>.ncu-rep (ncu --set full of one decode launch)
and gpurun_out/<tag>_launches_<w>.csv (gpu__time_duration of every launch of a
short bench run), writes
  profiles/ncu_decode_summary.json   per workload: dram bytes per launch, % of peak, tensor-pipe activity ...
  profiles/<tag>_ncu_<w>.txt         key metrics + step-kernel shares (timed steps only)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

WANT = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
]
UNIT_SCALE = {"Ghz": 1e9, "Mhz": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "s": 1}


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            out[w] = (vals[i], units[i])
    return out


def to_si(v, u):
    x = float(v.replace(",", ""))
    return x * UNIT_SCALE.get(u, 1.0)


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi, ui, idi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    seq = [(int(r[idi]), r[ki], to_si(r[vi], r[ui])) for r in rows[start + 1:]]
    seq.sort()
    # the timed steps are the tail: append, plan, decode, combine repeated; keep from the first decode on
    names = [s[1] for s in seq]
    first_dec = next(i for i, n in enumerate(names) if "mla_decode_" in n)
    # include the append/plan right before the first decode
    tail = seq[max(0, first_dec - 2):]
    agg = defaultdict(float)
    for _, n, t in tail:
        agg[n.split("(")[0]] += t
    tot = sum(agg.values())
    return {k: (v, v / tot) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])}, tot


def commit_hash():
    try:
        return subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
                              cwd=ROOT).stdout.strip() or None
    except OSError:
        return None


def kernel_name(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, vals = rows[0], rows[2]
    return vals[hdr.index("Kernel Name")].split("(")[0] if "Kernel Name" in hdr else None


def main():
    tag, works = sys.argv[1], sys.argv[2:]
    commit = os.environ.get("NCU_COMMIT") or commit_hash()
    os.makedirs(PROF, exist_ok=True)
    sp = os.path.join(PROF, "ncu_decode_summary.json")
    summary = json.load(open(sp)) if os.path.exists(sp) else {}
    for w in works:
        rep = os.path.join(OUT, f"{tag}_decode_{w}.ncu-rep")
        m = raw_metrics(rep)
        rd = to_si(*m["dram__bytes_read.sum"])
        wr = to_si(*m["dram__bytes_write.sum"])
        dur = to_si(*m["gpu__time_duration.sum"])
        entry = {
            "round": tag,
            "commit": commit,
            "kernel": kernel_name(rep),
            "dram_bytes_per_launch": rd + wr,
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "duration_s_ncu": dur,
            "dram_pct_peak": float(m["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "tensor_pipe_active_pct": float(m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                                                  m.get("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", ("nan",)))[0]),
            "sm_throughput_pct": float(m["sm__throughput.avg.pct_of_peak_sustained_elapsed"][0]),
            "sm_clock_hz": to_si(*m["sm__cycles_elapsed.avg.per_second"]) if m["sm__cycles_elapsed.avg.per_second"][1] != "cycle/second" else float(m["sm__cycles_elapsed.avg.per_second"][0]),
            "registers_per_thread": m["launch__registers_per_thread"][0],
            "grid": m["launch__grid_size"][0],
            "block": m["launch__block_size"][0],
        }
        lines = [f"# ncu summary {tag} / {w}: decode kernel (mla_decode_*), one launch (--set full, --clock-control none)", ""]
        for k, (v, u) in m.items():
            lines.append(f"{k:70s} {v} {u}")
        lp = os.path.join(OUT, f"{tag}_launches_{w}.csv")
        if os.path.exists(lp):
            shares, tot = launch_shares(lp)
            lines += ["", "# launch list (gpu__time_duration, serialized cold-cache; timed-step tail): kernel, total s, share"]
            for k, (v, f) in shares.items():
                lines.append(f"{k[:80]:80s} {v:.6e} {100 * f:5.1f}%")
            entry["decode_share_of_step_ncu"] = next((f for k, (v, f) in shares.items() if "mla_decode_" in k), None)
        key = w + ("_bf16" if "bf16" in tag else "") + ("_mx" if "mx" in tag else "")   # variants keep their own key
        summary[key] = entry
        open(os.path.join(PROF, f"{tag}_ncu_{w}.txt"), "w").write("\n".join(lines) + "\n")
        print(w, json.dumps(entry))
    json.dump(summary, open(sp, "w"), indent=1)


if __name__ == "__main__":
    main()
