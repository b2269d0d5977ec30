"""Aggregate ncu warp-stall samples of one kernel by warp-role region (split at the
setmaxnreg instructions) and list the top stalled SASS instructions per region.
  ncu -i rep --page source --csv --print-source sass > src.csv ; python scripts/ncu_stalls.py src.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
region, cur = [], "prologue"
for r in data:
    s = r[isrc]
    if "USETMAXREG.DEALLOC" in s and "0x28" in s: cur = "issue"
    elif "USETMAXREG.DEALLOC" in s and "0x78" in s: cur = "softmax"
    elif "USETMAXREG" in s and ("0xb0" in s or "0xa8" in s or "0xb8" in s): cur = "acc"
    region.append(cur)
def f(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
tot = collections.defaultdict(lambda: collections.Counter())
for r, g in zip(data, region):
    tot[g]["ALL"] += f(r[iall])
    for h, i in zip(reasons, ri): tot[g][h] += f(r[i])
grand = sum(t["ALL"] for t in tot.values())
for g, t in tot.items():
    print(f"== {g}: {t['ALL'] / grand * 100:.1f}% of samples;", ", ".join(f"{k[6:]} {v / t['ALL'] * 100:.0f}%" for k, v in t.most_common(8) if k != "ALL"))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for g in tot:
    lst = sorted(((f(r[iall]), r[isrc].strip(), max(((f(r[i]), h[6:]) for h, i in zip(reasons, ri))))
                  for r, gg in zip(data, region) if gg == g), reverse=True)[:top]
    print(f"-- top {g}")
    for v, s, (rv, rn) in lst: print(f"  {v:7.0f}  {rn:>14} {s[:90]}")
