"""Stall breakdown of an ncu source page (SASS): samples per stall reason and
the top sampled instructions with their dominant reasons.

  ncu -i x.ncu-rep --page source --csv --print-source sass > x.csv
  python tools/ncu_stalls.py x.csv [top N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = {r: 0 for r in reasons}
for r in data:
    for x in reasons:
        tot[x] += int(r[h.index(x)] or 0)
s = sum(tot.values())
print("total samples", s)
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"  {k:28s} {v:7d} {100 * v / s:5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top lines:")
for r in sorted(data, key=lambda r: -int(r[iss] or 0))[:n]:
    parts = ", ".join(f"{x[6:]}={r[h.index(x)]}" for x in reasons
                      if int(r[h.index(x)] or 0) > 0.1 * int(r[iss] or 1))
    print(f"{int(r[iss]):6d} {r[ia][-5:]} {r[isrc].strip()[:60]:60s} {parts}")
