"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ci, ii = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > ci]
tot = sum(int(r[ci] or 0) for r in data)
top = sorted(data, key=lambda r: -int(r[ci] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    print(f"{100*int(r[ci])/tot:5.1f}%  {r[0][-5:]}  {r[si].strip()[:90]}")
