"""Top stall locations from `ncu --page source --csv` output (SASS view)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Address":
        cur = (r, []); blocks.append(cur)
    elif cur and len(r) > 3 and r[0] not in ("Kernel Name",):
        cur[1].append(r)
for h, data in blocks:
    si = h.index("Warp Stall Sampling (All Samples)")
    vals = []
    for r in data:
        try:
            vals.append((float(r[si] or 0), r))
        except ValueError:
            pass
    tot = sum(v for v, _ in vals) or 1
    print("=== block", len(vals), "rows, samples", tot)
    for v, r in sorted(vals, key=lambda t: -t[0])[:n]:
        print(f"{v/tot*100:5.1f}%  {r[0]}  {r[1][:100]}")
