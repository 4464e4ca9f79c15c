"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel
(fused lambdas are identified by solver step and instance number)."""
import collections
import csv
import re
import sys


def short(name):
    m = re.match(r"void (?:mpk::)?(?:\(anonymous namespace\)::|<unnamed>::)?(\w+)", name)
    base = m.group(1) if m else name[:50]
    s = re.search(r"Solver<(\d), (\d)>::(\w+)\([^)]*\)::\[lambda[^\]]*\(instance (\d+)\)\]", name)
    if s:
        base += f" {s.group(3)}#{s.group(4)} K={s.group(1)}{' cx' if s.group(2) == '1' else ''}"
    t = re.search(r"sweep\w*_kernel<\(bool\)(\d), \(bool\)(\d)", name)
    if t:
        base += f" cx={t.group(1)} adj={t.group(2)}"
    return base


rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    k = short(r[ki])
    agg[k][0] += 1
    agg[k][1] += v
    tot += v
print(f"total {tot/1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:45]:
    print(f"{v/1e3:10.1f} us {100*v/tot:5.1f}%  n={c:4d} avg={v/c/1e3:8.2f} us  {k}")
