"""Summarise an ncu --csv launch list by kernel: time share, average duration and, when the
list carries them, the FP64-pipe utilisation and DRAM bytes per launch (fused lambdas are
identified by solver step and instance number)."""
import collections
import csv
import re
import sys

TIME = "gpu__time_duration.sum"
FP64 = "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"
RD, WR = "dram__bytes_read.sum", "dram__bytes_write.sum"
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "%": 1.0, "": 1.0}


def short(name):
    name = re.sub(r"\((?:int|bool)\)", "", name)
    m = re.match(r"(?:void )?(?:mpk::)?(?:\(anonymous namespace\)::|<?unnamed>::)?(\w+)(<[\d, ]+>)?", name)
    base = (m.group(1) + (m.group(2) or "")) if m else name[:50]
    r = re.match(r"(?:void )?(?:mpk::)?rows_kernel<(\d), (\d), (\d), (\d)", name)
    if r:
        base = f"rows_kernel<K={r.group(1)},cx={r.group(2)},NH={r.group(3)},NN={r.group(4)}>"
    s = re.search(r"Solver<(\d), (\d)>::(\w+)\([^)]*\)::\[lambda[^\]]*\(instance (\d+)\)\]", name)
    if s:
        base += f" {s.group(3)}#{s.group(4)}"
    t = re.search(r"sweep\w*_kernel<(\d), (\d)>", name)
    if t:
        base += f" cx={t.group(1)} adj={t.group(2)}"
    return base


rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ii, ki, mi, ui, vi = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                              "Metric Value"))
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) <= vi:
        continue
    names[r[ii]] = short(r[ki])
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
tot = 0.0
for lid, m in per.items():
    a = agg[names[lid]]
    t = m.get(TIME, 0.0)
    a[0] += 1
    a[1] += t
    a[2] += m.get(FP64, 0.0) * t
    a[3] += m.get(RD, 0.0)
    a[4] += m.get(WR, 0.0)
    tot += t
print(f"total {tot/1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches")
print("     time     share   launches   avg        fp64-pipe  DRAM rd+wr /launch   kernel")
for k, (c, v, f, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:45]:
    print(f"{v/1e3:10.1f} us {100*v/tot:5.1f}%  n={c:4d} avg={v/c/1e3:9.2f} us  "
          f"{(f/v if v else 0):5.1f}%  {rd/c/1e6:8.1f}+{wr/c/1e6:7.1f} MB  {k}")
