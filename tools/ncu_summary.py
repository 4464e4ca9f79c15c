"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv, re, sys, collections

def short(name):
    n = name
    m = re.search(r"(rows_kernel|fin_kernel|sweep_kernel|factor_kernel|sweep_reset_kernel|set_cond_kernel|relres_kernel|true_res_kernel_impl|to_planar_kernel|from_planar_kernel|gather_kernel|mc_kernel)", n)
    base = m.group(1) if m else n[:60]
    lam = re.search(r"Solver<(\d), (true|false)>::(\w+)\(\)::\[lambda[^\]]*#(\d+)\]", n)
    if lam:
        base += f" {lam.group(3)}#{lam.group(4)} K={lam.group(1)}"
    t = re.search(r"sweep_kernel<(true|false), (true|false)>", n)
    if t:
        base += f" cx={t.group(1)} adj={t.group(2)}"
    return base

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki = hdr.index("Kernel Name"); mi = hdr.index("Metric Name"); vi = hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit_ns = 1.0
    k = short(r[ki])
    agg[k][0] += 1
    agg[k][1] += v
    tot += v
print(f"total {tot/1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{v/1e3:10.1f} us {100*v/tot:5.1f}%  n={c:4d} avg={v/c/1e3:8.2f} us  {k}")
