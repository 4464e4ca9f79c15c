"""Stall-reason breakdown of `ncu --page source --csv --print-source sass`
rows inside an address range of one kernel (e.g. the unrolled step loop).

    python tools/ncu_stall_range.py src.csv KERNEL_SUBSTR LO_HEX HI_HEX [TOP]
"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
sub, lo, hi = sys.argv[2], int(sys.argv[3], 16), int(sys.argv[4], 16)
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
cur_k, hdr, base = None, None, None
agg = collections.Counter()
per = []
for r in rows:
    if r and r[0] == "Kernel Name":
        cur_k = r[1]; base = None; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if not hdr or not cur_k or sub not in cur_k or len(r) < 5:
        continue
    a = int(r[0], 16)
    if base is None:
        base = a
    off = a - base
    if not (lo <= off < hi):
        continue
    d = {hdr[i]: r[i] for i in range(len(hdr))}
    tot = float(d["Warp Stall Sampling (All Samples)"] or 0)
    per.append((tot, off, d["Source"].strip()[:70],
                {k: float(d[k] or 0) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}))
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            agg[k] += float(d[k] or 0)
T = sum(agg.values()) or 1
print("range samples", T)
for k, v in agg.most_common(12):
    print(f"  {k:28s} {v/T*100:5.1f}%")
for tot, off, src, st in sorted(per, key=lambda t: -t[0])[:top]:
    why = ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(st.items(), key=lambda t: -t[1])[:3] if v)
    print(f"{tot/T*100:5.1f}% {off:#06x} {src:70s} {why}")
