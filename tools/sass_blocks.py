"""Per-address-block stall/opcode breakdown of an ncu source page export
(ncu -i REP --page source --csv > X.csv). Usage: sass_blocks.py X.csv [kernel_index] [block]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
B = int(sys.argv[3]) if len(sys.argv) > 3 else 100
kernels = []
for r in rows:
    if r and r[0] == "Kernel Name":
        kernels.append([r[1], None, []])
    elif kernels and kernels[-1][1] is None:
        kernels[-1][1] = r
    elif kernels:
        kernels[-1][2].append(r)
name, hdr, data = kernels[kidx]
print(name, len(data), "instructions")
i = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
f = lambda v: float(v) if v not in ("", None) else 0.0
tot = sum(f(r[i]) for r in data)
for s in range(0, len(data), B):
    blk = data[s:s + B]
    smp = sum(f(r[i]) for r in blk)
    ex = sum(f(r[ie]) for r in blk)
    ops = collections.Counter()
    st = collections.Counter()
    for r in blk:
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += f(r[ie])
        for c in cols:
            st[c[6:]] += f(r[hdr.index(c)])
    if tot == 0 or smp / tot < 0.005:
        continue
    top = " ".join(f"{k}:{v / ex * 100:.0f}" for k, v in ops.most_common(4)) if ex else ""
    sts = " ".join(f"{k}:{v / smp * 100:.0f}" for k, v in st.most_common(3))
    print(f"{s:5d} smp {smp / tot * 100:5.1f}%  exec {ex / 1e6:6.1f}M  {top} | {sts}")
