"""Summarise an ncu report: per-kernel key metrics, SASS opcode mix and
stall reasons (reads `ncu -i ... --page raw/source --csv`).
Usage: ncu_summary.py REP.ncu-rep [kernel-substring]
       ncu_summary.py RAW.csv SASS.csv[.gz] [kernel-substring]  (exports made on the box)"""
import collections
import csv
import io
import subprocess
import sys

import gzip

rep = sys.argv[1]
pre = rep.endswith(".csv")
kfilter = sys.argv[3 if pre else 2] if len(sys.argv) > (3 if pre else 2) else "k_"
if pre:
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]
for r in data:
    if kfilter not in r[idx["Kernel Name"]]:
        continue
    print("----")
    for w in want:
        if w in idx:
            print(f"  {w} = {r[idx[w]]} {units[idx[w]]}")
if pre:
    sp = sys.argv[2]
    src = (gzip.open(sp, "rt") if sp.endswith(".gz") else open(sp)).read()
else:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          "regex:" + kfilter], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if pre:  # keep only the sections of matching kernels
    keep, cur = [], False
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = kfilter in r[1]
            continue
        if cur:
            keep.append(r)
    rows = keep
cnt = collections.Counter()
stall = collections.Counter()
tot = 0
h = None
for r in rows:
    if len(r) > 5 and r[0] == "Address":
        h = {k: i for i, k in enumerate(r)}
        continue
    if not h or len(r) < len(h):
        continue
    s = r[h["Source"]].strip()
    if not s:
        continue
    op = s.split()[0]
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    try:
        n = float(r[h["Instructions Executed"]] or 0)
    except ValueError:
        n = 0
    cnt[op] += n
    tot += n
    for k, i in h.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stall[k] += float(r[i] or 0)
            except ValueError:
                pass
print("opcode mix (all matching kernels):")
for op, n in cnt.most_common(18):
    print(f"  {op:10s} {n / 1e6:9.1f}M {100 * n / max(tot, 1):5.1f}%")
st = sum(stall.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100 * v / st:.1f}%" for k, v in stall.most_common(10)))
