"""Per-launch device times of one MVM (CUDA events through the ABI's
ts_operator_profile_device), median of REPS profiled MVMs.
Usage: python tools/launch_times.py [config] [reps]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_17981_b200 as T  # noqa: E402
from paper_2406_17981_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
op = W.make_operator(T, name)
info = op.info()
n = info["m"]
for v in W.CONFIGS[name][0]:
    n *= v
dt = torch.complex64 if info["precision"] == T.C64 else torch.complex128
x = torch.randn(n, dtype=dt, device="cuda")
y = torch.empty_like(x)
for _ in range(2):
    op.apply_device(x, y)
runs = [op.profile_device(x, y) for _ in range(reps)]
names = {1: "K1", 2: "K2", 3: "K3"}
med = [statistics.median(r[i]["ms"] for r in runs) for i in range(len(runs[0]))]
print(" ".join(f"{names.get(r['kind'], '?')}ax{r['axis']}:{m:.3f}" for r, m in zip(runs[0], med)),
      f"total {sum(med):.2f} ms")
