"""Per-launch device times of one MVM (CUDA events through the ABI's
ts_operator_profile_device). Usage: python tools/launch_times.py [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_17981_b200 as T  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
op = bench.make_operator(T, cfg, 0, 1, 0)
info = op.info()
n = info["m"]
for v in cfg[0]:
    n *= v
dt = torch.complex64 if info["precision"] == T.C64 else torch.complex128
x = torch.randn(n, dtype=dt, device="cuda")
y = torch.empty_like(x)
for _ in range(2):
    op.apply_device(x, y)
recs = op.profile_device(x, y)
names = {1: "K1", 2: "K2", 3: "K3"}
print(" ".join(f"{names.get(r['kind'], '?')}ax{r['axis']}:{r['ms']:.3f}" for r in recs),
      f"total {sum(r['ms'] for r in recs):.2f} ms")
