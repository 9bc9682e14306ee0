"""Small driver for ncu: build one operator of a bench config and run a few
device applies (no timing, no baselines). Usage:
    python tools/profile_apply.py [c3|c2|c4|c1] [applies]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_17981_b200 as T  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.CONFIGS[cfg_name]
op = bench.make_operator(T, cfg, 0, 1, 0)
info = op.info()
levels = cfg[0]
n = info["m"]
for v in levels:
    n *= v
dt = torch.complex64 if info["precision"] == T.C64 else torch.complex128
x = torch.randn(n, dtype=dt, device="cuda")
y = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(reps):
    op.apply_device(x, y)
torch.cuda.synchronize()
print("ok", cfg_name, info)
