"""Multi-RHS throughput: ts_operator_apply_batch_device (one launch sequence
for nrhs vectors; the leaf pass reads each spectra row once for all of them)
against nrhs single applies, device-resident, CUDA events.
Usage: python tools/batch_rate.py [config] [nrhs ...]  -> one JSON line per nrhs"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_17981_b200 as T  # noqa: E402
from paper_2406_17981_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
counts = [int(v) for v in sys.argv[2:]] or [4, 8]
op = W.make_operator(T, name)
info = op.info()
n = info["m"]
for v in W.CONFIGS[name][0]:
    n *= v
dt = torch.complex64 if info["precision"] == T.C64 else torch.complex128


def timed(fn, reps):
    for _ in range(3):  # the engine captures its launch graph on a repeated call
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for k in counts:
    x = torch.randn(k * n, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    reps = max(3, int(2000 / max(1, k * n // 100000)))
    reps = min(reps, 200)
    ms_b = timed(lambda: op.apply_batch_device(x, y, k), max(3, reps // k))
    ms_s = timed(lambda: [op.apply_device(x[r * n:(r + 1) * n], y[r * n:(r + 1) * n]) for r in range(k)],
                 max(3, reps // k))
    print(json.dumps({"config": name, "nrhs": k, "batched_mvm_per_s": k / (ms_b / 1e3),
                      "single_mvm_per_s": k / (ms_s / 1e3), "speedup": ms_s / ms_b,
                      "batched_ms": ms_b, "singles_ms": ms_s, "graph_replays": op.info()["graph_replays"]}))
    del x, y
    torch.cuda.empty_cache()
