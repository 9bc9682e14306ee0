"""Full circulant embedding: this library's hand-written engine
(ts_operator_create_embed_ex, complex64, mirror-corner symbols) against cuFFT
(tools/embed_baseline.py, full symbols) and the split engine, same x, device
resident, CUDA events. Usage: python tools/embed_compare.py [c1|c3] [steps]"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import embed_baseline  # noqa: E402
import paper_2406_17981_b200 as T  # noqa: E402
from paper_2406_17981_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
levels = W.CONFIGS[name][0]
s = math.prod(levels)
x = torch.from_numpy(W.input_vector(T, name)).to(torch.complex64).cuda()
y = torch.empty_like(x)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


out = {"config": name, "levels": levels}
sp = W.make_operator(T, name)
out["split_ms"] = timed(lambda: sp.apply_device(x, y))
y_split = y.clone()
del sp
torch.cuda.empty_cache()
T.reset_memory_peak(0)
emb = T.Operator.embed_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
ye = torch.empty_like(x)
out["embed_hand_ms"] = timed(lambda: emb.apply_device(x, ye))
out["embed_hand_peak_library_bytes"] = T.memory_stats(0)["peak_bytes"]
out["embed_hand_symbol_bytes"] = emb.info()["spectra_bytes"]
out["embed_hand_rel_l2_vs_split"] = (torch.linalg.vector_norm((ye - y_split).to(torch.complex128)) /
                                     torch.linalg.vector_norm(y_split.to(torch.complex128))).item()
del emb, ye
torch.cuda.empty_cache()
r = embed_baseline.run(levels, x, y_split, steps=steps, warmup=1)
out["embed_cufft_ms"] = r["ms_per_step"]
out["embed_cufft_peak_bytes"] = r["peak_device_bytes"]
out["embed_cufft_rel_l2_vs_split"] = r["rel_l2_vs_split_engine"]
print(json.dumps(out))
