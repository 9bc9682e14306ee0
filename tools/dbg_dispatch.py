"""Debug helper: which kernel family each pass of a (full-embedding or split)
apply goes to. TSK_DEBUG_DISPATCH=1 python tools/dbg_dispatch.py embed|split n0 n1 n2"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

import paper_2406_17981_b200 as T  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "embed"
levels = [int(v) for v in sys.argv[2:5]] if len(sys.argv) > 4 else [512, 4, 8]
bg = T.BlockGenerator.dyadic(levels)
op = (T.Operator.embed_ex if kind == "embed" else T.Operator.split_ex)(bg, precision=T.C64)
n = 3 * levels[0] * levels[1] * levels[2]
x = torch.randn(n, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
op.apply_device(x, y)
torch.cuda.synchronize()
t = time.time()
op.apply_device(x, y)
torch.cuda.synchronize()
print(f"{kind} {levels}: {1e3 * (time.time() - t):.2f} ms", file=sys.stderr)
