"""Probe: device applies with x / y offset by one element (8 B for complex64, 16 B for
complex128) from the allocation's alignment. Expected: the serial result, or a clean
TS error — never a fault. (It found the 512-point leaf faulting on an 8-byte-aligned y;
the ABI now refuses pointers that are not 16-byte aligned.) Usage: python tools/misaligned_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_17981_b200 as T  # noqa: E402

CASES = [([512, 512], "scalar", T.C64), ([256, 256], "scalar", T.C64), ([64, 64, 64], "dyadic", T.C64),
         ([8, 16, 512], "dyadic", T.C64), ([128, 32, 64], "scalar", T.C128), ([12, 40, 36], "scalar", T.C64),
         ([13, 64, 10], "scalar", T.C64), ([3, 4099], "scalar", T.C64), ([64, 64], "scalar", T.C64)]
bad = 0
for levels, kind, prec in CASES:
    if kind == "dyadic":
        bg, m = T.BlockGenerator.dyadic(levels), 3
    else:
        bg, m = T.BlockGenerator.from_scalar(T.Generator.random(levels, 9, 1.0, T.SYM_GENERAL)), 1
    op = T.Operator.split_ex(bg, precision=prec)
    dt = torch.complex64 if prec == T.C64 else torch.complex128
    n = m * int(np.prod(levels))
    x = torch.randn(n, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    op.apply_device(x, y)
    torch.cuda.synchronize()
    for ox, oy in ((1, 0), (0, 1), (1, 1), (3, 5)):
        xb = torch.zeros(n + 8, dtype=dt, device="cuda")
        yb = torch.zeros(n + 8, dtype=dt, device="cuda")
        xb[ox:ox + n] = x
        try:
            op.apply_device(xb[ox:ox + n], yb[oy:oy + n])
            torch.cuda.synchronize()
            ok = torch.equal(yb[oy:oy + n], y) and float(yb[:oy].abs().sum()) == 0 and float(yb[oy + n:].abs().sum()) == 0
            print(levels, kind, prec, (ox, oy), "equal" if ok else "MISMATCH", flush=True)
            bad += 0 if ok else 1
        except T.TsError as e:
            print(levels, kind, prec, (ox, oy), "clean error:", e, flush=True)
        except ValueError as e:
            print(levels, kind, prec, (ox, oy), "rejected:", e, flush=True)
print("misaligned probe:", bad, "mismatch(es)")
sys.exit(1 if bad else 0)
