"""Small applies through every kernel family (TMA strided passes at 512 / 256,
wide passes, the 512- / 256- / 64-point leaves, complex128, generic mixed radix
and primes, d = 4), each checked against the CPU oracle: a seconds-long check
of a new build on a GPU box before the full suite. (compute-sanitizer is closed
on this pool, so out-of-bounds hunting relies on cases like these.)
Usage: python tools/family_cases.py [case-substring]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2406_17981_b200 as T  # noqa: E402

O = oracle.Oracle()
flt = sys.argv[1] if len(sys.argv) > 1 else ""


def dyadic(levels, prec, tol):
    s = int(np.prod(levels))
    xs = O.random_vector([3] + levels, 2, 0.5)
    ys = np.concatenate(O.dyadic_apply(levels, [xs[i * s:(i + 1) * s] for i in range(3)]))
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=prec)
    err = oracle.rel_l2(op.apply(xs), ys)
    assert err <= tol, (levels, err)
    return err


def scalar(levels, sym, prec, tol):
    g = T.Generator.random(levels, 5, 0.5, sym)
    x = T.random_vector(levels, 6, 0.5)
    lags = O.random_lags(levels, 5, 0.5, sym)
    y_ref = O.split_apply(levels, O.precompute(levels, lags), x)
    op = T.Operator.split_ex(T.BlockGenerator.from_scalar(g), precision=prec)
    err = oracle.rel_l2(op.apply(x), y_ref)
    assert err <= tol, (levels, err)
    return err


CASES = {
    # TMA strided passes at 512 (axis 0), 8-point strided kernel (axis 1), 512-point FS leaf
    "wtma512_leaf512": lambda: dyadic([512, 4, 512], T.C64, 1e-5),
    # TMA strided passes at 256, 256-point FS leaf (two CTAs per SM)
    "wtma256_leaf256": lambda: dyadic([256, 8, 256], T.C64, 1e-5),
    # per-thread-load wide passes and the 64-point leaf (configs[1] shape, smaller)
    "wide64_leaf64": lambda: dyadic([64, 64, 64], T.C64, 1e-5),
    # complex128 wide + leaf
    "c128_128": lambda: dyadic([128, 4, 128], T.C128, 1e-12),
    # generic mixed-radix / prime kernels
    "generic": lambda: dyadic([12, 10, 14], T.C64, 1e-5),
    "generic_prime": lambda: scalar([13, 7, 9], T.SYM_GENERAL, T.C128, 1e-12),
    # scalar, d = 4 (configs[4] shape, smaller), full storage
    "scalar_d4": lambda: scalar([16, 16, 16, 64], T.SYM_GENERAL, T.C64, 1e-5),
    # configs[0]
    "c0": lambda: scalar([16, 16, 16], T.SYM_GENERAL, T.C128, 1e-12),
}

for name, fn in CASES.items():
    if flt in name:
        print(name, f"rel-L2 {fn():.2e}", flush=True)
print("family cases ok")
