"""Exploratory fuzz of the CUDA path against the CPU oracle (test infrastructure):
random level shapes (d = 1..5, axes of length 1, primes, powers of two), symmetry modes,
storage modes, precisions, device multi-RHS applies and branch partitions.
Usage: python tools/fuzz_oracle.py [count] [seed]   (prints one line per failure)"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2406_17981_b200 as T  # noqa: E402
from oracle import rel_l2  # noqa: E402

O = oracle.Oracle()
count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
pool = [1, 1, 2, 3, 4, 5, 7, 8, 9, 11, 12, 13, 16, 17, 20, 24, 31, 32, 33, 48, 64, 96, 100, 127, 128, 160, 255, 256,
        257, 512, 513, 1024, 2048, 4096, 4099]
fails = 0
t0 = time.time()
done = 0
while done < count:
    d = int(rng.integers(1, 6))
    lv = [int(rng.choice(pool)) for _ in range(d)]
    s = int(np.prod(lv))
    if not (2 <= s <= 600_000):
        continue
    done += 1
    sym = int(rng.integers(0, 3))
    symc = [T.SYM_GENERAL, T.SYM_SYMMETRIC, T.SYM_SKEW][sym]
    s0 = 0j if rng.random() < 0.6 else complex(rng.normal(), rng.normal())
    storage = int(rng.choice([T.STORAGE_AUTO, T.STORAGE_FULL]))
    sd = int(rng.integers(1, 1 << 30))
    tag = f"levels={lv} sym={sym} s0={s0} storage={storage} seed={sd}"
    try:
        g = T.Generator.random(lv, sd, 1.0, symc)
        lags = O.random_lags(lv, sd, 1.0, symc)
        v = O.random_vector(lv, sd, 1.0)
        signs = oracle.axis_signs(d, symc)
        if not np.abs(lags).max() > 0:  # a skew generator over an axis of length 1 is zero: nothing to compare
            done -= 1
            continue
        comp = (symc == T.SYM_SYMMETRIC or (symc == T.SYM_SKEW and s0 == 0)) if storage == T.STORAGE_AUTO else False
        blocks = O.precompute(lv, lags, s0, comp, signs)
        y_or = O.split_apply(lv, blocks, v, comp, signs)
        op128 = T.Operator.split(g, s0=s0, storage=storage)
        e = rel_l2(op128.apply(v), y_or)
        if not e <= 1e-12:
            fails += 1
            print("FAIL c128", tag, e, flush=True)
        if s0 == 0:
            bg = T.BlockGenerator.from_scalar(g)
            op64 = T.Operator.split_ex(bg, precision=T.C64, storage=storage)
            e = rel_l2(op64.apply(v), y_or)
            if not e <= 1e-5:
                fails += 1
                print("FAIL c64", tag, e, flush=True)
            # multi-RHS on device: column r is x scaled by (r + 1)
            nrhs = int(rng.integers(2, 5))
            x = torch.from_numpy(v).to(torch.complex64).cuda()
            xb = torch.cat([x * (r + 1) for r in range(nrhs)])
            yb = torch.empty_like(xb)
            op64.apply_batch_device(xb, yb, nrhs)
            y1 = torch.empty_like(x)
            op64.apply_device(x, y1)
            torch.cuda.synchronize()
            for r in range(nrhs):
                yr = yb[r * s:(r + 1) * s].cpu().numpy().astype(np.complex128)
                e = rel_l2(yr, y_or * (r + 1))
                if not e <= 1e-5:
                    fails += 1
                    print("FAIL batch", tag, "nrhs", nrhs, "r", r, e, flush=True)
            # branch partitions sum to the whole
            if d >= 2:
                nparts = int(rng.choice([2, 4]))
                if nparts <= (1 << (d - 1)) * 2:
                    acc = np.zeros(s, np.complex128)
                    ok = True
                    for p in range(nparts):
                        try:
                            opp = T.Operator.split_ex(bg, precision=T.C128, storage=storage, part=p, nparts=nparts)
                        except TypeError:
                            ok = False
                            break
                        acc += opp.apply(v)
                        opp.close()
                    if ok:
                        e = rel_l2(acc, y_or)
                        if not e <= 1e-12:
                            fails += 1
                            print("FAIL parts", tag, "nparts", nparts, e, flush=True)
            op64.close()
        op128.close()
    except Exception as ex:  # noqa: BLE001
        fails += 1
        print("EXC", tag, type(ex).__name__, ex, flush=True)
# ---- 3x3 dyadic operators (d = 3): both precisions, both storage modes, partitions, multi-RHS
dpool = [1, 2, 3, 4, 5, 6, 7, 8, 12, 13, 16, 20, 31, 32, 48, 64, 96, 128, 256, 512]
dy = 0
while dy < max(4, count // 5):
    lv = [int(rng.choice(dpool)) for _ in range(3)]
    s = int(np.prod(lv))
    if not (8 <= s <= 300_000):
        continue
    dy += 1
    storage = int(rng.choice([T.STORAGE_AUTO, T.STORAGE_FULL]))
    sd = int(rng.integers(1, 1 << 30))
    tag = f"dyadic levels={lv} storage={storage} seed={sd}"
    try:
        x = O.random_vector([3] + lv, sd, 0.5)
        xs = [x[i * s:(i + 1) * s] for i in range(3)]
        y_or = np.concatenate(O.dyadic_apply(lv, xs, mode="signs"))
        bg = T.BlockGenerator.dyadic(lv)
        for prec, tol in ((T.C128, 1e-12), (T.C64, 1e-5)):
            op = T.Operator.split_ex(bg, precision=prec, storage=storage)
            e = rel_l2(op.apply(x), y_or)
            if not e <= tol:
                fails += 1
                print("FAIL", tag, "prec", prec, e, flush=True)
            if prec == T.C64:
                nrhs = int(rng.integers(2, 4))
                xd = torch.from_numpy(x).to(torch.complex64).cuda()
                xb = torch.cat([xd * (r + 1) for r in range(nrhs)])
                yb = torch.empty_like(xb)
                op.apply_batch_device(xb, yb, nrhs)
                torch.cuda.synchronize()
                for r in range(nrhs):
                    e = rel_l2(yb[r * 3 * s:(r + 1) * 3 * s].cpu().numpy().astype(np.complex128), y_or * (r + 1))
                    if not e <= tol:
                        fails += 1
                        print("FAIL batch", tag, "nrhs", nrhs, "r", r, e, flush=True)
            op.close()
        nparts = int(rng.choice([2, 4, 8]))
        acc = np.zeros(3 * s, np.complex128)
        for p in range(nparts):
            opp = T.Operator.split_ex(bg, precision=T.C128, storage=storage, part=p, nparts=nparts)
            acc += opp.apply(x)
            opp.close()
        e = rel_l2(acc, y_or)
        if not e <= 1e-12:
            fails += 1
            print("FAIL parts", tag, "nparts", nparts, e, flush=True)
    except Exception as ex:  # noqa: BLE001
        fails += 1
        print("EXC", tag, type(ex).__name__, ex, flush=True)
    done += 1
print(f"fuzz: {done} cases, {fails} failure(s), {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
