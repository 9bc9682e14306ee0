"""Full-size oracle fixtures for BASELINE.json configs[2] (256^3), configs[3]
(512^3, the headline) and configs[4] (64^4), computed by the UNMODIFIED
reference library (oracle/_ref/libtoesplit_ref.so: /root/reference/proj's
core + C ABI compiled by oracle/Makefile against the FFTW-API shim) in
complex128 on the host cores.

    python tests/golden/make_fullsize.py c2|c3|c4 [--threads N] [--out PATH]

c2 and c4 fit this build container (8 cores, 62 GB); c3 needs ~80 GB of host
RAM and ~20 min, so it is run once on the GPU box's host (the prebuilt
oracle/_ref travels there; /root/reference does not) and the fixture is
copied back.

Inputs are exactly the bench's (paper_2406_17981_b200/workloads.py):
  * x: the reference's own ts_random_vector (seed per config, variance 0.5),
    SoA {3, n, n, n} for the dyadic configs;
  * dyadic 3x3 (configs[1] definition): 6 scalar reference operators built
    from the analytic lags (oracle.Oracle.dyadic_lags), G_ii symmetric
    (auto-compressed), G_ij general, 9 applies;
  * configs[4]: lags of ts_generator_random(seed 5, variance 0.5, general)
    (restated bit-exactly by oracle.Oracle.random_lags, pinned against the
    reference in tests/test_oracle_cpu.py) divided by 1 + |m|_2.

The full output (3 x 1.07 GB at 512^3) cannot be committed, so the fixture
keeps size-independent evidence of it:
  * y at 2^19 seeded random positions (numpy PCG64 seed 20240617),
  * every axis-plane sum: for component c and axis a, the sum of y over all
    other axes (m x d x n values — together they touch every element),
  * ||y||_2 per component and sum(y) per component,
  * SHA-256 of the reference's x bytes (the test proves its input identical).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2406_17981_b200 import workloads as W  # noqa: E402  (pure numpy; no GPU needed)

OUT = os.path.dirname(os.path.abspath(__file__))
SAMPLE_SEED = 20240617
SAMPLES = 1 << 19


def sample_positions(total: int, k: int = SAMPLES) -> np.ndarray:
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.unique(rng.integers(0, total, size=min(k, total), dtype=np.int64))


def summarize(y: np.ndarray, levels, m: int) -> dict:
    """The fixture's view of a full output vector (also used by the GPU test)."""
    d = len(levels)
    s = math.prod(levels)
    out = {}
    planes = np.zeros((m, d, max(levels)), np.complex128)
    norms = np.zeros(m)
    sums = np.zeros(m, np.complex128)
    for c in range(m):
        yc = y[c * s:(c + 1) * s].reshape(levels)
        for a in range(d):
            ax = tuple(b for b in range(d) if b != a)
            planes[c, a, :levels[a]] = yc.sum(axis=ax)
        norms[c] = np.linalg.norm(yc)
        sums[c] = yc.sum()
    out["plane_sums"] = planes
    out["norms"] = norms
    out["sums"] = sums
    return out


def reference_output(name: str, threads: int):
    """(fields, y): the reference's complex128 y = T x for configs[name]."""
    levels, kind, _, _, lag_seed, x_seed, cidx = W.CONFIGS[name]
    R = oracle.RefLib()
    O = oracle.Oracle()
    d = len(levels)
    s = math.prod(levels)
    t0 = time.time()
    log = []
    if kind == "dyadic":
        m = 3
        x = R.random_vector([3] + levels, x_seed, 0.5)
        xs = [x[i * s:(i + 1) * s] for i in range(3)]
        y = np.zeros(3 * s, np.complex128)
        for i in range(3):
            for j in range(i, 3):
                t1 = time.time()
                lags = O.dyadic_lags(levels, i, j, threads=threads)
                g = R.generator(levels, lags, oracle.SYM_SYMMETRIC if i == j else oracle.SYM_GENERAL)
                del lags
                op = R.split(g)
                R.destroy_gen(g)
                t2 = time.time()
                y[i * s:(i + 1) * s] += R.apply(op, xs[j], parallel=threads)
                if i != j:
                    y[j * s:(j + 1) * s] += R.apply(op, xs[i], parallel=threads)
                R.destroy_op(op)
                log.append({"component": [i, j], "setup_s": t2 - t1, "apply_s": time.time() - t2})
                print(f"  G_{i}{j}: setup {t2 - t1:.1f} s, apply {time.time() - t2:.1f} s", flush=True)
    else:
        m = 1
        x = R.random_vector(levels, x_seed, 0.5)
        lags = W.scale_lags_by_offset(O.random_lags(levels, lag_seed, 0.5, oracle.SYM_GENERAL), levels)
        g = R.generator(levels, lags, oracle.SYM_GENERAL)
        del lags
        t1 = time.time()
        op = R.split(g)
        R.destroy_gen(g)
        t2 = time.time()
        y = R.apply(op, x, parallel=threads)
        R.destroy_op(op)
        log.append({"setup_s": t2 - t1, "apply_s": time.time() - t2})
    res = {
        "levels": np.array(levels), "components": np.array(m),
        "x_sha256": np.array(hashlib.sha256(x.tobytes()).hexdigest()),
        "meta": np.array(json.dumps({
            "config": f"BASELINE.json configs[{cidx}]", "name": name, "x_seed": x_seed,
            "lag_seed": lag_seed, "engine": "oracle/_ref (unmodified reference + FFTW-API shim), "
            "complex128, TS_POLICY_PARALLEL", "threads": threads, "seconds": time.time() - t0,
            "host_cores": os.cpu_count(), "steps": log})),
    }
    return res, y


def run(name: str, threads: int) -> dict:
    res, y = reference_output(name, threads)
    levels = [int(v) for v in res["levels"]]
    m = int(res["components"])
    pos = sample_positions(m * math.prod(levels))
    res.update({"positions": pos, "y_at": y[pos], **summarize(y, levels, m)})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c2", "c3", "c4"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = run(a.config, a.threads)
    levels = [int(v) for v in res["levels"]]
    path = a.out or os.path.join(OUT, f"{a.config}_{'x'.join(map(str, levels))}_ref.npz")
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    np.savez_compressed(path, **res)
    print(json.loads(str(res["meta"])))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
