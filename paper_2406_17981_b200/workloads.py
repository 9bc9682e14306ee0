"""The BASELINE.json workloads (configs[0..4]) as operators and inputs of this
library, shared by bench.py and the full-size parity tests so that both build
exactly the same operator from exactly the same seeded inputs.

Conventions: "CN(0,1)" is variance 0.5 per real/imaginary
part in the reference RNG (ref proj/src/core/instance.cpp:13); 3x3 vectors are
SoA, drawn as ts_random_vector(d+1, {3, n, ...}, seed, 0.5) (component
outermost); the dyadic kernel is configs[1]'s G with k = 2 pi/10 and
G(0) = (1 + 0.1i) I.
"""
from __future__ import annotations

import math

import numpy as np

# name: (levels, kind, precision, storage, lag seed, x seed, BASELINE.json configs index)
CONFIGS = {
    "c0": ([16, 16, 16], "random", "c128", "full", 0, 1, 0),
    "c1": ([64, 64, 64], "dyadic", "c64", "full", None, 2, 1),
    "c1_128": ([64, 64, 64], "dyadic", "c128", "full", None, 2, 1),
    "c1m": ([64, 64, 64], "dyadic", "c64", "auto", None, 2, 1),  # mirror-compressed spectra
    "c2": ([256, 256, 256], "dyadic", "c64", "auto", None, 3, 2),
    "c3": ([512, 512, 512], "dyadic", "c64", "auto", None, 4, 3),
    "c3full": ([512, 512, 512], "dyadic", "c64", "full", None, 4, 3),  # full 6-unique spectra
    "c4": ([64, 64, 64, 64], "scaled", "c64", "full", 5, 6, 4),
}


def components(name: str) -> int:
    return 3 if CONFIGS[name][1] == "dyadic" else 1


def lag_offset_norms(levels) -> np.ndarray:
    """|m|_2 for every lag offset m in [-(n_a-1), n_a-1]^d, in the reference's
    lag layout (row-major, level 1 outermost, lag m_a at m_a + n_a - 1;
    ref proj/src/core/generator.hpp:14-19)."""
    r2 = np.zeros([2 * n - 1 for n in levels], np.float64)
    for a, n in enumerate(levels):
        m = np.arange(-(n - 1), n, dtype=np.float64) ** 2
        shape = [1] * len(levels)
        shape[a] = 2 * n - 1
        r2 += m.reshape(shape)
    return np.sqrt(r2).reshape(-1)


def scale_lags_by_offset(lags, levels) -> np.ndarray:
    """configs[4]: t_m -> t_m / (1 + |m|_2) (complex128, reference lag layout)."""
    lags = np.asarray(lags, np.complex128).reshape(-1)
    if lags.size != math.prod(2 * n - 1 for n in levels):
        raise ValueError("lag tensor does not match levels")
    return lags / (1.0 + lag_offset_norms(levels))


def block_generator(T, name: str):
    """The configs[i] generator as a ts_block_generator of this library."""
    levels, kind, _, _, lag_seed, _, _ = CONFIGS[name]
    if kind == "dyadic":
        return T.BlockGenerator.dyadic(levels)
    sym = T.SYM_GENERAL
    g = T.Generator.random(levels, lag_seed, 0.5, sym)
    if kind == "random":
        return T.BlockGenerator.from_scalar(g)
    lags = scale_lags_by_offset(g.lags(), levels)
    del g
    return T.BlockGenerator.create(levels, 1, [0], [lags], [[0] * len(levels)])


def make_operator(T, name: str, part: int = 0, nparts: int = 1, device: int = -1):
    levels, kind, prec, storage, _, _, _ = CONFIGS[name]
    st = {"auto": T.STORAGE_AUTO, "full": T.STORAGE_FULL,
          "compressed": T.STORAGE_COMPRESSED}[storage]
    pr = T.C64 if prec == "c64" else T.C128
    return T.Operator.split_ex(block_generator(T, name), precision=pr, storage=st,
                               device=device, part=part, nparts=nparts)


def input_vector(T, name: str) -> np.ndarray:
    """x i.i.d. CN(0,1) from the reference RNG (complex128, SoA)."""
    levels, kind, _, _, _, seed, _ = CONFIGS[name]
    comp = components(name)
    lv = ([comp] + list(levels)) if comp > 1 else list(levels)
    return T.random_vector(lv, seed, 0.5)
