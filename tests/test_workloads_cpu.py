"""CPU checks of the BASELINE.json workload definitions the bench and the
full-size parity tests share (paper_2406_17981_b200/workloads.py): the inputs
are the reference RNG's, bit for bit, and configs[4]'s lag scaling
t_m / (1 + |m|_2) is the stated formula on the reference lag layout."""
import itertools
import json
import math
import os

import numpy as np

import oracle
import paper_2406_17981_b200 as T
from paper_2406_17981_b200 import workloads as W

O = oracle.Oracle()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_configs_follow_baseline_json():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        cfgs = json.load(f)["configs"]
    assert len(cfgs) == 5
    for name, (levels, kind, prec, storage, lag_seed, x_seed, cidx) in W.CONFIGS.items():
        text = cfgs[cidx]
        assert "x".join(map(str, levels)).replace("x", "×") in text
        assert (prec == "c128") == ("complex128" in text and "complex64" not in text) or name == "c1_128"
        if kind == "dyadic":
            assert "3×3" in text
        assert f"seed {x_seed}" in text
        if lag_seed is not None:
            assert f"seed {lag_seed}" in text


def test_lag_offset_norms_and_scaling_on_reference_layout():
    levels = [3, 2, 4]
    lags = O.random_lags(levels, 5, 0.5, oracle.SYM_GENERAL)
    got = W.scale_lags_by_offset(lags, levels)
    # independent loop over the lag layout (ref generator.hpp:14-19): lag m_a
    # at index m_a + n_a - 1, row-major, level 1 outermost
    want = np.empty_like(lags)
    ranges = [range(-(n - 1), n) for n in levels]
    for off, m in enumerate(itertools.product(*ranges)):
        want[off] = lags[off] / (1.0 + math.sqrt(sum(v * v for v in m)))
    assert np.array_equal(got, want)


def test_c4_generator_lags_are_the_reference_draws_scaled():
    levels = [4, 3, 2, 5]
    g = T.Generator.random(levels, 5, 0.5, T.SYM_GENERAL)
    assert np.array_equal(g.lags(), O.random_lags(levels, 5, 0.5, oracle.SYM_GENERAL))


def test_inputs_are_reference_rng_bit_exact():
    for name in ("c0", "c1", "c4"):
        levels, kind, _, _, _, seed, _ = W.CONFIGS[name]
        x = W.input_vector(T, name)
        lv = [3] + levels if kind == "dyadic" else levels
        assert np.array_equal(x, O.random_vector(lv, seed, 0.5)), name
    try:
        R = oracle.RefLib()
    except FileNotFoundError:
        return
    levels = W.CONFIGS["c1"][0]
    assert np.array_equal(W.input_vector(T, "c1"), R.random_vector([3] + levels, 2, 0.5))
