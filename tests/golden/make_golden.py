"""Regenerate the golden fixtures from the UNMODIFIED reference library
(oracle/_ref/libtoesplit_ref.so, compiled from /root/reference/proj by
oracle/Makefile against the FFTW-API shim). Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

Fixtures are small (.npz); every value in them comes out of the reference's
own C ABI (ts_generator_random / ts_random_vector / ts_operator_apply /
ts_naive_matvec), so tests that compare against them pin both the oracle
restatement and the B200 engine to the reference itself.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    R = oracle.RefLib()
    O = oracle.Oracle()
    # configs[0]: d=3, 16^3, general, lags seed 0, x seed 1, CN(0,1) = variance 0.5
    lv = [16, 16, 16]
    g = R.generator(lv, seed=0, symmetry=0, variance=0.5)
    x = R.random_vector(lv, 1, 0.5)
    op = R.split(g)
    y, m = R.apply(op, x, metrics=True)
    yp = R.apply(op, x, parallel=8)
    assert yp.tobytes() == y.tobytes()
    yn = R.naive(g, x)
    lags = O.random_lags(lv, 0, 0.5, 0)
    np.savez_compressed(os.path.join(OUT, "c0_16cubed.npz"), x=x, y_split_ref=y, y_naive_ref=yn,
                        lags_sum=lags.sum(), lags_head=lags[:8],
                        counters=np.array([m.fft_forward, m.fft_inverse, m.diag_mults,
                                           m.phase_mults, m.peak_live_elems, m.kernel_elems]))
    # symmetric / skew / mixed-length scalar instances through the reference
    cases = {}
    for name, lv, sym, seed in [("sym_345", [3, 4, 5], 1, 7), ("skew_444", [4, 4, 4], 2, 8),
                                ("gen_prime", [7, 5, 3], 0, 9), ("gen_d4", [3, 2, 4, 2], 0, 10)]:
        g = R.generator(lv, seed=seed, symmetry=sym)
        x = R.random_vector(lv, seed)
        op = R.split(g)
        cases[name + "_x"] = x
        cases[name + "_y"] = R.apply(op, x)
        cases[name + "_ye"] = R.apply(R.embed(g), x)
        cases[name + "_levels"] = np.array(lv)
        cases[name + "_sym"] = np.array(sym)
        cases[name + "_seed"] = np.array(seed)
    np.savez_compressed(os.path.join(OUT, "scalar_cases.npz"), **cases)
    # 3x3 dyadic (configs[1] kernel) at n = 6, composed the reference's way:
    # G_ii symmetric (auto-compressed), G_ij general, 9 applies
    lv = [6, 6, 6]
    s = 216
    xall = O.random_vector([3] + lv, 2, 0.5)
    xs = [xall[i * s:(i + 1) * s] for i in range(3)]
    ys = R.dyadic_apply(lv, xs, O)
    np.savez_compressed(os.path.join(OUT, "dyadic_6cubed.npz"), x=xall, y=np.concatenate(ys))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
