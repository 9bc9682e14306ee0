"""The full-embedding engine on this library's own FFT passes
(ts_operator_create_embed_ex; ref proj/src/core/engine_embed.cpp:61-168): m x m
blocks, complex64 / complex128, full symbols and mirror corners with
per-component axis signs, against the CPU oracle and the split engine."""
import numpy as np
import pytest

import oracle
import paper_2406_17981_b200 as T
from oracle import max_rel, rel_l2

pytestmark = pytest.mark.gpu
O = oracle.Oracle()


def _dyadic_x(levels, seed):
    return O.random_vector([3] + list(levels), seed, 0.5)


@pytest.mark.parametrize("levels", [[6, 6, 6], [8, 5, 7], [16, 16, 16]])
@pytest.mark.parametrize("prec,tol", [(T.C128, 1e-12), (T.C64, 1e-5)])
@pytest.mark.parametrize("storage", [T.STORAGE_AUTO, T.STORAGE_FULL])
def test_dyadic_embed_vs_oracle_and_split(levels, prec, tol, storage):
    s = int(np.prod(levels))
    x = _dyadic_x(levels, 3)
    ys = np.concatenate(O.dyadic_apply(levels, [x[i * s:(i + 1) * s] for i in range(3)], mode="signs"))
    bg = T.BlockGenerator.dyadic(levels)
    emb = T.Operator.embed_ex(bg, precision=prec, storage=storage)
    inf = emb.info()
    assert inf["is_embed"] == 1 and inf["m"] == 3 and inf["n_unique"] == 6
    assert inf["storage"] == (T.STORAGE_COMPRESSED if storage == T.STORAGE_AUTO else T.STORAGE_FULL)
    ye, m = emb.apply(x, metrics=True)
    assert rel_l2(ye, ys) <= tol
    assert m["fft_forward"] == 3 * 3 and m["diag_mults"] == 8 * s * 9
    ysp = T.Operator.split_ex(bg, precision=prec).apply(x)
    assert rel_l2(ye, ysp) <= 2 * tol


@pytest.mark.parametrize("sym", [T.SYM_GENERAL, T.SYM_SYMMETRIC, T.SYM_SKEW])
def test_scalar_embed_ex_matches_reference_embed(sym):
    levels = [5, 4, 6]
    g = T.Generator.random(levels, 17, 1.0, sym)
    v = T.random_vector(levels, 17, 1.0)
    y_ref = T.Operator.embed(g).apply(v)  # the reference-ABI embed operator (c128)
    y_naive = O.naive(levels, O.random_lags(levels, 17, 1.0, sym), v)
    assert max_rel(y_ref, y_naive) <= 1e-10
    bg = T.BlockGenerator.from_scalar(g)
    assert max_rel(T.Operator.embed_ex(bg, precision=T.C128).apply(v), y_ref) <= 1e-12
    assert rel_l2(T.Operator.embed_ex(bg, precision=T.C64).apply(v), y_ref) <= 1e-5


def test_embed_long_strided_axis_1024():
    # embedded axis 0 of length 1024 runs the wide strided passes at N = 1024
    levels = [512, 4, 8]
    s = int(np.prod(levels))
    x = _dyadic_x(levels, 5)
    ys = np.concatenate(O.dyadic_apply(levels, [x[i * s:(i + 1) * s] for i in range(3)], mode="signs"))
    emb = T.Operator.embed_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
    assert rel_l2(emb.apply(x), ys) <= 1e-5


def test_embed_device_and_batch_apply():
    import torch

    levels = [8, 8, 16]
    n = 3 * int(np.prod(levels))
    emb = T.Operator.embed_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
    x = torch.from_numpy(O.random_vector([2, 3] + levels, 7, 0.5)).to(torch.complex64).cuda()
    y = torch.empty_like(x)
    emb.apply_batch_device(x, y, 2)
    y1 = torch.empty_like(x[:n])
    emb.apply_device(x[n:], y1)
    torch.cuda.synchronize()
    assert torch.equal(y[n:], y1)
    yh = emb.apply(x[:n].cpu().numpy().astype(np.complex128))
    assert rel_l2(y[:n].cpu().numpy().astype(np.complex128), yh) <= 1e-6


def test_embed_storage_errors():
    g = T.Generator.random([4, 4], 3, 1.0, T.SYM_GENERAL)
    with pytest.raises(T.TsError) as e:
        T.Operator.embed_ex(T.BlockGenerator.from_scalar(g), storage=T.STORAGE_COMPRESSED)
    assert e.value.code == T.TS_ERR_SYMMETRY
