"""TSKF kernel-spectra files (ref proj/src/core/kernel.cpp:456-537, format
proj/README.md:158-170): interoperability with the reference library in both
directions (version 1: scalar complex128 whole-tree operators) and round trips
of this library's version 2 (complex64, 3x3 blocks, per-axis signs,
partitions).
"""
import os
import tempfile

import numpy as np
import pytest

import oracle
import paper_2406_17981_b200 as T
from oracle import rel_l2

pytestmark = pytest.mark.gpu

O = oracle.Oracle()


def _ref():
    try:
        return oracle.RefLib()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("levels,sym", [([4, 6], T.SYM_GENERAL), ([5, 4, 3], T.SYM_SYMMETRIC),
                                        ([4, 4, 4], T.SYM_SKEW), ([3, 2, 4, 2], T.SYM_GENERAL)])
def test_reference_written_file_loads_here(levels, sym):
    R = _ref()
    g = R.generator(levels, seed=21, symmetry=sym, variance=1.0)
    rop = R.split(g)
    v = R.random_vector(levels, 21, 1.0)
    y_ref = R.apply(rop, v)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "ref.tskf")
        R._ok(R.L.ts_operator_save_kernel(rop, p.encode()))
        op = T.Operator.load_split(p)
        assert op.levels == levels
        k = np.zeros(1, np.uint64)
        R._ok(R.L.ts_operator_kernel_elems(rop, k.ctypes.data_as(oracle.C.POINTER(oracle.C.c_uint64))))
        assert op.kernel_elems == int(k[0])
        y = op.apply(v)
    assert rel_l2(y, y_ref) <= 1e-12
    R.destroy_op(rop)
    R.destroy_gen(g)


@pytest.mark.parametrize("levels,sym", [([4, 6], T.SYM_GENERAL), ([5, 4, 3], T.SYM_SYMMETRIC),
                                        ([4, 4, 4], T.SYM_SKEW)])
def test_file_written_here_loads_in_reference(levels, sym):
    R = _ref()
    g = T.Generator.random(levels, 23, 1.0, sym)
    op = T.Operator.split(g)
    v = T.random_vector(levels, 23, 1.0)
    y = op.apply(v)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "b200.tskf")
        op.save_kernel(p)
        with open(p, "rb") as f:
            assert f.read(8) == b"TSKF\x01\x00\x00\x00"  # version 1, the reference's
        rop = oracle.C.c_void_p()
        R._ok(R.L.ts_operator_load_split(p.encode(), oracle.C.byref(rop)))
        y_ref = R.apply(rop, v)
        R.destroy_op(rop)
    assert rel_l2(y, y_ref) <= 1e-12


@pytest.mark.parametrize("prec,storage", [(T.C64, T.STORAGE_AUTO), (T.C64, T.STORAGE_FULL),
                                          (T.C128, T.STORAGE_AUTO)])
def test_v2_round_trip_dyadic_blocks(prec, storage):
    levels = [8, 6, 16]
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=prec, storage=storage)
    x = O.random_vector([3] + levels, 5, 0.5)
    y = op.apply(x)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "g.tskf")
        op.save_kernel(p)
        with open(p, "rb") as f:
            assert f.read(8) == b"TSKF\x02\x00\x00\x00"
        op2 = T.Operator.load_split(p)
        i1, i2 = op.info(), op2.info()
        for k in ("m", "n_unique", "precision", "storage", "spectra_bytes"):
            assert i1[k] == i2[k], k
        assert op2.apply(x).tobytes() == y.tobytes()


@pytest.mark.parametrize("nparts", [2, 4])
def test_v2_round_trip_partitions(nparts):
    levels = [8, 8, 8]
    bg = T.BlockGenerator.dyadic(levels)
    x = O.random_vector([3] + levels, 6, 0.5)
    y_full = T.Operator.split_ex(bg, precision=T.C64).apply(x)
    acc = np.zeros_like(y_full)
    with tempfile.TemporaryDirectory() as td:
        for part in range(nparts):
            op = T.Operator.split_ex(bg, precision=T.C64, part=part, nparts=nparts)
            p = os.path.join(td, f"p{part}.tskf")
            op.save_kernel(p)
            op2 = T.Operator.load_split(p)
            assert op2.info()["part"] == part and op2.info()["nparts"] == nparts
            yp = op2.apply(x)
            assert yp.tobytes() == op.apply(x).tobytes()
            acc += yp
    assert rel_l2(acc, y_full) <= 1e-5


def test_corrupt_files_map_to_reference_status_codes():
    levels = [4, 4]
    op = T.Operator.split(T.Generator.random(levels, 3, 1.0, T.SYM_GENERAL))
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "k.tskf")
        op.save_kernel(p)
        raw = open(p, "rb").read()
        bad = os.path.join(td, "bad.tskf")
        open(bad, "wb").write(b"XXXX" + raw[4:])
        with pytest.raises(T.TsError) as e:
            T.Operator.load_split(bad)
        assert e.value.code == T.TS_ERR_IO
        open(bad, "wb").write(raw[:-9])  # truncated
        with pytest.raises(T.TsError) as e:
            T.Operator.load_split(bad)
        assert e.value.code == T.TS_ERR_IO
