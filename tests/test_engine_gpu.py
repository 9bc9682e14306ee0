"""GPU tests of the engine around the kernels: per-stream apply contexts
(workspace kept across calls), CUDA-graph replay of small operators, the
multi-RHS batched apply, the device-memory meter, argument validation, and
the NCCL paths of the library (one-process-many-GPU operator and the
per-rank communicator) on the single GPU a test box has. Results are
compared bit for bit with the direct single-vector path, which the parity
tests pin to the oracle.
"""
import numpy as np
import pytest

import oracle
import paper_2406_17981_b200 as T
from oracle import rel_l2

pytestmark = pytest.mark.gpu

O = oracle.Oracle()


def _dev(a, prec):
    import torch

    dt = torch.complex64 if prec == T.C64 else torch.complex128
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dt)


def _dyadic_x(levels, seed, nrhs=1):
    return O.random_vector([nrhs, 3] + list(levels), seed, 0.5)


def test_graph_replay_bit_identical_and_counted():
    import torch

    levels = [32, 32, 64]  # 3 x 64K c64: captured as a CUDA graph from the 2nd call
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
    x = _dev(_dyadic_x(levels, 5), T.C64)
    y = torch.empty_like(x)
    outs = []
    for _ in range(5):
        op.apply_device(x, y)
        outs.append(y.clone())
    torch.cuda.synchronize()
    assert op.info()["graph_replays"] >= 3
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    # a new output buffer is a new key: direct run first, then capture
    y2 = torch.empty_like(x)
    for _ in range(3):
        op.apply_device(x, y2)
    torch.cuda.synchronize()
    assert torch.equal(y2, outs[0])
    ys = outs
    ref = np.concatenate(O.dyadic_apply(levels, np.split(_dyadic_x(levels, 5), 3), mode="signs"))
    assert rel_l2(ys[0].cpu().numpy().astype(np.complex128), ref) <= 1e-5


@pytest.mark.parametrize("levels,prec,storage", [
    ([16, 16, 512], T.C64, T.STORAGE_AUTO),     # 512-point leaf, compressed
    ([512, 16, 32], T.C64, T.STORAGE_AUTO),     # TMA strided passes over 3 x nrhs components
    ([8, 32, 256], T.C64, T.STORAGE_FULL),      # 256-point leaf, full storage
    ([4, 8, 64], T.C128, T.STORAGE_AUTO),       # complex128 leaf1
    ([5, 6, 7], T.C64, T.STORAGE_AUTO),         # generic kernels, per-RHS leaf launches
])
def test_batch_apply_bit_identical_to_single(levels, prec, storage):
    import torch

    nrhs = 3
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=prec, storage=storage)
    n = 3 * int(np.prod(levels))
    x = _dev(_dyadic_x(levels, 8, nrhs), prec)
    y = torch.empty_like(x)
    mb = op.apply_batch_device(x, y, nrhs, metrics=True)
    ys = torch.empty_like(x)
    for r in range(nrhs):
        m1 = op.apply_device(x[r * n:(r + 1) * n], ys[r * n:(r + 1) * n], metrics=True)
    torch.cuda.synchronize()
    assert torch.equal(y, ys)
    assert mb["fft_forward"] == nrhs * m1["fft_forward"]
    assert mb["diag_mults"] == nrhs * m1["diag_mults"]
    assert mb["peak_live_elems"] == nrhs * m1["peak_live_elems"]
    xs = _dyadic_x(levels, 8, nrhs)
    ref = np.concatenate(O.dyadic_apply(levels, np.split(xs[:n], 3), mode="signs"))
    tol = 1e-5 if prec == T.C64 else 1e-12
    assert rel_l2(y[:n].cpu().numpy().astype(np.complex128), ref) <= tol


def test_peak_live_elems_is_measured_schedule():
    # ref tests/unit/test_engine_split.cpp:156-206: lazy peak (d+1) s; a
    # partition holds x, y and d-1-q children
    import torch

    levels = [4, 8, 16, 8]
    s = int(np.prod(levels))
    g = T.Generator.random(levels, 3, 1.0, T.SYM_GENERAL)
    bg = T.BlockGenerator.from_scalar(g)
    x = _dev(T.random_vector(levels, 3, 1.0), T.C128)
    y = torch.empty_like(x)
    for nparts, vectors in ((1, 5), (2, 4), (4, 3), (8, 2), (16, 2)):
        op = T.Operator.split_ex(bg, part=nparts - 1, nparts=nparts)
        m = op.apply_device(x, y, metrics=True)
        assert m["peak_live_elems"] == vectors * s, (nparts, m)


def test_memory_meter_counts_library_buffers():
    import gc

    import torch

    gc.collect()
    torch.cuda.synchronize()
    levels = [64, 64, 64]
    T.reset_memory_peak(0)
    before = T.memory_stats(0)
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
    inf = op.info()
    after_create = T.memory_stats(0)
    assert after_create["live_bytes"] - before["live_bytes"] == inf["spectra_bytes"] + inf["table_bytes"]
    x = _dev(_dyadic_x(levels, 1), T.C64)
    y = torch.empty_like(x)
    op.apply_device(x, y)
    torch.cuda.synchronize()
    inf = op.info()
    st = T.memory_stats(0)
    assert inf["cached_bytes"] == inf["workspace_bytes"] == 2 * x.numel() * 8  # (d-1) children
    assert st["live_bytes"] - before["live_bytes"] == inf["spectra_bytes"] + inf["table_bytes"] + inf["cached_bytes"]
    assert st["peak_bytes"] >= st["live_bytes"]
    # the precompute's staging is in the peak: the embedded-and-folded half
    # tensor (4 s complex128; the (2n)^3 embedding itself is never stored)
    # plus the deeper fold levels, next to the spectra
    s = int(np.prod(levels))
    peak_setup = st["peak_bytes"] - before["live_bytes"]
    assert peak_setup >= inf["spectra_bytes"] + 4 * s * 16
    assert peak_setup < inf["spectra_bytes"] + 8 * s * 16
    del op
    assert T.memory_stats(0)["live_bytes"] == before["live_bytes"]


def test_device_argument_validation():
    import torch

    levels = [4, 4, 8]
    op = T.Operator.split_ex(T.BlockGenerator.dyadic(levels), precision=T.C64)
    n = 3 * 128
    x = torch.zeros(n, dtype=torch.complex64, device="cuda")
    y = torch.zeros(n, dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        op.apply_device(x.to(torch.complex128), y.to(torch.complex128))  # wrong precision
    with pytest.raises(ValueError):
        op.apply_device(x[:-1], y[:-1])  # short
    with pytest.raises(ValueError):
        op.apply_device(torch.zeros(2 * n, dtype=torch.complex64, device="cuda")[::2], y)  # strided
    with pytest.raises(ValueError):
        op.apply_device(x.cpu(), y.cpu())
    # partially overlapping x / y are refused by the library itself
    buf = torch.zeros(2 * n, dtype=torch.complex64, device="cuda")
    st = T.lib.ts_operator_apply_device(op._h, T.C.c_void_p(buf.data_ptr()),
                                        T.C.c_void_p(buf[n // 2:].data_ptr()), None, None)
    assert st == T.TS_ERR_INVALID_ARGUMENT


def test_multi_gpu_operator_on_one_device_matches_single():
    # ts_operator_create_split_multi over the GPUs a box has (1 here: the NCCL
    # communicator, broadcast and per-component reduce run with one rank)
    import torch

    levels = [16, 32, 64]
    bg = T.BlockGenerator.dyadic(levels)
    ndev = torch.cuda.device_count()
    devs = list(range(1 << (ndev.bit_length() - 1)))[:8]
    mop = T.Operator.split_multi(bg, devs, precision=T.C64)
    op = T.Operator.split_ex(bg, precision=T.C64)
    assert mop.info()["ndevices"] == len(devs)
    xs = _dyadic_x(levels, 12)
    x = _dev(xs, T.C64)
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    for _ in range(2):
        mop.apply_device(x, y1)
    op.apply_device(x, y2)
    torch.cuda.synchronize()
    assert rel_l2(y1.cpu().numpy(), y2.cpu().numpy()) <= 1e-6
    if len(devs) == 1:
        assert torch.equal(y1, y2)
    yh = mop.apply(xs)  # host ABI path through the multi-GPU operator
    assert rel_l2(yh, y2.cpu().numpy().astype(np.complex128)) <= 1e-6


def test_comm_apply_single_rank():
    # ts_comm with one rank: broadcast + per-component reduce are NCCL no-ops
    # around the same schedule as apply_device
    import torch

    levels = [8, 16, 64]
    bg = T.BlockGenerator.dyadic(levels)
    op = T.Operator.split_ex(bg, precision=T.C64, part=0, nparts=1)
    comm = T.Comm(T.Comm.unique_id(), 1, 0, 0)
    x = _dev(_dyadic_x(levels, 4), T.C64)
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    m = op.apply_device_comm(comm, x, y1, metrics=True)
    op.apply_device(x, y2)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert m["fft_forward"] == 3 * 14
    bad = T.Operator.split_ex(bg, precision=T.C64, part=1, nparts=2)
    with pytest.raises(T.TsError):
        bad.apply_device_comm(comm, x, y1)
    comm.close()


def test_multi_requires_distinct_devices():
    bg = T.BlockGenerator.dyadic([4, 4, 4])
    with pytest.raises(T.TsError) as e:
        T.Operator.split_multi(bg, [0, 0])
    assert e.value.code == T.TS_ERR_INVALID_ARGUMENT
    with pytest.raises(T.TsError):
        T.Operator.split_multi(bg, [0, 1, 2])  # not a power of two
