"""Concurrent applies of ONE operator (the reference's
SplitOperator::apply is const and may be entered from several threads,
proj/src/core/engine_split.cpp:104-135; here every stream gets its own apply
context with its own child buffers, csrc/sched.cpp acquire_ctx). Host threads
run through ctypes (the GIL is released inside the C-ABI call). The results
must be bit-identical to serial applies of the same inputs.
"""
import threading

import numpy as np
import pytest

import oracle
import paper_2406_17981_b200 as T
from oracle import rel_l2

pytestmark = pytest.mark.gpu

O = oracle.Oracle()


def _run_threads(fns):
    errs = []

    def wrap(f):
        def g():
            try:
                f()
            except BaseException as e:  # noqa: BLE001 - re-raised in the main thread
                errs.append(e)
        return g

    ts = [threading.Thread(target=wrap(f)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("levels,prec", [([64, 64, 64], T.C64), ([16, 24, 20], T.C128), ([256, 64], T.C64)])
def test_device_applies_from_threads_on_their_own_streams(levels, prec):
    import torch

    nthreads, reps = 4, 6
    g = T.Generator.random(levels, 41, 1.0, T.SYM_GENERAL)
    op = T.Operator.split_ex(T.BlockGenerator.from_scalar(g), precision=prec)
    dt = torch.complex64 if prec == T.C64 else torch.complex128
    xs = [torch.from_numpy(T.random_vector(levels, 100 + i, 1.0)).to(dt).cuda() for i in range(nthreads)]
    serial = []
    for x in xs:
        y = torch.empty_like(x)
        op.apply_device(x, y)
        serial.append(y)
    torch.cuda.synchronize()
    # the serial result itself is the oracle's (complex128 oracle, BASELINE tolerance)
    lags = O.random_lags(levels, 41, 1.0, T.SYM_GENERAL)
    blocks = O.precompute(levels, lags, 0j, False, oracle.axis_signs(len(levels), T.SYM_GENERAL))
    y_or = O.split_apply(levels, blocks, xs[0].cpu().numpy().astype(np.complex128), False,
                         oracle.axis_signs(len(levels), T.SYM_GENERAL))
    assert rel_l2(serial[0].cpu().numpy().astype(np.complex128), y_or) <= (1e-5 if prec == T.C64 else 1e-12)

    outs = [[torch.empty_like(x) for _ in range(reps)] for x in xs]
    streams = [torch.cuda.Stream() for _ in range(nthreads)]
    start = threading.Barrier(nthreads)

    def worker(i):
        def f():
            start.wait()
            for r in range(reps):
                op.apply_device(xs[i], outs[i][r], stream=streams[i])
            streams[i].synchronize()
        return f

    _run_threads([worker(i) for i in range(nthreads)])
    torch.cuda.synchronize()
    for i in range(nthreads):
        for r in range(reps):
            assert torch.equal(outs[i][r], serial[i]), (i, r)
    # the contexts the threads created stay bounded (sched.cpp: kMaxCtx = 8 per operator)
    per_ctx = max(1, (len(levels) - 1)) * xs[0].numel() * xs[0].element_size()
    assert op.info()["cached_bytes"] <= 8 * (per_ctx + 2 * xs[0].numel() * 16)


def test_device_applies_from_threads_sharing_one_stream():
    # two host threads enqueue on the SAME stream: the second one finds the stream's
    # context busy and gets a fresh one; both results are the serial ones
    import torch

    levels = [32, 48, 16]
    bg = T.BlockGenerator.dyadic(levels)
    op = T.Operator.split_ex(bg, precision=T.C64)
    n = 3 * int(np.prod(levels))
    xs = [torch.randn(n, dtype=torch.complex64, device="cuda", generator=torch.Generator("cuda").manual_seed(s))
          for s in (1, 2)]
    serial = []
    for x in xs:
        y = torch.empty_like(x)
        op.apply_device(x, y)
        serial.append(y)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    outs = [[torch.empty_like(x) for _ in range(8)] for x in xs]
    start = threading.Barrier(2)

    def worker(i):
        def f():
            start.wait()
            for r in range(8):
                op.apply_device(xs[i], outs[i][r], stream=st)
        return f

    _run_threads([worker(0), worker(1)])
    st.synchronize()
    for i in range(2):
        for r in range(8):
            assert torch.equal(outs[i][r], serial[i]), (i, r)


def test_host_abi_applies_from_threads():
    # ts_operator_apply (host buffers, the reference call) entered from several threads:
    # each call owns a stream and staging buffers for its duration
    levels = [40, 33, 36]
    g = T.Generator.random(levels, 7, 1.0, T.SYM_SYMMETRIC)
    op = T.Operator.split(g)
    vs = [T.random_vector(levels, 200 + i, 1.0) for i in range(4)]
    serial = [op.apply(v) for v in vs]
    got = [[None] * 3 for _ in vs]
    start = threading.Barrier(len(vs))

    def worker(i):
        def f():
            start.wait()
            for r in range(3):
                got[i][r] = op.apply(vs[i])
        return f

    _run_threads([worker(i) for i in range(len(vs))])
    for i in range(len(vs)):
        for r in range(3):
            assert np.array_equal(got[i][r], serial[i]), (i, r)


def test_different_operators_from_threads():
    # several operators of different shapes (power-of-two, mixed-radix and prime axes:
    # every kernel family's launcher and its per-kernel shared-memory opt-in) applied at
    # once from their own threads
    import torch

    cases = [([64, 64, 64], T.C64), ([128, 32, 64], T.C64), ([12, 40, 36], T.C128), ([13, 64, 10], T.C64),
             ([256, 256], T.C64), ([24, 16, 20], T.C64)]
    ops, xs, serial = [], [], []
    for k, (levels, prec) in enumerate(cases):
        g = T.Generator.random(levels, 60 + k, 1.0, T.SYM_GENERAL)
        ops.append(T.Operator.split_ex(T.BlockGenerator.from_scalar(g), precision=prec))
        dt = torch.complex64 if prec == T.C64 else torch.complex128
        xs.append(torch.from_numpy(T.random_vector(levels, 300 + k, 1.0)).to(dt).cuda())
        y = torch.empty_like(xs[-1])
        ops[-1].apply_device(xs[-1], y)
        serial.append(y)
    torch.cuda.synchronize()
    reps = 10
    outs = [[torch.empty_like(x) for _ in range(reps)] for x in xs]
    streams = [torch.cuda.Stream() for _ in cases]
    start = threading.Barrier(len(cases))

    def worker(i):
        def f():
            start.wait()
            for r in range(reps):
                ops[i].apply_device(xs[i], outs[i][r], stream=streams[i])
            streams[i].synchronize()
        return f

    _run_threads([worker(i) for i in range(len(cases))])
    torch.cuda.synchronize()
    for i in range(len(cases)):
        for r in range(reps):
            assert torch.equal(outs[i][r], serial[i]), (cases[i], r)


def test_large_host_abi_applies_from_threads():
    # >= 64 MB of host complex128 per call: the chunked pinned-staging transfer (csrc/transfer.cpp,
    # worker threads, shared pinned-slot pool) entered from two threads at once
    levels = [64, 128, 513]
    g = T.Generator.random(levels, 29, 1.0, T.SYM_GENERAL)
    op = T.Operator.split_ex(T.BlockGenerator.from_scalar(g), precision=T.C64)
    vs = [T.random_vector(levels, 29 + i, 1.0) for i in range(2)]
    assert vs[0].nbytes >= 64 << 20
    serial = [op.apply(v) for v in vs]
    got = [[None] * 2 for _ in vs]
    start = threading.Barrier(len(vs))

    def worker(i):
        def f():
            start.wait()
            for r in range(2):
                got[i][r] = op.apply(vs[i])
        return f

    _run_threads([worker(i) for i in range(len(vs))])
    for i in range(len(vs)):
        for r in range(2):
            assert np.array_equal(got[i][r], serial[i]), (i, r)


def test_embedding_engine_applies_from_threads():
    # the full-embedding engine (ref proj/src/core/engine_embed.cpp:113-168) shares the apply contexts
    levels = [24, 20, 18]
    g = T.Generator.random(levels, 3, 1.0, T.SYM_GENERAL)
    op = T.Operator.embed(g)
    vs = [T.random_vector(levels, 400 + i, 1.0) for i in range(3)]
    serial = [op.apply(v) for v in vs]
    got = [[None] * 4 for _ in vs]
    start = threading.Barrier(len(vs))

    def worker(i):
        def f():
            start.wait()
            for r in range(4):
                got[i][r] = op.apply(vs[i])
        return f

    _run_threads([worker(i) for i in range(len(vs))])
    for i in range(len(vs)):
        for r in range(4):
            assert np.array_equal(got[i][r], serial[i]), (i, r)
