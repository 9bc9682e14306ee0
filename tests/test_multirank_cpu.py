"""World-size-2 (and 4) tests of the multi-GPU path's host logic with the
gloo backend: each rank owns the branch subtree of partition.owned_branches,
computes its projected partial output (here with the CPU oracle — the GPU
ranks do it with ts_operator_create_split_ex(part, nparts)), and
partition.reduce_partials sums the partials into rank 0, which must equal the
whole-tree product. Rendezvous on 127.0.0.1.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_17981_b200 import partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, levels, sym, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        O = oracle.Oracle()
        lags = O.random_lags(levels, 3, 1.0, sym)
        v = O.random_vector(levels, 3, 1.0)
        comp = sym != 0
        signs = oracle.axis_signs(len(levels), sym)
        blocks = O.precompute(levels, lags, 0j, comp, signs)
        part = O.split_apply_partial(levels, blocks, v, rank, world, comp, signs)
        y = torch.from_numpy(part.view(np.float64).copy())
        partition.reduce_partials(y, dst=0)
        if rank == 0:
            full = O.split_apply(levels, blocks, v, comp, signs)
            err = np.linalg.norm(y.numpy().view(np.complex128) - full) / np.linalg.norm(full)
            out.put(float(err))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("sym", [0, 1])
def test_partition_reduce_over_gloo(world, sym):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, [4, 6, 5], sym, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=5) <= 1e-13


def test_partition_logic():
    assert partition.check_world(8, 3) == 3
    with pytest.raises(ValueError):
        partition.check_world(3, 3)
    with pytest.raises(ValueError):
        partition.check_world(16, 3)
    seen = []
    for r in range(4):
        own = partition.owned_branches(r, 4, 3)
        assert len(own) == 2 and all(b & 3 == r for b in own)
        seen += own
    assert sorted(seen) == list(range(8))
    assert partition.path_bits(5, 8) == [1, 0, 1]
    # SURVEY.md §8(e) per-GPU vector traffic table
    assert [partition.per_gpu_vector_passes(3, p) for p in (1, 2, 4, 8)] == [26, 14, 10, 10]
    assert [partition.per_gpu_vector_passes(4, p) for p in (1, 2, 4, 8)] == [58, 30, 18, 14]


def _lib_worker(rank, world, port, out):
    """One rank: this library's partition operator (part = rank) on cuda:0,
    partial output to the host, summed over gloo. (Every rank uses the one
    test GPU for its own independent kernels; the reduce is on the CPU, so no
    rank's kernels wait on another's.)"""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2406_17981_b200 as T

        levels = [8, 6, 16]
        bg = T.BlockGenerator.dyadic(levels)
        x = oracle.Oracle().random_vector([3] + levels, 9, 0.5)
        op = T.Operator.split_ex(bg, precision=T.C128, part=rank, nparts=world)
        y = torch.from_numpy(op.apply(x).view(np.float64).copy())
        partition.reduce_partials(y, dst=0)
        if rank == 0:
            s = int(np.prod(levels))
            ys = np.concatenate(oracle.Oracle().dyadic_apply(levels, [x[i * s:(i + 1) * s] for i in range(3)],
                                                             mode="signs"))
            got = y.numpy().view(np.complex128)
            out.put(float(np.linalg.norm(got - ys) / np.linalg.norm(ys)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_library_partials_reduce_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lib_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=5) <= 1e-12
