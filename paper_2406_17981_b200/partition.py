"""Branch partitioning across GPUs, one process per GPU (torchrun layout).

The 2^d leaves of the split recursion are independent:
    y = 2^{-d} sum_b conj(P^b) F^{-1}(T[b] F(P^b x)).
Rank r of a world of P = 2^q ranks owns the subtree of branch ids whose low q
bits equal r (the axes split first), stores only its spectra blocks
(ts_split_options.part / nparts) and produces that subtree's projected partial
output; the partials are summed by an NCCL reduce (the paper's outlook,
PAPER.md:97-99).

``PartitionedOperator`` is the per-rank driver: it builds the rank's
partition operator, joins a library-owned NCCL communicator (the unique id
travels over the caller's torch.distributed group) and applies through
``ts_operator_apply_device_comm``, which broadcasts x, runs the subtree and
reduces the partials component by component, overlapping the reduce with the
last inverse-merge pass — all inside libtoesplit. The helpers below it are the
partition arithmetic (validated on CPU with gloo).
"""
from __future__ import annotations


def check_world(world: int, d: int) -> int:
    """Return q = log2(world); world must be a power of two <= 2^d."""
    if world < 1 or world & (world - 1):
        raise ValueError(f"world size {world} must be a power of two")
    q = world.bit_length() - 1
    if q > d:
        raise ValueError(f"at most 2^d = {2 ** d} ranks (one branch each)")
    return q


def owned_branches(rank: int, world: int, d: int) -> list[int]:
    """Branch ids (bit a = odd along axis a) owned by `rank`."""
    check_world(world, d)
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return [b for b in range(2 ** d) if b & (world - 1) == rank]


def path_bits(rank: int, world: int) -> list[int]:
    """Parity taken at each of the q single-child path levels (axes 0..q-1)."""
    q = world.bit_length() - 1
    return [(rank >> a) & 1 for a in range(q)]


def per_gpu_vector_passes(d: int, world: int) -> int:
    """HBM passes over the vector per GPU (units of c*s*S_e), SURVEY.md §8(e):
    4q + T(m) with T(m) = 4*2^m - 6 for m = d - q >= 1, and 4q - 2 for m = 0."""
    q = check_world(world, d)
    m = d - q
    return 4 * q + (4 * 2 ** m - 6) if m >= 1 else 4 * q - 2


def reduce_partials(y, dst: int = 0, group=None):
    """Sum the ranks' partial outputs into rank `dst` with torch.distributed
    (gloo in the CPU tests; the GPU path reduces inside the library)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(y, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return y


def exchange_unique_id(rank: int, make_id, group=None) -> bytes:
    """Rank 0's NCCL unique id on every rank (over the torch.distributed group)."""
    import torch.distributed as dist

    box = [make_id() if rank == 0 else None]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast_object_list(box, src=0, group=group)
    return box[0]


class PartitionedOperator:
    """This rank's share of a split operator plus the library communicator.

    build(bg) receives the rank's (part, nparts, device) and returns the
    partition operator (e.g. workloads.make_operator); apply(x, y) computes
    y = T x on root (x replicated, or broadcast from root with bcast_x)."""

    def __init__(self, T, build, rank: int, world: int, device: int, d: int, group=None):
        check_world(world, d)
        self.T = T
        self.rank, self.world, self.device = rank, world, device
        self.op = build(rank, world, device)
        uid = exchange_unique_id(rank, T.Comm.unique_id, group)
        self.comm = T.Comm(uid, world, rank, device)

    def info(self):
        return self.op.info()

    def apply(self, x, y, stream=None, bcast_x=False, root=0, metrics=False):
        return self.op.apply_device_comm(self.comm, x, y, root=root, bcast_x=bcast_x,
                                         stream=stream, metrics=metrics)

    def close(self):
        self.comm.close()
        self.op.close()
