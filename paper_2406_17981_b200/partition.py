"""Host-side branch partitioning across GPUs (one process per GPU).

The 2^d leaves of the split recursion are independent:
    y = 2^{-d} sum_b conj(P^b) F^{-1}(T[b] F(P^b x)).
Rank r of a world of P = 2^q ranks owns the subtree of branch ids whose low q
bits equal r (the axes split first), stores only its spectra blocks
(ts_split_options.part / nparts) and produces that subtree's projected partial
output; the partials are summed with one NCCL reduce (the paper's outlook,
PAPER.md:97-99). This module holds the pure logic (validated on CPU with gloo)
and the reduce wrapper the bench uses.
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
    """Sum the ranks' partial outputs into rank `dst` (torch.distributed;
    NCCL on GPUs, gloo in CPU tests). y is reduced in place."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(y, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return y
