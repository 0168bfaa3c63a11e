"""Host-side logic of the z-slab decomposition: which layers a
rank owns, which layers and checksum rows cross each slab face after a sweep,
and the reductions bench.py uses for max-over-ranks timing.  No numerics: the
halo itself moves inside libabft_stencil.so (NCCL send/recv over NVLink,
`exchange_nccl`, or device copies for a local group); this module states the
same plan so it can be checked on CPU with the gloo backend.

Buffer-layer convention of the library (include/abft_stencil.h):
a slab of zc layers lives in buffer layers 1..zc; layer 0 and zc+1 hold the
neighbours' boundary layers (the halo), or nothing at a global domain face
(the clamp of P:289-292 reuses layer 1 / zc there).
"""
from __future__ import annotations

from typing import List, Optional, Tuple


def slab(nz: int, world: int, rank: int) -> Tuple[int, int]:
    """(z_begin, z_count) of `rank`: contiguous, the first nz % world ranks get
    one layer more.  Every rank owns >= 1 layer (requires nz >= world)."""
    if not (0 <= rank < world) or nz < world:
        raise ValueError(f"cannot split {nz} layers over {world} ranks")
    base, extra = divmod(nz, world)
    z0 = rank * base + min(rank, extra)
    return z0, base + (1 if rank < extra else 0)


def weak_nz(nz_per_rank: int, world: int) -> int:
    """Global layer count of a weak-scaling run: every rank owns nz_per_rank."""
    return nz_per_rank * world


def neighbours(rank: int, world: int, periodic: bool = False) -> Tuple[Optional[int], Optional[int]]:
    """(lower, upper) neighbour rank in z, None at a global face; a periodic
    domain over several ranks closes the ring."""
    if periodic and world > 1:
        return ((rank - 1) % world, (rank + 1) % world)
    return (rank - 1 if rank > 0 else None, rank + 1 if rank + 1 < world else None)


def halo_plan(rank: int, world: int, zc: int, periodic: bool = False) -> List[Tuple[int, int, int]]:
    """(peer, send_layer, recv_layer) per face, in buffer layers: the boundary
    layer goes to the neighbour, whose boundary layer lands in the halo slot.
    The checksum rows a[layer], b[layer] (or the offline prediction rows) of the
    same layers travel with them.  Lower face first -- the order the library
    posts its sends / receives inside one NCCL group."""
    lo, hi = neighbours(rank, world, periodic)
    plan = []
    if lo is not None:
        plan.append((lo, 1, 0))
    if hi is not None:
        plan.append((hi, zc, zc + 1))
    return plan


def exchange(rank: int, plan, send_fn, recv_fn) -> None:
    """Run a halo plan with point-to-point callables that may block: on every
    face the lower rank sends first and the upper rank receives first, faces in
    plan order (lower face first), so a chain of blocking pairs cannot deadlock."""
    for peer, s_layer, r_layer in plan:
        if rank < peer:
            send_fn(peer, s_layer)
            recv_fn(peer, r_layer)
        else:
            recv_fn(peer, r_layer)
            send_fn(peer, s_layer)


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank value (bench timing: the slowest rank defines the step)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---- offline partial re-execution over slabs (recovery PARTIAL, Q28)
# The library's host logic (offline_window / partial_window / widen in
# csrc/abft_stencil.cu) stated once more so that it can be run on CPU.

def flagged_over_ranks(own_layers, nz: int, world: int):
    """The global layers any rank's window check flagged: every rank marks its
    own layers in an array indexed by global layer, max-reduced over ranks
    (the library: ncclMax in place, or bits in the IPC slots)."""
    import torch
    t = torch.zeros(nz, dtype=torch.int32)
    for z in own_layers:
        t[z] = 1
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [z for z in range(nz) if int(t[z])]


def widen(ranges, m: int, nz: int) -> List[Tuple[int, int]]:
    """Ascending inclusive ranges, each widened by m layers, clipped to the
    domain and merged where they touch."""
    out: List[Tuple[int, int]] = []
    for lo, hi in ranges:
        lo, hi = max(0, lo - m), min(nz - 1, hi + m)
        if out and lo <= out[-1][1] + 1:
            out[-1] = (out[-1][0], max(out[-1][1], hi))
        else:
            out.append((lo, hi))
    return out


def reexecution_ranges(flagged, L: int, nz: int, periodic: bool = False) -> List[Tuple[int, int]]:
    """Layers a dirty window of L sweeps re-executes: within 2 (L - 1) of a
    flagged layer (an error spreads L - 1 layers, a flag lies within that
    reach of its origin); periodic z: everything once a reach passes a face."""
    r = 2 * (L - 1)
    if periodic and flagged and (min(flagged) - r < 0 or max(flagged) + r > nz - 1):
        return [(0, nz - 1)]
    return widen([(z, z) for z in sorted(flagged)], r, nz)


def cones(ranges, k: int, L: int, nz: int) -> List[Tuple[int, int]]:
    """What sweep k (1..L) of the re-execution computes: the ranges widened by
    L - k layers, so that sweep k + 1 finds every layer it reads."""
    return widen(ranges, L - k, nz)


def local_pieces(rs, z0: int, zc: int) -> List[Tuple[int, int]]:
    """The slab-local half-open pieces [za, zb) of global inclusive ranges."""
    out = []
    for lo, hi in rs:
        za, zb = max(0, lo - z0), min(zc, hi - z0 + 1)
        if za < zb:
            out.append((za, zb))
    return out
