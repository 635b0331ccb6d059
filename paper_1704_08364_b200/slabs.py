"""Slab sharding of a sinogram volume over ranks (one process per GPU).

Slices are independent (the reference maps its Q-blocks with no cross-slice
state, pipeline.py:395-400, 552-554), so a volume of S slices is split into
contiguous z-slabs, one per rank; the data path has no collective.  The only
cross-rank operations are the timing barrier / MAX reduction of bench.py and,
optionally, a final gather of the image slabs to rank 0 (object collective on
host tensors, not on the hot path).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def split(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous [begin, end) slabs of n items over `parts` owners (the
    first n % parts owners take one extra item)."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    base, extra = divmod(n, parts)
    out, b = [], 0
    for p in range(parts):
        e = b + base + (1 if p < extra else 0)
        out.append((b, e))
        b = e
    return out


def rank_slab(n: int, world: int, rank: int) -> tuple[int, int]:
    """This rank's slab [begin, end) of an n-slice volume."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return split(n, world)[rank]


def _initialized() -> bool:
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(x: float, device=None) -> float:
    """MAX all-reduce of one float (per-rank device time -> job time)."""
    if not _initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_slabs(local: torch.Tensor, n: int, dst: int = 0) -> torch.Tensor | None:
    """Collect every rank's image slab [slab][n_out][n_out] into the full
    volume on rank `dst` (None elsewhere).  Host-side object gather: outside
    the timed hot path."""
    if not _initialized() or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    parts = [None] * world if rank == dst else None
    dist.gather_object(local.cpu(), parts, dst=dst)
    if rank != dst:
        return None
    slabs = split(n, world)
    vol = torch.empty((n,) + tuple(local.shape[1:]), dtype=local.dtype)
    for (b, e), part in zip(slabs, parts):
        if part.shape[0] != e - b:
            raise RuntimeError("slab size mismatch")
        vol[b:e] = part
    return vol
