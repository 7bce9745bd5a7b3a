"""Multi-GPU row sharding of the sketch -- host-side plumbing only.

Rows of A (= columns of S) are split into contiguous ranges [r_g, r_{g+1}); rank g plans its
local CSC with ``row_offset = r_g`` so the Philox keys use GLOBAL row indices and every rank
regenerates only its own columns of S from the shared seed (the CBRNG property of
PAPER.md:489-492, 511 that makes the partition invisible in the result).  Each rank produces
a full d x n partial Â_g = S[:, r_g:r_{g+1}] · A[r_g:r_{g+1}, :], and one collective sums them:
Â = Σ_g Â_g (NCCL over NVLink / NVSwitch; ``gloo`` in the CPU tests).  This is the outer-loop
parallelism of PAPER.md:327-332 moved from threads to GPUs, along the inner dimension m that
Algorithm 1 leaves unblocked.
"""
from __future__ import annotations

import numpy as np


def shard_range(m: int, world: int, rank: int):
    """Contiguous rows [floor(g m / G), floor((g+1) m / G)) of rank g."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return (rank * m) // world, ((rank + 1) * m) // world


def balanced_row_shards(row_nnz, world: int):
    """Shard boundaries at nnz quantiles of the per-row nonzero histogram (for skewed rows).
    Returns world + 1 non-decreasing boundaries with b[0] = 0 and b[-1] = m."""
    row_nnz = np.asarray(row_nnz, dtype=np.int64)
    m = row_nnz.shape[0]
    csum = np.concatenate([[0], np.cumsum(row_nnz)])
    total = csum[-1]
    b = [0]
    for g in range(1, world):
        target = (total * g) // world
        r = int(np.searchsorted(csum, target, side="left"))
        b.append(max(b[-1], min(r, m)))
    b.append(m)
    return b


def reduce_partials(out, group=None, mode: str = "all_reduce", dst: int = 0):
    """Â = Σ_g Â_g across the process group (in place).  ``mode`` is "all_reduce" (every
    rank gets Â) or "reduce" (rank ``dst`` only)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return out
    if mode == "all_reduce":
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    elif mode == "reduce":
        dist.reduce(out, dst=dst, op=dist.ReduceOp.SUM, group=group)
    else:
        raise ValueError(mode)
    return out


def sketch_row_sharded(colptr, rowidx, vals, d: int, m_local: int, row_offset: int, seed: int,
                       dist_name: str, group=None, mode: str = "all_reduce", out=None, plan=None):
    """One rank's part of the sharded sketch: fused kernel on the local rows, then the
    cross-GPU sum.  Returns (out, plan); pass ``plan`` back in to reuse it."""
    from . import sketch as sk
    if plan is None:
        dtype = "f64" if str(vals.dtype) == "torch.float64" else "f32"
        plan = sk.Plan(colptr, rowidx, d, m_local, dtype, row_offset=row_offset)
    out = plan.apply(vals, seed, dist_name, out=out)
    reduce_partials(out, group=group, mode=mode)
    return out, plan
