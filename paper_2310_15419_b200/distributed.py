"""Multi-GPU sharding of the sketch -- host-side plumbing only.

Rows of A (= columns of S) are split into contiguous ranges [r_g, r_{g+1}); rank g plans its
local CSC with ``row_offset = r_g`` so the Philox keys use GLOBAL row indices and every rank
regenerates only its own columns of S from the shared seed (the CBRNG property of
PAPER.md:489-492, 511 that makes the partition invisible in the result).  Each rank produces
a full d x n partial Â_g = S[:, r_g:r_{g+1}] · A[r_g:r_{g+1}, :], and one collective sums them:
Â = Σ_g Â_g (NCCL over NVLink / NVSwitch; ``gloo`` in the CPU tests).  This is the outer-loop
parallelism of PAPER.md:327-332 moved from threads to GPUs, along the inner dimension m that
Algorithm 1 leaves unblocked.

Column sharding is the zero-communication alternative: rank g owns the
columns [c_g, c_{g+1}) of A (and of Â), split at nnz quantiles so skewed column lengths (config
c3's power law) still balance, and computes its d x (c_{g+1} - c_g) block of Â over all rows with
no reduction at all; an all_gather assembles Â only if a consumer needs it on every rank.  Each
rank then reads only its columns' nonzeros but needs every row of A they touch.

`sketch_row_sharded_overlapped` is the row-sharded form with the reduction overlapped with the
compute: the columns are processed in groups, and group g's all_reduce (on a communication stream)
runs while group g + 1 is being sketched.
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


def _host_staged(t, group=None) -> bool:
    """True when the group's backend cannot run this collective on a CUDA tensor directly (gloo
    implements only broadcast / all_reduce for CUDA tensors): the call then goes through a host copy."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def reduce_partials(out, group=None, mode: str = "all_reduce", dst: int = 0):
    """Â = Σ_g Â_g across the process group (in place).  ``mode`` is "all_reduce" (every
    rank gets Â) or "reduce" (rank ``dst`` only)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return out
    if mode == "all_reduce":
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    elif mode == "reduce":
        if _host_staged(out, group):
            h = out.cpu()
            dist.reduce(h, dst=dst, op=dist.ReduceOp.SUM, group=group)
            if dist.get_rank(group) == dst:
                out.copy_(h)
        else:
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


def balanced_col_shards(colptr, world: int):
    """Column boundaries [c_0 = 0, ..., c_world = n] at nnz quantiles of the CSC colptr (every
    rank gets about nnz / world nonzeros; boundaries are non-decreasing, ranks may be empty)."""
    colptr = np.asarray(colptr, dtype=np.int64)
    n = colptr.shape[0] - 1
    total = int(colptr[-1] - colptr[0])
    b = [0]
    for g in range(1, world):
        target = int(colptr[0]) + (total * g) // world
        c = int(np.searchsorted(colptr, target, side="left"))
        b.append(max(b[-1], min(c, n)))
    b.append(n)
    return b


def col_shard_csc(colptr, rowidx, vals, c0: int, c1: int):
    """Columns [c0, c1) of a CSC matrix as (colptr rebased to 0, rowidx, vals) views/copies."""
    colptr = np.asarray(colptr, dtype=np.int64)
    p0, p1 = int(colptr[c0]), int(colptr[c1])
    return colptr[c0:c1 + 1] - p0, rowidx[p0:p1], vals[p0:p1]


def gather_col_blocks(block, bounds, group=None):
    """All-gather the (c_{g+1} - c_g, d) blocks (torch (n_g, d) = column-major d x n_g) of every
    rank into the full (n, d) Â on every rank."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return block
    world = dist.get_world_size(group)
    d = block.shape[1]
    widths = [bounds[g + 1] - bounds[g] for g in range(world)]
    wmax = max(max(widths), 1)
    staged = _host_staged(block, group)
    pad = torch.zeros((wmax, d), dtype=block.dtype, device="cpu" if staged else block.device)
    pad[:block.shape[0]].copy_(block)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:w] for o, w in zip(outs, widths)], dim=0).to(block.device)


def sketch_col_sharded(colptr_local, rowidx_local, vals_local, d: int, m: int, seed: int, dist_name: str,
                       plan=None, out=None):
    """One rank's part of the column-sharded sketch: its columns of Â over all m rows (no
    collective).  colptr_local is rebased to 0; returns (out (n_local, d), plan)."""
    from . import sketch as sk
    if plan is None:
        dtype = "f64" if str(vals_local.dtype) == "torch.float64" else "f32"
        plan = sk.Plan(colptr_local, rowidx_local, d, m, dtype)
    return plan.apply(vals_local, seed, dist_name, out=out), plan


def overlap_groups(colptr, groups: int, group=None, device=None):
    """Column groups [g_0 = 0, ..., g_G = n] with balanced nnz for the overlapped reduction.  Under an
    initialised process group the per-column counts are summed across ranks first, so every rank
    cuts the same groups (each group is one collective of identical size on every rank)."""
    colptr = np.asarray(colptr, dtype=np.int64)
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        import torch
        cnt = torch.from_numpy(np.diff(colptr))
        if dist.get_backend(group) == "nccl":
            cnt = cnt.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
        colptr = np.concatenate([[0], np.cumsum(cnt.cpu().numpy())])
    return balanced_col_shards(colptr, groups)


def sketch_row_sharded_overlapped(colptr_h, colptr, rowidx, vals, d: int, m_local: int, row_offset: int,
                                  seed: int, dist_name: str, groups: int = 4, group=None, out=None):
    """Row-sharded sketch whose cross-GPU sum overlaps the compute: the columns are sketched in
    `groups` nnz-balanced groups (the same on every rank) on the current stream, and each group's all_reduce is issued on a
    side stream as soon as that group's kernel is done.  colptr_h is the host copy of colptr.
    Returns out (n, d) after all reductions completed on the current stream."""
    import torch
    import torch.distributed as dist
    from . import sketch as sk
    n = len(colptr_h) - 1
    if out is None:
        out = torch.empty((n, d), dtype=vals.dtype, device=vals.device)
    bounds = overlap_groups(colptr_h, groups, group=group, device=vals.device)
    comp = torch.cuda.current_stream()
    comm = torch.cuda.Stream()
    dtype = "f64" if vals.dtype == torch.float64 else "f32"
    plans, works = [], []
    for g in range(len(bounds) - 1):
        c0, c1 = bounds[g], bounds[g + 1]
        if c1 == c0:
            continue
        p0, p1 = int(colptr_h[c0]), int(colptr_h[c1])
        cp = colptr[c0:c1 + 1] - p0
        pl = sk.Plan(cp, rowidx[p0:p1], d, m_local, dtype, row_offset=row_offset)
        plans.append(pl)
        pl.apply(vals[p0:p1], seed, dist_name, out=out[c0:c1])
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            ev = torch.cuda.Event()
            ev.record(comp)
            with torch.cuda.stream(comm):
                comm.wait_event(ev)
                dist.all_reduce(out[c0:c1], op=dist.ReduceOp.SUM, group=group)
    comp.wait_stream(comm)
    for pl in plans:
        pl.close()
    return out


def sketch_row_sharded_e2e(h_colptr, h_rowidx, h_vals, d: int, m_local: int, row_offset: int, seed: int,
                           dist_name: str, out_host, group=None, work=None):
    """End-to-end row-sharded sketch from HOST buffers (the bench's ``e2e`` leg at N > 1): this rank's
    shard goes through ``sketch_apply_host`` (pinned host A -> device, plan, fused apply, column groups
    pipelined on copy streams) into a device buffer, the d x n partials are summed across ranks, and Â
    comes back into ``out_host`` (pinned, (n, d)).  ``work`` is an optional device (n, d) buffer to reuse.
    Returns out_host."""
    import torch
    from . import sketch as sk
    n = len(h_colptr) - 1
    if work is None:
        work = torch.empty((n, d), dtype=out_host.dtype, device="cuda")
    sk.sketch_apply_host(seed, dist_name, d, m_local, h_colptr, h_rowidx, h_vals, out=work, row_offset=row_offset)
    reduce_partials(work, group=group, mode="all_reduce")
    out_host.copy_(work)
    return out_host
