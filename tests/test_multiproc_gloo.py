"""World-size-2 `gloo` tests (CPU) of the multi-GPU host logic: row shards keyed by global
rows, partials summed by the product's reduce_partials, result equal to the unsharded
sketch.  The per-rank partial is computed by the oracle here (no GPU on this box); on the
GPU box the same shards go through libsketch (tests/test_gpu_parity.py::test_row_offset_and_shards)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads
from paper_2310_15419_b200.distributed import balanced_row_shards, reduce_partials, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = workloads.random_csc(3000, 9, 40, seed=21)
        r0, r1 = shard_range(A.m, world, rank)
        Ag = workloads.shard_csc(A, world, rank)
        assert (Ag.row_offset, Ag.row_offset + Ag.m) == (r0, r1)
        part, _ = oracle.sketch(5, "uniform", 120, Ag.m, Ag.n, Ag.colptr, Ag.rowidx, Ag.vals,
                                row_offset=Ag.row_offset, want_bound=False)
        t = torch.from_numpy(np.ascontiguousarray(part))
        reduce_partials(t, mode=mode, dst=0)
        if mode == "all_reduce" or rank == 0:
            q.put((rank, t.numpy()))
        else:
            q.put((rank, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["all_reduce", "reduce"])
def test_row_sharded_sum_equals_full_sketch(mode):
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = workloads.random_csc(3000, 9, 40, seed=21)
    full, B = oracle.sketch(5, "uniform", 120, A.m, A.n, A.colptr, A.rowidx, A.vals)
    for r, v in res.items():
        if v is None:
            continue
        assert np.all(np.abs(v - full) <= 1e-14 * B)


def test_shard_ranges_partition_rows():
    for m in (0, 1, 7, 50_000_000):
        for world in (1, 2, 3, 8):
            rs = [shard_range(m, world, g) for g in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert rs == [workloads.shard_rows(m, world, g) for g in range(world)]


def test_balanced_shards_follow_nnz_quantiles():
    rng = np.random.default_rng(0)
    row_nnz = rng.zipf(1.8, size=10000).clip(max=500)
    b = balanced_row_shards(row_nnz, 4)
    assert b[0] == 0 and b[-1] == 10000 and all(x <= y for x, y in zip(b, b[1:]))
    parts = [row_nnz[b[g]:b[g + 1]].sum() for g in range(4)]
    assert max(parts) - min(parts) <= 2 * row_nnz.max()


def test_c5_shards_are_generated_consistently():
    # any row shard of c5 is produced identically and independently (chunked seeds):
    # the union of 3 shards equals the full generation of the same rows
    cfg = workloads.CONFIGS["c5"]
    rows = (0, 3_000_000)
    full = workloads.make_config("c5", row_range=rows)
    parts = [workloads.make_config("c5", row_range=(rows[0] + a, rows[0] + b))
             for a, b in [(0, 1_000_003), (1_000_003, 2_500_000), (2_500_000, 3_000_000)]]
    dense_cols = np.empty(rows[1] - rows[0], dtype=np.int64)
    dense_vals = np.empty(rows[1] - rows[0])
    for P in parts:
        for k in range(P.n):
            r, v = P.column(k)
            dense_cols[P.row_offset - rows[0] + r] = k
            dense_vals[P.row_offset - rows[0] + r] = v
    for k in range(full.n):
        r, v = full.column(k)
        assert np.all(dense_cols[r] == k) and np.array_equal(dense_vals[r], v)
    assert full.nnz == rows[1] - rows[0] and full.n == cfg.n


# ---------------------------------------------------------------- column sharding (§8(f) f4)

def _col_worker(rank, world, port, q):
    import oracle
    from paper_2310_15419_b200.distributed import balanced_col_shards, col_shard_csc, gather_col_blocks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = workloads.random_csc(4000, 11, [5, 300, 0, 40, 2, 900, 7, 0, 60, 33, 1], seed=23)
        b = balanced_col_shards(A.colptr, world)
        cp, ri, va = col_shard_csc(A.colptr, A.rowidx, A.vals, b[rank], b[rank + 1])
        part, _ = oracle.sketch(9, "gaussian", 77, A.m, b[rank + 1] - b[rank], cp, ri, va, want_bound=False)
        block = torch.from_numpy(np.ascontiguousarray(part.T))            # (n_local, d): column-major Â block
        full = gather_col_blocks(block, b)
        q.put((rank, full.numpy().T.copy()))
    finally:
        dist.destroy_process_group()


def test_col_sharded_blocks_assemble_the_full_sketch():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_col_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A = workloads.random_csc(4000, 11, [5, 300, 0, 40, 2, 900, 7, 0, 60, 33, 1], seed=23)
    full, _ = oracle.sketch(9, "gaussian", 77, A.m, A.n, A.colptr, A.rowidx, A.vals)
    for r, v in res.items():
        assert np.array_equal(v, full)          # same per-column order on both sides: bit-identical


def test_balanced_col_shards_split_nnz():
    from paper_2310_15419_b200.distributed import balanced_col_shards
    rng = np.random.default_rng(1)
    lens = rng.zipf(1.5, size=3000).clip(max=20000)
    colptr = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 3, 8):
        b = balanced_col_shards(colptr, world)
        assert b[0] == 0 and b[-1] == 3000 and len(b) == world + 1
        assert all(x <= y for x, y in zip(b, b[1:]))
        parts = [int(colptr[b[g + 1]] - colptr[b[g]]) for g in range(world)]
        assert sum(parts) == int(colptr[-1])
        assert max(parts) - min(parts) <= 2 * int(lens.max())


# ---------------------------------------------------------------- overlapped reduce: same groups on every rank

def _groups_worker(rank, world, port, q):
    from paper_2310_15419_b200.distributed import overlap_groups
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # row shards whose per-column nnz differ by rank: rank 0's mass sits in the first columns,
        # rank 1's in the last, so locally balanced groups would differ and the collectives mismatch
        lens = [4000, 10, 10, 10, 10, 10, 10, 4000] if rank == 0 else [10, 10, 10, 10, 10, 10, 3000, 9000]
        colptr = np.concatenate([[0], np.cumsum(lens)])
        q.put((rank, overlap_groups(colptr, 4)))
    finally:
        dist.destroy_process_group()


def test_overlap_groups_agree_across_ranks():
    from paper_2310_15419_b200.distributed import balanced_col_shards
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_groups_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    total = np.array([4010, 20, 20, 20, 20, 20, 3010, 13000])
    assert res[0] == balanced_col_shards(np.concatenate([[0], np.cumsum(total)]), 4)
