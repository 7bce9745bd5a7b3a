"""Multi-rank GPU tests of the cross-GPU reduce (SURVEY.md §8 a6 / e / f4): every rank's partial
comes from libsketch, goes through the real collective, and the result is compared with the oracle.

Two ranks run as two processes.  With >= 2 visible GPUs each rank owns one and the group is NCCL
(the product configuration).  On a 1-GPU box both ranks share cuda:0 and the group is gloo
(all_reduce on CUDA tensors; reduce / all_gather host-staged by distributed.py): the device-buffer ->
collective -> Â path, the stream ordering of the apply and the side communication stream, and the
in-place reduce into `out[c0:c1]` slices are the same code.  No kernel waits on another rank's
kernel, so sharing one GPU is safe (B200_PROFILING.md: only mutually-waiting kernels must not share).
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

WORLD = 2
D = 900
CASES = [("rademacher", 31), ("uniform", 32), ("gaussian", 33)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix():
    # columns long enough that each rank's row shard keeps >= 1280 nonzeros (tensor-core ±1 path), plus
    # mid-length, short and empty columns (SIMT path)
    lens = [2700 + 100 * k for k in range(12)] + [300 + 50 * k for k in range(12)] + [0, 3, 90, 255]
    return workloads.random_csc(120_000, len(lens), lens, seed=51)


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(rank % ndev)
    dev = torch.device("cuda", rank % ndev)
    backend = "nccl" if ndev >= world else "gloo"
    if backend == "nccl":
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                                device_id=dev)
    else:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2310_15419_b200 import distributed as skd
        from paper_2310_15419_b200 import sketch as sk
        sk.load_library()
        A = _matrix()
        As = workloads.shard_csc(A, world, rank)
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        res = {"backend": np.array(backend)}
        for dist_name, seed in CASES:
            # (1) row shard -> libsketch partial -> all_reduce (every rank gets Â)
            out, plan = skd.sketch_row_sharded(t(As.colptr), t(As.rowidx), t(As.vals), D, As.m, As.row_offset,
                                               seed, dist_name, mode="all_reduce")
            torch.cuda.synchronize()
            res[f"{dist_name}_allreduce"] = out.T.cpu().numpy()
            # (2) the same partial, reduce to rank 0 only
            out2, _ = skd.sketch_row_sharded(t(As.colptr), t(As.rowidx), t(As.vals), D, As.m, As.row_offset,
                                             seed, dist_name, mode="reduce", plan=plan)
            torch.cuda.synchronize()
            if rank == 0:
                res[f"{dist_name}_reduce"] = out2.T.cpu().numpy()
            plan.close()
            # (3) overlapped: 4 column groups, each group's all_reduce on a side stream into out[c0:c1]
            out3 = skd.sketch_row_sharded_overlapped(As.colptr, t(As.colptr), t(As.rowidx), t(As.vals), D, As.m,
                                                     As.row_offset, seed, dist_name, groups=4)
            torch.cuda.synchronize()
            res[f"{dist_name}_overlapped"] = out3.T.cpu().numpy()
            # (4) column shards (no reduction) + all_gather of the blocks
            b = skd.balanced_col_shards(A.colptr, world)
            Ac = workloads.col_slice(A, b[rank], b[rank + 1])
            blk, pc = skd.sketch_col_sharded(t(Ac.colptr), t(Ac.rowidx), t(Ac.vals), D, A.m, seed, dist_name)
            full = skd.gather_col_blocks(blk, b)
            torch.cuda.synchronize()
            res[f"{dist_name}_colshard"] = full.T.cpu().numpy()
            pc.close()
            # (5) end to end from pinned host buffers (the bench's e2e leg at N > 1)
            h_out = torch.empty((A.n, D), dtype=torch.float64).pin_memory()
            skd.sketch_row_sharded_e2e(torch.from_numpy(As.colptr).pin_memory(), torch.from_numpy(As.rowidx).pin_memory(),
                                       torch.from_numpy(As.vals).pin_memory(), D, As.m, As.row_offset, seed,
                                       dist_name, h_out)
            res[f"{dist_name}_e2e"] = h_out.numpy().T.copy()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    with tempfile.TemporaryDirectory() as td:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, WORLD, port, td)) for r in range(WORLD)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=600)
        codes = [p.exitcode for p in procs]
        assert codes == [0] * WORLD, f"rank exit codes {codes}"
        yield [dict(np.load(os.path.join(td, f"rank{r}.npz"))) for r in range(WORLD)]


def _check(got, ref, bound):
    err = np.abs(got - ref)
    assert np.all(got[bound == 0] == 0)
    worst = float((err / np.maximum(bound, 1e-300)).max())
    assert np.all(err <= 1e-12 * bound), worst


@pytest.mark.parametrize("dist_name,seed", CASES, ids=[c[0] for c in CASES])
def test_multirank_collectives_match_oracle(results, dist_name, seed):
    A = _matrix()
    ref, B = oracle.sketch(seed, dist_name, D, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    for rank, r in enumerate(results):
        for kind in ("allreduce", "overlapped", "colshard", "e2e"):
            _check(r[f"{dist_name}_{kind}"], ref, B)
        # every rank ends with the same Â (one collective result)
        assert np.array_equal(r[f"{dist_name}_allreduce"], results[0][f"{dist_name}_allreduce"])
    _check(results[0][f"{dist_name}_reduce"], ref, B)
    # column shards compute each column exactly as the unsharded plan does
    assert np.array_equal(results[0][f"{dist_name}_colshard"], results[1][f"{dist_name}_colshard"])


def test_backend_is_recorded(results):
    import torch
    want = "nccl" if torch.cuda.device_count() >= WORLD else "gloo"
    assert all(str(r["backend"]) == want for r in results)
