"""Sketch-and-precondition least squares -- host tests.

LSQR and the SAP driver run on CPU torch here with the sketch supplied by the CPU oracle; the
GPU test (tests/test_gpu_parity.py::test_sap_solve_on_gpu) runs the same driver with the fused
kernel.  Pins: dense least-squares solutions (numpy lstsq / normal equations), the paper's
Error(x) metric, and the preconditioning effect (iteration counts)."""
import numpy as np
import pytest
import torch

import oracle
import workloads
from paper_2310_15419_b200 import sap


def _dense(A):
    M = np.zeros((A.m, A.n))
    for k in range(A.n):
        r, v = A.column(k)
        np.add.at(M[:, k], r, v)
    return M


def _torch_csc(A):
    return (torch.from_numpy(A.colptr), torch.from_numpy(A.rowidx.astype(np.int64)),
            torch.from_numpy(A.vals.astype(np.float64)))


def _oracle_sketch(A):
    def fn(d, seed, dist):
        ref, _ = oracle.sketch(seed, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=4, want_bound=False)
        return torch.from_numpy(np.ascontiguousarray(ref.T))
    return fn


def test_lsqr_matches_dense_least_squares():
    A, b = workloads.ls_problem(400, 30, 25, seed=3)
    M = _dense(A)
    op = sap.SparseOperator(*_torch_csc(A), A.m, A.n)
    res = sap.lsqr(op.matvec, op.rmatvec, torch.from_numpy(b), A.n, atol=1e-14, btol=1e-14)
    xref = np.linalg.lstsq(M, b, rcond=None)[0]
    assert res.istop in (1, 2)
    assert np.linalg.norm(res.x.numpy() - xref) <= 1e-9 * np.linalg.norm(xref)
    # residual norm estimate is the true residual norm
    assert abs(res.rnorm - np.linalg.norm(M @ res.x.numpy() - b)) <= 1e-8 * np.linalg.norm(b)


def test_error_metric_is_the_papers_formula():
    A, b = workloads.ls_problem(300, 20, 15, seed=4)
    M = _dense(A)
    x = np.random.default_rng(0).standard_normal(A.n)
    r = M @ x - b
    want = np.linalg.norm(M.T @ r) / (np.linalg.norm(M, "fro") * np.linalg.norm(r))
    op = sap.SparseOperator(*_torch_csc(A), A.m, A.n)
    got = sap.error_metric(op, torch.from_numpy(x), torch.from_numpy(b))
    assert abs(got - want) <= 1e-12 * want


@pytest.mark.parametrize("method", ["qr", "svd"])
@pytest.mark.parametrize("decades", [0.0, 3.0])
def test_sap_solves_to_the_papers_tolerance(method, decades):
    # d = 2n Gaussian sketch: the preconditioned operator is well conditioned whatever cond(A)
    # is (column scaling by 10^±3 here), so LSQR stops on its 1e-14 rule in a few dozen steps
    A, b = workloads.ls_problem(3000, 40, 60, seed=5, col_scale_decades=decades)
    M = _dense(A)
    res = sap.sap_solve(*_torch_csc(A), A.m, A.n, torch.from_numpy(b), d=2 * A.n, seed=11, dist="gaussian",
                        method=method, sketch_fn=_oracle_sketch(A))
    xref = np.linalg.lstsq(M, b, rcond=None)[0]
    assert res.istop in (1, 2) and res.rank == A.n
    assert res.iterations <= 80
    assert res.error <= 1e-13
    assert np.linalg.norm(res.x.numpy() - xref) <= 1e-8 * np.linalg.norm(xref)


def test_preconditioning_cuts_iterations():
    A, b = workloads.ls_problem(3000, 40, 60, seed=6, col_scale_decades=3.0)
    op = sap.SparseOperator(*_torch_csc(A), A.m, A.n)
    plain = sap.lsqr(op.matvec, op.rmatvec, torch.from_numpy(b), A.n, atol=1e-14, btol=1e-14, iter_lim=2000)
    res = sap.sap_solve(*_torch_csc(A), A.m, A.n, torch.from_numpy(b), d=2 * A.n, seed=11,
                        sketch_fn=_oracle_sketch(A))
    assert res.iterations * 3 < plain.itn


def test_svd_drops_tiny_singular_values():
    # a rank-deficient A (a repeated column): SAP-SVD keeps rank n - 1 and still reaches the bar
    A, b = workloads.ls_problem(2000, 25, 40, seed=8)
    lo, hi = A.colptr[3], A.colptr[4]
    A.rowidx[A.colptr[7]:A.colptr[8]] = A.rowidx[lo:hi][:A.colptr[8] - A.colptr[7]]
    A.vals[A.colptr[7]:A.colptr[8]] = A.vals[lo:hi][:A.colptr[8] - A.colptr[7]]
    res = sap.sap_solve(*_torch_csc(A), A.m, A.n, torch.from_numpy(b), d=2 * A.n, seed=2, method="svd",
                        sketch_fn=_oracle_sketch(A))
    assert res.rank == A.n - 1
    assert res.error <= 1e-12
