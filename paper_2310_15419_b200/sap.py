"""Sketch-and-precondition least squares (§5.3).

Solves min_x ||A x - b||_2 for a tall sparse A (m x n, CSC) the way the paper's SAP-QR / SAP-SVD
does: sketch Â = S A with the fused kernel (d = 2n by default), factor the small
d x n sketch, and run LSQR (Paige & Saunders, ACM TOMS 8(1), 1982) on the right-preconditioned
operator A P until its internal error metric falls below `atol` (1e-14 in the paper,
PAPER.md:800-804):
  * SAP-QR:  Â = Q R,            P = R^{-1};
  * SAP-SVD: Â = U Σ V^T,        P = V_k Σ_k^{-1}, dropping σ_i < σ_max / 1e12.
The solution is x = P y.  The reported quality metric is the paper's
  Error(x) = ||A^T (A x - b)||_2 / (||A||_F ||A x - b||_2).

Everything except the sketch is library work on the GPU (cuSOLVER QR / SVD, cuSPARSE SpMV through
torch.sparse, triangular solves); the sketch is `sketch.Plan.apply`.  `sketch_fn` replaces the
sketch for host-only tests (they pass the CPU oracle's Â); the product path never falls back.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np


@dataclass
class LsqrResult:
    x: "object"              # torch tensor (n,)
    istop: int               # 1: ||r|| small (consistent), 2: ||Ā^T r|| / (||Ā|| ||r||) <= atol, 7: iteration limit
    itn: int
    rnorm: float             # estimate of ||b - Ā y||
    arnorm: float            # estimate of ||Ā^T (b - Ā y)||
    anorm: float             # Frobenius-norm estimate of Ā
    acond: float             # condition-number estimate of Ā


def lsqr(matvec, rmatvec, b, n: int, *, atol: float = 1e-14, btol: float = 1e-14, iter_lim: int | None = None):
    """LSQR for min ||Ā y - b|| with Ā given by matvec (y -> Ā y) and rmatvec (u -> Ā^T u).

    Golub-Kahan bidiagonalisation with the QR update of Paige & Saunders (1982), their stopping
    rules 1 and 2 (no damping, no conlim): stop when ||r|| <= btol ||b|| + atol ||Ā|| ||y|| or
    ||Ā^T r|| <= atol ||Ā|| ||r||.  Works on any torch device/dtype the operators use."""
    import torch
    if iter_lim is None:
        iter_lim = 4 * n + 100
    x = torch.zeros(n, dtype=b.dtype, device=b.device)
    u = b.clone()
    beta = float(torch.linalg.vector_norm(u))
    bnorm = beta
    if beta == 0.0:
        return LsqrResult(x, 0, 0, 0.0, 0.0, 0.0, 0.0)
    u /= beta
    v = rmatvec(u)
    alpha = float(torch.linalg.vector_norm(v))
    if alpha == 0.0:
        return LsqrResult(x, 2, 0, beta, 0.0, 0.0, 0.0)
    v /= alpha
    w = v.clone()
    phibar, rhobar = beta, alpha
    anorm2 = 0.0
    ddnorm = 0.0
    xnorm = 0.0
    rnorm, arnorm = beta, alpha * beta
    z, cs2, sn2, xxnorm = 0.0, -1.0, 0.0, 0.0
    istop, itn = 7, 0
    while itn < iter_lim:
        itn += 1
        # bidiagonalisation: beta u = Ā v - alpha u ; alpha v = Ā^T u - beta v
        u = matvec(v) - alpha * u
        beta = float(torch.linalg.vector_norm(u))
        if beta > 0.0:
            u /= beta
            anorm2 += alpha * alpha + beta * beta
            v = rmatvec(u) - beta * v
            alpha = float(torch.linalg.vector_norm(v))
            if alpha > 0.0:
                v /= alpha
        # plane rotation eliminating beta
        rho = math.hypot(rhobar, beta)
        cs, sn = rhobar / rho, beta / rho
        theta = sn * alpha
        rhobar = -cs * alpha
        phi = cs * phibar
        phibar = sn * phibar
        # update x and w
        t1, t2 = phi / rho, -theta / rho
        dk = w / rho
        x = x + t1 * w
        w = v + t2 * w
        ddnorm += float(torch.linalg.vector_norm(dk)) ** 2
        # ||x|| estimate (Paige & Saunders §5.1)
        delta = sn2 * rho
        gambar = -cs2 * rho
        rhs = phi - delta * z
        zbar = rhs / gambar
        xnorm = math.sqrt(xxnorm + zbar * zbar)
        gamma = math.hypot(gambar, theta)
        cs2, sn2 = gambar / gamma, theta / gamma
        z = rhs / gamma
        xxnorm += z * z
        # norms and stopping rules
        anorm = math.sqrt(anorm2)
        acond = anorm * math.sqrt(ddnorm)
        rnorm = phibar
        arnorm = alpha * abs(sn * phi)
        test1 = rnorm / bnorm
        test2 = arnorm / (anorm * rnorm) if anorm * rnorm > 0 else 0.0
        rtol = btol + atol * anorm * xnorm / bnorm
        if test1 <= rtol:
            istop = 1
            break
        if test2 <= atol:
            istop = 2
            break
    return LsqrResult(x, istop, itn, rnorm, arnorm, math.sqrt(anorm2), anorm * math.sqrt(ddnorm))


@dataclass
class SapResult:
    x: "object"
    istop: int
    iterations: int
    error: float                       # Error(x) of PAPER.md:805-808
    rank: int                          # numerical rank kept by the preconditioner
    times: dict = field(default_factory=dict)


class SparseOperator:
    """A (m x n) from CSC arrays as two torch CSR matrices: A^T (n x m; CSR of A^T = CSC of A)
    and A (m x n), for cuSPARSE SpMV on the GPU (or torch's CPU kernels)."""

    def __init__(self, colptr, rowidx, vals, m: int, n: int):
        import torch
        self.m, self.n = m, n
        self.At = torch.sparse_csr_tensor(colptr.to(torch.int64), rowidx.to(torch.int64), vals, size=(n, m))
        self.A = self.At.t().to_sparse_csr()
        self.fro = float(torch.linalg.vector_norm(vals))

    def matvec(self, v):
        return (self.A @ v.unsqueeze(1)).squeeze(1)

    def rmatvec(self, u):
        return (self.At @ u.unsqueeze(1)).squeeze(1)


def error_metric(op: SparseOperator, x, b) -> float:
    """Error(x) = ||A^T (A x - b)|| / (||A||_F ||A x - b||)."""
    import torch
    r = op.matvec(x) - b
    rn = float(torch.linalg.vector_norm(r))
    if rn == 0.0:
        return 0.0
    return float(torch.linalg.vector_norm(op.rmatvec(r))) / (op.fro * rn)


def sap_solve(colptr, rowidx, vals, m: int, n: int, b, *, d: int | None = None, seed: int = 0,
              dist: str = "gaussian", method: str = "qr", atol: float = 1e-14, iter_lim: int | None = None,
              sketch_fn=None) -> SapResult:
    """Sketch-and-precondition LSQR for min ||A x - b|| (A given as CSC torch tensors on one
    device).  sketch_fn(d, seed, dist) -> Â as a torch (n, d) tensor (column-major d x n) replaces
    the fused kernel (host-only tests)."""
    import torch
    if d is None:
        d = 2 * n
    dev = vals.device
    t0 = time.perf_counter()
    if sketch_fn is None:
        from . import sketch as sk
        dtype = "f64" if vals.dtype == torch.float64 else "f32"
        plan = sk.Plan(colptr, rowidx, d, m, dtype)
        Ahat_t = plan.apply(vals, seed, dist)
        plan.close()
    else:
        Ahat_t = sketch_fn(d, seed, dist)
    Ahat = Ahat_t.T.to(torch.float64)                        # d x n
    if dev.type == "cuda":
        torch.cuda.synchronize()
    t1 = time.perf_counter()
    if method == "qr":
        R = torch.linalg.qr(Ahat, mode="r")[1]
        rank = n

        def P(y):
            return torch.linalg.solve_triangular(R, y.unsqueeze(1), upper=True).squeeze(1)

        def PT(z):
            return torch.linalg.solve_triangular(R.T, z.unsqueeze(1), upper=False).squeeze(1)
    elif method == "svd":
        _, s, Vh = torch.linalg.svd(Ahat, full_matrices=False)
        keep = s > s[0] / 1e12
        rank = int(keep.sum())
        V = Vh[keep].T / s[keep]                            # n x k: V_k Σ_k^{-1}

        def P(y):
            return V @ y

        def PT(z):
            return V.T @ z
    else:
        raise ValueError(method)
    if dev.type == "cuda":
        torch.cuda.synchronize()
    t2 = time.perf_counter()
    op = SparseOperator(colptr, rowidx, vals.to(torch.float64), m, n)
    bb = b.to(torch.float64)
    res = lsqr(lambda y: op.matvec(P(y)), lambda u: PT(op.rmatvec(u)), bb, rank, atol=atol, btol=atol,
               iter_lim=iter_lim)
    x = P(res.x)
    if dev.type == "cuda":
        torch.cuda.synchronize()
    t3 = time.perf_counter()
    return SapResult(x, res.istop, res.itn, error_metric(op, x, bb), rank,
                     {"sketch_s": t1 - t0, "factor_s": t2 - t1, "lsqr_s": t3 - t2})
