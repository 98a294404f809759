"""GPU Krylov solvers on general CSR operators (sparse_core.py:126-278).

`cg_solve`, `cg_solve_block` and `eig_extremes` keep the reference's
signatures, return types and error behaviour; the iterations run on the
device (csrc/gb_krylov.cu: warp-per-row CSR SpMV with fused reductions, the
CG / power-iteration state in device memory, the loop driven from C with the
GIL released).  Inputs: a scipy sparse matrix or a dense 2-D array (converted
to canonical CSR), or anything exposing `shape` and `@` is rejected -- the
device needs the matrix itself.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as nat
from . import device as dv
from .errors import InvalidArgumentError, NumericalError
from .sparse_core import CgReport, as_csr

__all__ = ["cg_solve", "cg_solve_block", "eig_extremes"]


def _require(cond, msg):
    if not cond:
        raise InvalidArgumentError(msg)


class _DevCsr:
    def __init__(self, A):
        if not sp.issparse(A):
            arr = np.asarray(A, dtype=float)
            _require(arr.ndim == 2, f"expected a 2-d matrix, got shape {arr.shape}")
            A = arr
        A = as_csr(A)
        self.shape = A.shape
        self.n = A.shape[0]
        self.indptr = dv.to_dev(A.indptr.astype(np.int32))
        self.indices = dv.to_dev(A.indices.astype(np.int32))
        self.data = dv.to_dev(A.data.astype(np.float64))

    def apply(self, x, y):
        nat.call("gb_csr_apply", self.n, dv.ptr(self.indptr), dv.ptr(self.indices),
                 dv.ptr(self.data), dv.ptr(x), dv.ptr(y), dv.stream())


def _state():
    from .gamblet_fast import _Krylov
    return _Krylov(0)


def _cg_dev(op, b, rel_tol, max_iter, x0=None, kr=None):
    from .gamblet_fast import MAX_ITER_CAP
    n = op.n
    kr = kr or _state()
    st = dv.stream()
    x, r, p, Ap = (dv.empty(n) for _ in range(4))
    nat.call("gb_state_reset", dv.ptr(kr.state), int(max_iter), st)
    Ax0 = None
    if x0 is not None:
        Ax0 = dv.empty(n)
        op.apply(x0, Ax0)
    nat.call("gb_cg_init", n, dv.ptr(b), dv.ptr(x0), dv.ptr(Ax0), dv.ptr(x), dv.ptr(r),
             dv.ptr(p), float(rel_tol), int(min(max_iter, MAX_ITER_CAP)), dv.ptr(kr.state),
             dv.ptr(kr.part), st)
    nat.call("gb_csr_cg_solve", n, dv.ptr(op.indptr), dv.ptr(op.indices), dv.ptr(op.data),
             dv.ptr(x), dv.ptr(r), dv.ptr(p), dv.ptr(Ap), dv.ptr(kr.state), dv.ptr(kr.part),
             kr.host.data_ptr(), 128, st)
    return x, kr.host_view()


def cg_solve(A, b, rel_tol=1e-10, max_iter=None, x0=None):
    """Conjugate gradients (sparse_core.py:126-165): stops when
    ||b - A x|| <= rel_tol ||b||; max_iter is reported, not fatal;
    p^T A p <= 0 raises NumericalError."""
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    _require(tuple(A.shape) == (n, n), f"shape mismatch: {A.shape} vs rhs {b.shape}")
    if max_iter is None:
        max_iter = max(200, 2 * n)
    op = _DevCsr(A)
    bd = dv.to_dev(b)
    x0d = None if x0 is None else dv.to_dev(np.asarray(x0, dtype=float))
    x, h = _cg_dev(op, bd, rel_tol, max_iter, x0d)
    if h["breakdown"]:
        raise NumericalError(f"CG breakdown at iteration {int(h['breakdown'])}: p^T A p <= 0 "
                             "(matrix is not SPD)")
    bn = float(h["bnorm"])
    rel = float(h["rnorm"] / bn) if bn > 0 else 0.0
    return dv.to_host(x), CgReport(int(h["it"]), rel, bool(h["converged"]))


def cg_solve_block(A, B, rel_tol=1e-10, max_iter=None):
    """Column-wise CG on the block B (sparse_core.py:168-229): per-column
    iteration counts equal a sequential column-by-column solve, which is how
    the device runs it.  Returns (X, iterations, rel_residuals, converged)."""
    B = np.asarray(B, dtype=float)
    _require(B.ndim == 2, f"rhs block must be 2-d, got shape {B.shape}")
    n, m = B.shape
    _require(tuple(A.shape) == (n, n), f"shape mismatch: {A.shape} vs rhs {B.shape}")
    if max_iter is None:
        max_iter = max(200, 2 * n)
    op = _DevCsr(A)
    kr = _state()
    X = np.zeros((n, m))
    iters = np.zeros(m, dtype=int)
    rel = np.zeros(m)
    conv = np.ones(m, dtype=bool)
    for j in range(m):
        if not np.any(B[:, j]):
            continue
        x, h = _cg_dev(op, dv.to_dev(np.ascontiguousarray(B[:, j])), rel_tol, max_iter, kr=kr)
        if h["breakdown"]:
            raise NumericalError(f"CG breakdown at iteration {int(h['breakdown'])} in column "
                                 "block (matrix is not SPD)")
        X[:, j] = dv.to_host(x)
        iters[j] = int(h["it"])
        rel[j] = float(h["rnorm"] / h["bnorm"])
        conv[j] = bool(h["converged"])
    return X, iters, rel, conv


def eig_extremes(A, tol=1e-2, max_iter=500, seed=24337):
    """(lambda_min, lambda_max) by power iteration and inverse iteration with
    inner CG, start vectors from default_rng(seed) (sparse_core.py:232-278)."""
    _require(A.shape[0] == A.shape[1], f"A must be square, got {A.shape}")
    op = _DevCsr(A)
    n = op.n
    rng = np.random.default_rng(seed)
    x1 = rng.standard_normal(n)
    x2 = rng.standard_normal(n)
    kr = _state()
    st = dv.stream()
    x = dv.to_dev(x1 / np.linalg.norm(x1))
    y = dv.empty(n)
    nat.call("gb_state_reset", dv.ptr(kr.state), int(max_iter), st)
    nat.call("gb_csr_pow_solve", n, dv.ptr(op.indptr), dv.ptr(op.indices), dv.ptr(op.data),
             dv.ptr(x), dv.ptr(y), float(tol), dv.ptr(kr.state), dv.ptr(kr.part),
             kr.host.data_ptr(), 128, st)
    h = kr.host_view()
    lam_max = float(h["lam"])
    inner = max(1e-12, 1e-3 * tol)
    x = dv.to_dev(x2 / np.linalg.norm(x2))
    lam_min, lam_prev, y_prev = lam_max, np.inf, None
    ykr = _state()
    dots = dv.empty(4)
    for _ in range(max_iter):
        yv, hh = _cg_dev(op, x, inner, max(200, 2 * n), x0=y_prev, kr=ykr)
        if hh["breakdown"]:
            raise NumericalError(f"CG breakdown at iteration {int(hh['breakdown'])}: "
                                 "p^T A p <= 0 (matrix is not SPD)")
        nat.call("gb_dot2", n, dv.ptr(yv), dv.ptr(yv), None, dv.ptr(dots), dv.ptr(kr.state),
                 dv.ptr(kr.part), st)
        xn, yp = dv.empty(n), dv.empty(n)
        nat.call("gb_scale_by_norm", n, dv.ptr(yv), dv.ptr(dots), 0, dv.ptr(xn), dv.ptr(yp), st)
        Ax = dv.empty(n)
        op.apply(xn, Ax)
        nat.call("gb_dot2", n, dv.ptr(xn), dv.ptr(Ax), None, dv.ptr(dots[2:]),
                 dv.ptr(kr.state), dv.ptr(kr.part), st)
        d = kr.read_dots(dots)
        if d[0] == 0.0:
            raise NumericalError("inverse iteration broke down: A^{-1} x = 0")
        lam_min = float(d[2])
        x, y_prev = xn, yp
        if abs(lam_min - lam_prev) <= 0.5 * tol * abs(lam_min):
            break
        lam_prev = lam_min
    return lam_min, lam_max
