"""Exact (global-gamblet) transform on the GPU -- Algorithm 1, config 0.

Mirrors gamblets/gamblet_exact.py:115-263.  Every intermediate is dense
FP64 on the device (the reference holds them dense too); the reference's CG
solves (cg_solve / cg_solve_block to tol 1e-14 in tight mode) are replaced
by Cholesky factorizations (csrc/gb_dense.cu), which agree with tight mode to
~1e-13.

Per downward step k -> k-1 with W = W^(k), pibar = pi/4:
    B = W A W^T,  w = B^-1 W g,  increment = Psi^T W^T w,
    D = -B^-1 W A pibar^T,  R = pibar + D^T W,
    A' = R A R^T,  Psi' = R Psi,  g' = R g.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from . import device as dv
from .errors import InvalidArgumentError, NumericalError
from .grid_fem import LoadVector
from .hierarchy import w_template

__all__ = ["GambletLevel", "SolveRecord", "MultiresSolution", "exact_solve",
           "init_level_q", "level_step", "solve_coarsest", "HostDict"]

SYMMETRY_REPAIR_TOL = 1e-12
DEFAULT_TOL_MASS = 1e-10
DEFAULT_TOL_SUBBAND = 1e-10


@dataclass
class SolveRecord:
    """One solve (or column batch) with per-column iteration counts
    (gamblet_exact.py:51-65).  Direct solves record 1 iteration per column."""

    level: int
    kind: str
    size: int
    columns: int
    tol: float
    iterations: np.ndarray
    rel_residual: np.ndarray

    @property
    def max_iterations(self):
        return int(np.max(self.iterations)) if self.iterations.size else 0


class HostDict(dict):
    """dict whose device-tensor values are copied to numpy on first access."""

    def _host(self, key):
        v = dict.__getitem__(self, key)
        if isinstance(v, torch.Tensor):
            v = v.cpu().numpy()
            dict.__setitem__(self, key, v)
        return v

    def __getitem__(self, key):
        return self._host(key)

    def get(self, key, default=None):
        return self._host(key) if key in self else default

    def values(self):
        return [self._host(k) for k in self.keys()]

    def items(self):
        return [(k, self._host(k)) for k in self.keys()]

    def device(self, key):
        """The value without host conversion (torch tensor when on device)."""
        return dict.__getitem__(self, key)


@dataclass
class MultiresSolution:
    """Telescoping solution (gamblet_exact.py:83-92)."""

    u: np.ndarray
    u1_coarse: np.ndarray
    subband_coeffs: dict = field(default_factory=HostDict)
    increments: dict = field(default_factory=HostDict)
    partials: dict = field(default_factory=HostDict)
    records: list = field(default_factory=list)


class _Dense:
    """Row-major dense device matrix with lazy numpy view."""

    def __init__(self, t, rows, cols):
        self.t, self.rows, self.cols = t, rows, cols

    def host(self):
        return self.t.view(self.rows, self.cols).cpu().numpy()


class GambletLevel:
    """Level-k data of the exact sweep (gamblet_exact.py:68-80); dense fields
    are numpy arrays materialized from the device on first access."""

    _DENSE = ("psi", "stiffness", "subband", "correction", "restriction")

    def __init__(self, k, psi, stiffness, load, null_w=None, subband=None,
                 correction=None, restriction=None, symmetry_repair=0.0):
        self.k = k
        self._f = {}
        self.psi = psi
        self.stiffness = stiffness
        self.load = load
        self.null_w = null_w
        self.subband = subband
        self.correction = correction
        self.restriction = restriction
        self.symmetry_repair = symmetry_repair

    def __setattr__(self, name, value):
        if name in GambletLevel._DENSE or name == "load":
            self._f[name] = value
        else:
            object.__setattr__(self, name, value)

    def __getattr__(self, name):
        f = self.__dict__.get("_f", {})
        if name in f:
            v = f[name]
            if isinstance(v, _Dense):
                v = v.host()
                f[name] = v
            elif isinstance(v, torch.Tensor):
                v = v.cpu().numpy()
                f[name] = v
            return v
        raise AttributeError(name)

    def _dev(self, name):
        return self._f.get(name)


def _as_rhs(b, N):
    if isinstance(b, LoadVector):
        b = b.b
    b = np.asarray(b, dtype=float)
    if b.shape != (N,):
        raise InvalidArgumentError(f"rhs shape {b.shape} does not match N={N}")
    return b


class _Ops:
    """Thin wrappers over the dense C entry points on the current stream."""

    def __init__(self):
        self.s = dv.stream()
        self.status = dv.zeros(2, torch.int64)
        self.stats = []

    def mat(self, rows, cols):
        return dv.empty(rows * cols)

    def gemm(self, m, n, k, A, lda, ta, B, ldb, tb, alpha=1.0, beta=0.0, C=None, ldc=None):
        if C is None:
            C = self.mat(m, n)
            beta = 0.0
        nat.call("gb_dense_gemm", m, n, k, alpha, dv.ptr(A), lda, ta, dv.ptr(B), ldb, tb,
                 beta, dv.ptr(C), n if ldc is None else ldc, self.s)
        return C

    def chol(self, A, n):
        L = A.clone()
        nat.call("gb_dense_potrf", n, dv.ptr(L), n, dv.ptr(self.status), self.s)
        return L

    def solve(self, L, n, B, nrhs):
        X = B.clone()
        nat.call("gb_dense_potrs", n, nrhs, dv.ptr(L), n, dv.ptr(X), nrhs, self.s)
        return X

    def sym(self, X, n, what):
        out = self.mat(n, n)
        st = dv.zeros(2)
        nat.call("gb_dense_sym", n, dv.ptr(X), n, dv.ptr(out), dv.ptr(st), self.s)
        self.stats.append((what, st))
        return out, st

    def check(self):
        st = self.status.cpu().numpy()
        if st[0] != 0:
            raise NumericalError(f"dense Cholesky: matrix is not positive definite "
                                 f"(pivot {int(st[1])})")


def _repair(st):
    md, ma = st.cpu().numpy()
    return 0.0 if ma == 0.0 else float(md / ma)


def _check_repair(what, rep):
    if rep >= SYMMETRY_REPAIR_TOL:
        raise NumericalError(f"{what} lost symmetry beyond rounding: relative repair {rep:.3e}")


def _csr_dense(mat, ops):
    n0, n1 = mat.shape
    ip = dv.to_dev(np.asarray(mat.indptr, np.int32))
    ix = dv.to_dev(np.asarray(mat.indices, np.int32))
    da = dv.to_dev(np.asarray(mat.data, np.float64))
    out = ops.mat(n0, n1)
    nat.call("gb_csr_to_dense", n0, n1, dv.ptr(ip), dv.ptr(ix), dv.ptr(da), dv.ptr(out),
             ops.s)
    return out


def init_level_q(M, A, b, tree, tol_mass=DEFAULT_TOL_MASS, mode="mass_inverse",
                 records=None, block_columns=1024):
    """Finest level: Psi = M^-1 by Cholesky, A^(q) = Psi A Psi^T, g = Psi b
    (gamblet_exact.py:115-161); mode "nodal": Psi = I, A^(q) = A, g = b."""
    N = 4 ** tree.q
    if M.shape != (N, N) or A.shape != (N, N):
        raise InvalidArgumentError(f"matrix shapes {M.shape}/{A.shape} do not match q={tree.q}")
    b = _as_rhs(b, N)
    if mode not in ("mass_inverse", "nodal"):
        raise InvalidArgumentError(f"unknown level-q init mode {mode!r}")
    ops = _Ops()
    Ad = _csr_dense(A, ops)
    bd = dv.to_dev(b)
    if mode == "nodal":
        psi = ops.mat(N, N)
        nat.call("gb_eye", N, dv.ptr(psi), ops.s)
        a_q, st = ops.sym(Ad, N, "A^(q)")
        rep = _repair(st)
        _check_repair("A^(q)", rep)
        return GambletLevel(tree.q, _Dense(psi, N, N), _Dense(a_q, N, N), bd.clone(),
                            symmetry_repair=rep), ops
    Md = _csr_dense(M, ops)
    Lm = ops.chol(Md, N)
    eye = ops.mat(N, N)
    nat.call("gb_eye", N, dv.ptr(eye), ops.s)
    psi = ops.solve(Lm, N, eye, N)          # M^-1 (symmetric): rows are basis rows
    T = ops.gemm(N, N, N, Ad, N, 0, psi, N, 1)          # A psi^T
    raw = ops.gemm(N, N, N, psi, N, 0, T, N, 0)         # psi (A psi^T)
    a_q, st = ops.sym(raw, N, "A^(q)")
    g = ops.gemm(N, 1, N, psi, N, 0, bd, 1, 0)
    ops.check()
    rep = _repair(st)
    _check_repair("A^(q)", rep)
    if records is not None:
        records.append(SolveRecord(tree.q, "mass_inverse", N, N, tol_mass,
                                   np.ones(N, int), np.zeros(N)))
    return GambletLevel(tree.q, _Dense(psi, N, N), _Dense(a_q, N, N), g,
                        symmetry_repair=rep), ops


def level_step(level, tree, w_variant="orthonormal", tol_subband=DEFAULT_TOL_SUBBAND,
               records=None, ops=None):
    """One dense downward step k -> k-1 (gamblet_exact.py:164-211); returns
    (next_level, w_k, increment) with w_k / increment as device tensors."""
    k = level.k
    if k < 2:
        raise InvalidArgumentError(f"level_step needs k >= 2, got k={k}")
    ops = ops or _Ops()
    N = 4 ** tree.q
    Ik, Ic, J = 4 ** k, 4 ** (k - 1), 3 * 4 ** (k - 1)
    tmpl = w_template(w_variant)
    W = ops.mat(J, Ik)
    nat.call("gb_dense_build_w", 1 << k, tmpl.ctypes.data, dv.ptr(W), ops.s)
    A_k = level._dev("stiffness").t
    psi = level._dev("psi").t
    g = level._dev("load")
    T = ops.gemm(J, Ik, Ik, W, Ik, 0, A_k, Ik, 0)            # W A
    Braw = ops.gemm(J, J, Ik, W, Ik, 0, T, Ik, 1)            # W (W A)^T
    B, stb = ops.sym(Braw, J, f"B^({k})")
    LB = ops.chol(B, J)
    rhs_w = ops.gemm(J, 1, Ik, W, Ik, 0, g, 1, 0)
    w_k = ops.solve(LB, J, rhs_w, 1)
    v = ops.gemm(Ik, 1, J, W, Ik, 1, w_k, 1, 0)               # W^T w
    inc = ops.gemm(N, 1, Ik, psi, N, 1, v, 1, 0)              # Psi^T W^T w
    P = ops.mat(Ic, Ik)
    nat.call("gb_dense_build_p", 1 << k, dv.ptr(P), 1.0, ops.s)
    PA = ops.gemm(Ic, Ik, Ik, P, Ik, 0, A_k, Ik, 0)
    rhs_d = ops.gemm(J, Ic, Ik, W, Ik, 0, PA, Ik, 1, alpha=-0.25)   # -(W (P A)^T)/4
    D = ops.solve(LB, J, rhs_d, Ic)
    R = ops.mat(Ic, Ik)
    nat.call("gb_dense_build_p", 1 << k, dv.ptr(R), 0.25, ops.s)
    ops.gemm(Ic, Ik, J, D, Ic, 1, W, Ik, 0, alpha=1.0, beta=1.0, C=R)   # pibar + D^T W
    T2 = ops.gemm(Ik, Ic, Ik, A_k, Ik, 0, R, Ik, 1)          # A R^T
    raw = ops.gemm(Ic, Ic, Ik, R, Ik, 0, T2, Ic, 0)          # R (A R^T)
    A_next, sta = ops.sym(raw, Ic, f"A^({k - 1})")
    psi_next = ops.gemm(Ic, N, Ik, R, Ik, 0, psi, N, 0)
    g_next = ops.gemm(Ic, 1, Ik, R, Ik, 0, g, 1, 0)
    ops.check()
    rep_b, rep_a = _repair(stb), _repair(sta)
    _check_repair(f"B^({k})", rep_b)
    _check_repair(f"A^({k - 1})", rep_a)
    if records is not None:
        records.append(SolveRecord(k, "subband", J, 1, tol_subband, np.ones(1, int),
                                   np.zeros(1)))
        records.append(SolveRecord(k, "correction", J, Ic, tol_subband,
                                   np.ones(Ic, int), np.zeros(Ic)))
    level.null_w = tree.null_basis(k, w_variant)
    level.subband = _Dense(B, J, J)
    level.correction = _Dense(D, J, Ic)
    level.restriction = _Dense(R, Ic, Ik)
    level.symmetry_repair = max(level.symmetry_repair, rep_b)
    nxt = GambletLevel(k - 1, _Dense(psi_next, Ic, N), _Dense(A_next, Ic, Ic), g_next,
                       symmetry_repair=rep_a)
    return nxt, w_k, inc


def solve_coarsest(level, tol=DEFAULT_TOL_SUBBAND, records=None, ops=None):
    """A^(1) U = g^(1) (gamblet_exact.py:214-225); returns device (U, Psi^T U)."""
    if level.k != 1:
        raise InvalidArgumentError(f"expected level 1, got {level.k}")
    ops = ops or _Ops()
    N = level._dev("psi").cols
    L1 = ops.chol(level._dev("stiffness").t, 4)
    U = ops.solve(L1, 4, level._dev("load"), 1)
    u1 = ops.gemm(N, 1, 4, level._dev("psi").t, N, 1, U, 1, 0)
    ops.check()
    if records is not None:
        records.append(SolveRecord(1, "coarse", 4, 1, tol, np.ones(1, int), np.zeros(1)))
    return U, u1


def exact_solve(M, A, b, tree, w_variant="orthonormal", tol_mass=DEFAULT_TOL_MASS,
                tol_subband=DEFAULT_TOL_SUBBAND, level_q_init="mass_inverse"):
    """Full dense sweep q -> 1 plus reassembly (gamblet_exact.py:228-263)."""
    records = []
    levels = {}
    level, ops = init_level_q(M, A, b, tree, tol_mass=tol_mass, mode=level_q_init,
                              records=records)
    levels[tree.q] = level
    coeffs, incs = HostDict(), HostDict()
    for k in range(tree.q, 1, -1):
        nxt, w_k, inc = level_step(level, tree, w_variant=w_variant,
                                   tol_subband=tol_subband, records=records, ops=ops)
        coeffs[k] = w_k
        incs[k] = inc
        levels[k - 1] = nxt
        level = nxt
    U1, u1 = solve_coarsest(level, tol=tol_subband, records=records, ops=ops)
    incs[1] = u1
    partials = HostDict({1: u1})
    prev = u1
    for k in range(2, tree.q + 1):
        out = dv.empty(prev.numel())
        nat.call("gb_vadd", prev.numel(), dv.ptr(prev), dv.ptr(incs.device(k)),
                 dv.ptr(out), ops.s)
        partials[k] = out
        prev = out
    u = prev.cpu().numpy()
    sol = MultiresSolution(u=u, u1_coarse=U1.cpu().numpy(), subband_coeffs=coeffs,
                           increments=incs, partials=partials, records=records)
    return sol, levels
