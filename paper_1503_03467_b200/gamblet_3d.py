"""BASELINE config 4: the localized gamblet transform + subband solve on the
3-D unit cube (128^3 cells at q = 7, Q1 trilinear elements, 27-point
stencil, rho = 2).

The reference package is 2-D only (grid_fem.py:1-14, hierarchy.py:1-14;
SPEC.md:140 lists 3-D as a non-goal).  This module runs its algorithm
(gamblet_fast.py:464-775) in d = 3, as restated by the test oracle
oracle/gamblets_oracle_nd.py:

* inputs: tensor-product Q1 elements (the reference's 2-D element matrices
  are the d = 2 instance of the Kronecker forms, grid_fem.py:46-57), Dirichlet
  elimination, b = M g (grid_fem.py:189-245);
* hierarchy: 8 children per aggregate (lexicographic offsets, axis 0
  slowest), pibar = pi / 8, W = 7 Helmert rows per parent (PAPER.md:906-916,
  Lemma 4.14; its n = 4 instance is hierarchy.py:35-42), chi = 7 ball + c;
* transform: psi^(q) by local mass-matrix solves, A^(q) = drop(sym(psi A
  psi^T)), per level B = drop(sym(W A W^T)), G = W A pibar^T, correction
  patches (S B S)[chi, chi] z = s (-G)[chi, i] solved by Cholesky, D^T row
  trim, R = pibar + D^T W, A^(k-1) = drop(sym(P A P^T/64 + G^T D + D^T G +
  D^T B D)) -- every step a kernel of csrc/gb_3d.cu;
* solve: w^(k) by CG on S B^(k) S to the subband tolerance, g <- R g, the
  coarse CG, and the increments psi^(k)T W^T w^(k).

Deliberate difference (documented in DESIGN.md): psi^(k) for k < q is not
materialized (its 3-D windows would need ~15 K values per fine DOF at
q = 7); the increments use psi^(k) = R^(k+1) psi^(k+1) through the
prolongation chain psi^(q)T R^(q)T ... R^(k+1)T, i.e. without the
reference's 1e-11 row-tail drops of psi^(k<q) (a 1e-11-relative effect,
far below the 1e-9 bar on u).  Level operators stay in HBM; `.stiffness`,
`.subband`, `.correction`, `.restriction`, `.psi` (level q) export to
canonical scipy CSR on access.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as nat
from . import device as dv
from .errors import InvalidArgumentError, NumericalError
from .gamblet_exact import MultiresSolution, SolveRecord
from .gamblet_fast import (_Krylov, _start_vectors, make_schedule, SYMMETRY_REPAIR_TOL,
                           MAX_ITER_CAP, LANCZOS_CAP, LANCZOS_TOL)
from .sparse_core import as_csr

__all__ = ["Grid3D", "build_grid_3d", "coefficient_example_3d", "coefficient_checkerboard_3d",
           "gaussian_load_3d", "assemble_mass_3d", "assemble_stiffness_3d",
           "assemble_load_3d", "w_template_3d", "fast_solve_3d", "Level3D", "FastResult3D",
           "box3_from_csr"]

D = 3
NCH = 8        # children per aggregate
NSUB = 7       # W rows per parent


# ---------------------------------------------------------------------------
# inputs (grid_fem.py:46-57, 92-245 in d = 3)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Grid3D:
    """n = 2^q interior nodes per axis, h = 1/(n+1); node (i, j, k) in
    {1..n}^3 flattened row-major (axis 0 slowest); cells in {0..n}^3."""
    q: int
    n: int
    h: float

    @property
    def num_nodes(self):
        return self.n ** 3

    @property
    def num_cells(self):
        return (self.n + 1) ** 3


def build_grid_3d(q):
    """Grid at depth q, 1 <= q <= 8 (grid_fem.py:92-99 with a 3-D range)."""
    if isinstance(q, bool) or not isinstance(q, (int, np.integer)):
        raise InvalidArgumentError(f"q must be an integer, got {q!r}")
    if not 1 <= q <= 8:
        raise InvalidArgumentError(f"q must be in [1, 8] in 3-D, got {q}")
    n = 1 << int(q)
    return Grid3D(q=int(q), n=n, h=1.0 / (n + 1))


def _kron(mats):
    out = np.array([[1]], dtype=np.int64)
    for m in mats:
        out = np.kron(out, m)
    return out


def element_matrices_3d():
    """(mass / h^3, stiffness / h) of the trilinear element, lexicographic
    corners: Kronecker products of the 1-D Q1 matrices h/6 [[2,1],[1,2]] and
    1/h [[1,-1],[-1,1]] formed in exact integers, one division each."""
    m1 = np.array([[2, 1], [1, 2]], dtype=np.int64)
    k1 = np.array([[1, -1], [-1, 1]], dtype=np.int64)
    mass = _kron([m1] * 3).astype(float) / 216.0
    stiff = sum(_kron([k1 if a == ax else m1 for a in range(3)]) for ax in range(3))
    return mass, stiff.astype(float) / 36.0


def _cell_corners(grid):
    n = grid.n
    m = n + 1
    ci = np.arange(m)
    cx, cy, cz = np.meshgrid(ci, ci, ci, indexing="ij")
    cells = np.stack([cx.ravel(), cy.ravel(), cz.ravel()], axis=1)
    offs = np.array(list(itertools.product((0, 1), repeat=3)), dtype=np.int64)
    idx = cells[:, None, :] + offs[None, :, :]
    interior = np.all((idx >= 1) & (idx <= n), axis=2)
    flat = ((idx[:, :, 0] - 1) * n + (idx[:, :, 1] - 1)) * n + (idx[:, :, 2] - 1)
    return np.where(interior, flat, -1)


def _assemble(grid, element, cell_scale):
    corners = _cell_corners(grid)
    nc = corners.shape[1]
    rows = np.repeat(corners, nc, axis=1).ravel()
    cols = np.tile(corners, (1, nc)).ravel()
    vals = (np.asarray(cell_scale, float)[:, None, None] * element[None, :, :]).ravel()
    keep = (rows >= 0) & (cols >= 0)
    N = grid.num_nodes
    return as_csr(sp.coo_array((vals[keep], (rows[keep], cols[keep])), shape=(N, N)))


def assemble_mass_3d(grid):
    mass, _ = element_matrices_3d()
    return _assemble(grid, mass, np.full(grid.num_cells, grid.h ** 3))


def assemble_stiffness_3d(grid, coef):
    coef = np.asarray(coef, dtype=float)
    if coef.shape != (grid.num_cells,):
        raise InvalidArgumentError(f"expected {grid.num_cells} cell values, got {coef.shape}")
    if not np.all(coef > 0.0):
        raise InvalidArgumentError("coefficient values must be strictly positive")
    _, stiff = element_matrices_3d()
    return _assemble(grid, stiff, coef * grid.h)


def coefficient_example_3d(grid, kmax=5):
    """BASELINE config 4: prod_{k=1..5} (1 + cos(2^k pi (x+y+z))/2)
    (1 + sin(2^k pi (z - 3x + y))/2) at the cell's lower corner index
    (c / (n+1)), the sampling convention of grid_fem.py:136-155."""
    m = grid.n + 1
    ci = np.arange(m)
    cx, cy, cz = np.meshgrid(ci, ci, ci, indexing="ij")
    s = (cx + cy + cz) / m
    t = (cz - 3.0 * cx + cy) / m
    vals = np.ones_like(s, dtype=float)
    for k in range(1, kmax + 1):
        w = (2.0 ** k) * np.pi
        vals *= (1.0 + 0.5 * np.cos(w * s)) * (1.0 + 0.5 * np.sin(w * t))
    return vals.ravel()


def coefficient_checkerboard_3d(grid, contrast, seed):
    """Log-uniform cell values on [1, contrast] (grid_fem.py:167-176)."""
    u = np.random.default_rng(int(seed)).random(grid.num_cells)
    return np.exp(u * np.log(float(contrast)))


def gaussian_load_3d(grid, seed):
    """Nodal g ~ N(0, 1) i.i.d. from default_rng(seed) (BASELINE config 4)."""
    return np.random.default_rng(int(seed)).standard_normal(grid.num_nodes)


def assemble_load_3d(grid, g_nodal, mass=None):
    M = mass if mass is not None else assemble_mass_3d(grid)
    g = np.asarray(g_nodal, dtype=float)
    if g.shape != (grid.num_nodes,):
        raise InvalidArgumentError(f"load shape {g.shape} does not match N={grid.num_nodes}")
    return M @ g


def w_template_3d():
    """The 7 x 8 null-basis template: the row-orthonormalized U^(8) of
    Lemma 4.14 without its all-ones row (row t = (1,..,1 [t], -t, 0..) /
    sqrt(t + t^2)); rows annihilate constants over the 8 children."""
    U = np.zeros((NSUB, NCH))
    for t in range(1, NCH):
        U[t - 1, :t] = 1.0
        U[t - 1, t] = -float(t)
    return np.ascontiguousarray(U * (1.0 / np.sqrt((U ** 2).sum(axis=1)))[:, None])


# ---------------------------------------------------------------------------
# device boxes and their CSR export
# ---------------------------------------------------------------------------

def slots3(w, nc):
    return (2 * w + 1) ** 3 * nc


def _offsets3(w):
    r = np.arange(-w, w + 1)
    dx, dy, dz = np.meshgrid(r, r, r, indexing="ij")
    return dx.ravel(), dy.ravel(), dz.ravel()


def _box3_csr(vals, L, nr, w, nc, kind="square"):
    """Canonical CSR of a 3-D box (host export).  kind 'square': columns
    (p + d, c'); 'child': R rows, columns = the 8 children of p + d on the
    2L grid; 'dt': the stored rows are D^T, the matrix returned is D."""
    v = dv.to_host(vals).reshape(L ** 3 * nr, -1)
    rows, slots = np.nonzero(v)
    data = v[rows, slots]
    p = rows // nr
    px, py, pz = p // (L * L), (p // L) % L, p % L
    dx, dy, dz = _offsets3(w)
    if kind == "child":
        j = slots % NCH
        t = slots // NCH
        qx, qy, qz = px + dx[t], py + dy[t], pz + dz[t]
        Lk = 2 * L
        cols = ((2 * qx + (j >> 2)) * Lk + (2 * qy + ((j >> 1) & 1))) * Lk + 2 * qz + (j & 1)
        shape = (L ** 3, Lk ** 3)
    else:
        c = slots % nc
        t = slots // nc
        qx, qy, qz = px + dx[t], py + dy[t], pz + dz[t]
        cols = ((qx * L + qy) * L + qz) * nc + c
        shape = (L ** 3 * nr, L ** 3 * nc)
    m = sp.csr_array((data, (rows, cols)), shape=shape)
    if kind == "dt":
        m = sp.csr_array(m.T)
    return as_csr(m)


def _psi3_csr(vals, L, rho, wd):
    v = dv.to_host(vals).reshape(L ** 3, wd, wd, wd)
    rows, ex, ey, ez = np.nonzero(v)
    data = v[rows, ex, ey, ez]
    px, py, pz = rows // (L * L), (rows // L) % L, rows % L
    ox = np.clip(px - rho, 0, L - wd)
    oy = np.clip(py - rho, 0, L - wd)
    oz = np.clip(pz - rho, 0, L - wd)
    cols = ((ox + ex) * L + oy + ey) * L + oz + ez
    return as_csr(sp.csr_array((data, (rows, cols)), shape=(L ** 3, L ** 3)))


def _check(status, what):
    st = dv.to_host(status)
    code, det = int(st[0]), int(st[1])
    if code == 0:
        return
    if code == 1:
        raise NumericalError(f"{what}: nonpositive diagonal entry (row {det})")
    if code == 2:
        raise NumericalError(f"{what}: patch {det} is not positive definite")
    if code == 3:
        raise InvalidArgumentError(f"{what}: entry outside the 27-point stencil (row {det})")
    raise NumericalError(f"{what}: device status {code} (detail {det})")


class Level3D:
    """One level of the 3-D transform (LocalGambletLevel's fields); the
    operators stay in HBM and export to canonical scipy CSR on access."""

    def __init__(self, k, q):
        self.k, self.q = k, q
        self.L = 1 << k
        self._A = self._B = self._Dt = self._R = self._psi = None
        self.wA = self.wB = self.rho = None
        self.subband_scale_dev = None
        self.lambda_min_subband = self.lambda_max_subband = None
        self.symmetry_repair = 0.0
        self._cache = {}

    def _csr(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    @property
    def stiffness(self):
        return None if self._A is None else self._csr(
            "A", lambda: _box3_csr(self._A, self.L, 1, self.wA, 1))

    @property
    def subband(self):
        return None if self._B is None else self._csr(
            "B", lambda: _box3_csr(self._B, self.L // 2, NSUB, self.wB, NSUB))

    @property
    def correction(self):
        return None if self._Dt is None else self._csr(
            "D", lambda: _box3_csr(self._Dt, self.L // 2, 1, self.rho, NSUB, kind="dt"))

    @property
    def restriction(self):
        return None if self._R is None else self._csr(
            "R", lambda: _box3_csr(self._R, self.L // 2, 1, self.rho, NCH, kind="child"))

    @property
    def psi(self):
        return None if self._psi is None else self._csr(
            "psi", lambda: _psi3_csr(self._psi[0], self.L, self._psi[1], self._psi[2]))

    @property
    def subband_scale(self):
        return None if self.subband_scale_dev is None else dv.to_host(self.subband_scale_dev)


@dataclass
class FastResult3D:
    solution: MultiresSolution
    levels: dict
    radii: tuple
    iterations: dict = field(default_factory=dict)
    operators: dict = field(default_factory=dict)  # k -> S B^(k) S Krylov operator


# ---------------------------------------------------------------------------
# Krylov on the 3-D box operator S B S (sparse_core.py:126-165, 232-278)
# ---------------------------------------------------------------------------

class _Op3:
    def __init__(self, box, L, nr, w, s):
        self.box, self.L, self.nr, self.w, self.s = box, L, nr, w, s
        self.n = L ** 3 * nr

    def apply(self, x, y):
        nat.call("gb3_apply", self.L, self.nr, self.w, dv.ptr(self.box), dv.ptr(self.s),
                 dv.ptr(x), dv.ptr(y), dv.stream())

    def cg(self, b, rel_tol, x0=None, max_iter=None):
        """Plain CG from x0 (or 0), stop at ||r|| <= tol ||b||: (x, its, conv, brk)."""
        n = self.n
        if max_iter is None:
            max_iter = max(200, 2 * n)
        max_iter = min(max_iter, MAX_ITER_CAP)
        kr = _Krylov(n)
        st = dv.stream()
        x, r, p, Ap = (dv.zeros(n) for _ in range(4))
        nat.call("gb_state_reset", dv.ptr(kr.state), max_iter, st)
        Ax0 = None
        if x0 is not None:
            Ax0 = dv.empty(n)
            self.apply(x0, Ax0)
        nat.call("gb_cg_init", n, dv.ptr(b), dv.ptr(x0), dv.ptr(Ax0), dv.ptr(x), dv.ptr(r),
                 dv.ptr(p), float(rel_tol), int(max_iter), dv.ptr(kr.state), dv.ptr(kr.part),
                 st)
        nat.call("gb3_cg_solve", self.L, self.nr, self.w, dv.ptr(self.box), dv.ptr(self.s),
                 dv.ptr(x), dv.ptr(r), dv.ptr(p), dv.ptr(Ap), dv.ptr(kr.state),
                 dv.ptr(kr.part), kr.host.data_ptr(), 128, st)
        h = kr.host_view()
        return x, int(h["it"]), bool(h["converged"]), int(h["breakdown"])

    def eig_extremes(self, tol=0.1, max_iter=500, seed=24337, method="lanczos"):
        """sparse_core.py:232-278: power iteration (lambda_max) and, for
        lambda_min, the inverse iteration -- evaluated from the Lanczos
        moments of its start vector (method "lanczos", default: the iteration
        with exact inner solves) or run with warm-started inner CG to
        max(1e-12, 1e-3 tol) ("cg", the reference verbatim); start vectors
        from default_rng(seed)."""
        n = self.n
        st = dv.stream()
        x1, x2 = _start_vectors(n, seed)
        kr = _Krylov(n)
        x = x1.clone()
        y = dv.zeros(n)
        nat.call("gb_dot2", n, dv.ptr(x), dv.ptr(x), None, dv.ptr(kr.dots), dv.ptr(kr.state),
                 dv.ptr(kr.part), st)
        nat.call("gb_scale_by_norm", n, dv.ptr(x), dv.ptr(kr.dots), 0, dv.ptr(x), None, st)
        nat.call("gb_state_reset", dv.ptr(kr.state), max_iter, st)
        nat.call("gb3_pow_solve", self.L, self.nr, self.w, dv.ptr(self.box), dv.ptr(self.s),
                 dv.ptr(x), dv.ptr(y), float(tol), dv.ptr(kr.state), dv.ptr(kr.part),
                 kr.host.data_ptr(), 128, st)
        h = kr.host_view()
        lam_max = float(h["lam"])
        if method == "lanczos":
            # the inverse-iteration sequence from the Lanczos moments of its
            # unit start vector (csrc/gb_lanczos.h; the 2-D engine's default)
            x = x2.clone()
            nat.call("gb_dot2", n, dv.ptr(x), dv.ptr(x), None, dv.ptr(kr.dots), dv.ptr(kr.state),
                     dv.ptr(kr.part), st)
            nat.call("gb_scale_by_norm", n, dv.ptr(x), dv.ptr(kr.dots), 0, dv.ptr(x), None, st)
            cap = int(min(n, LANCZOS_CAP))
            ab = dv.empty(2 * cap)
            hab = torch.empty(2 * cap, dtype=torch.float64, pin_memory=True)
            lam = nat.ctypes.c_double(0.0)
            outer = nat.ctypes.c_int(0)
            its = nat.ctypes.c_int(0)
            vp, wv = dv.empty(n), dv.empty(n)
            nat.call("gb3_lanczos_min", self.L, self.nr, self.w, dv.ptr(self.box),
                     dv.ptr(self.s), dv.ptr(x), dv.ptr(vp), dv.ptr(wv), dv.ptr(kr.state),
                     dv.ptr(kr.part), kr.host.data_ptr(), dv.ptr(ab), hab.data_ptr(), cap,
                     float(tol), int(max_iter), float(LANCZOS_TOL), nat.ctypes.byref(lam),
                     nat.ctypes.byref(outer), nat.ctypes.byref(its), st)
            self.spectral_passes = int(h["it"]) + int(its.value)
            return float(lam.value), lam_max
        inner = max(1e-12, 1e-3 * tol)
        x = x2.clone()
        nat.call("gb_dot2", n, dv.ptr(x), dv.ptr(x), None, dv.ptr(kr.dots), dv.ptr(kr.state),
                 dv.ptr(kr.part), st)
        nat.call("gb_scale_by_norm", n, dv.ptr(x), dv.ptr(kr.dots), 0, dv.ptr(x), None, st)
        lam_min, lam_prev, y_prev = lam_max, np.inf, None
        dots = dv.empty(4)
        for _ in range(max_iter):
            yv, its, conv, brk = self.cg(x, inner, x0=y_prev)
            if brk:
                raise NumericalError(f"CG breakdown at iteration {brk}: p^T A p <= 0 "
                                     "(matrix is not SPD)")
            nat.call("gb_dot2", n, dv.ptr(yv), dv.ptr(yv), None, dv.ptr(dots),
                     dv.ptr(kr.state), dv.ptr(kr.part), st)
            xn, yp = dv.empty(n), dv.empty(n)
            nat.call("gb_scale_by_norm", n, dv.ptr(yv), dv.ptr(dots), 0, dv.ptr(xn),
                     dv.ptr(yp), st)
            Ax = dv.empty(n)
            self.apply(xn, Ax)
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


# ---------------------------------------------------------------------------
# transform (gamblet_fast.py:464-674 in d = 3)
# ---------------------------------------------------------------------------

def _sym_drop(L, nr, w, raw, what):
    out = dv.empty(raw.numel())
    dmin = dv.empty(1)
    stats = dv.zeros(2)
    nat.call("gb3_box_sym_drop", L, nr, w, dv.ptr(raw), dv.ptr(out), dv.ptr(dmin),
             dv.ptr(stats), dv.stream())
    sx = dv.to_host(stats)
    rep = 0.0 if sx[0] == 0.0 else float(sx[1] / sx[0])
    if rep >= SYMMETRY_REPAIR_TOL:
        raise NumericalError(f"{what} lost symmetry beyond rounding: relative repair {rep:.3e}")
    return out, rep


def box3_from_csr(mat, L, w=1):
    """Upload a canonical 27-point CSR on the L^3 grid into the 3-D box
    layout (a device tensor, reusable as fast_solve_3d input)."""
    return _csr3_to_box(mat, L, w)


def _csr3_to_box(mat, L, w=1):
    if isinstance(mat, torch.Tensor):  # already a device box
        if mat.numel() != L ** 3 * slots3(w, 1):
            raise InvalidArgumentError("device box input has the wrong size")
        return mat
    mat = as_csr(mat)
    box = dv.empty(L ** 3 * slots3(w, 1))
    st = dv.zeros(2, torch.int64)
    ip = dv.to_dev(mat.indptr.astype(np.int32))
    ix = dv.to_dev(mat.indices.astype(np.int32))
    vv = dv.to_dev(mat.data)
    nat.call("gb3_csr_to_box", L, w, dv.ptr(ip), dv.ptr(ix), dv.ptr(vv), dv.ptr(box),
             dv.ptr(st), dv.stream())
    _check(st, "input")
    return box


def _level_q(M, A, q, rho):
    """psi^(q) and A^(q) = drop(sym(psi A psi^T)) (gamblet_fast.py:464-498,
    650-665)."""
    L = 1 << q
    N = L ** 3
    s = dv.stream()
    Mb = _csr3_to_box(M, L)
    sM = dv.empty(N)
    st = dv.zeros(2, torch.int64)
    nat.call("gb3_box_scale", N, 1, 1, dv.ptr(Mb), dv.ptr(sM), dv.ptr(st), s)
    _check(st, "mass scaling")
    rho = int(min(rho, L - 1))
    wd = min(2 * rho + 1, L)
    psi = dv.empty(N * wd ** 3)
    with dv.phase("3d_mass_patches"):
        nat.call("gb3_mass_patches", L, dv.ptr(Mb), dv.ptr(sM), rho, wd, dv.ptr(psi),
                 dv.ptr(st), s)
    _check(st, "mass patches")
    del Mb
    Ab = _csr3_to_box(A, L)
    wX = min(rho + 1, L - 1)
    wR = min(2 * rho + 1, L - 1)
    X = dv.empty(N * slots3(wX, 1))
    raw = dv.empty(N * slots3(wR, 1))
    with dv.phase("3d_psi_A_psiT"):
        nat.call("gb3_psi_galerkin", L, rho, wd, dv.ptr(psi), dv.ptr(Ab), wX, dv.ptr(X), wR,
                 dv.ptr(raw), s)
    del X, Ab
    Aq, rep = _sym_drop(L, 1, wR, raw, "A^(q),loc")
    return (psi, rho, wd), Aq, wR, rep


def _level_step(lv, nxt, rho, W, ctas):
    """One step k -> k-1 (gamblet_fast.py:501-632): B, G, P A P^T, lambda
    estimates, correction patches, R, A^(k-1)."""
    k = lv.k
    Lk, Lp = 1 << k, 1 << (k - 1)
    P, J = Lp ** 3, NSUB * Lp ** 3
    s = dv.stream()
    wA = lv.wA
    wB = min((wA + 1) // 2, Lp - 1)
    rho = int(min(rho, Lp - 1))
    w8 = W.ctypes.data
    Braw = dv.empty(J * slots3(wB, NSUB))
    G = dv.empty(J * slots3(wB, 1))
    PAPt = dv.empty(P * slots3(wB, 1))
    with dv.phase("3d_level_blocks"):
        nat.call("gb3_level_blocks", Lk, wA, dv.ptr(lv._A), w8, wB, dv.ptr(Braw), dv.ptr(G),
                 dv.ptr(PAPt), s)
        B, rep_b = _sym_drop(Lp, NSUB, wB, Braw, f"B^({k}),loc")
    del Braw
    sB = dv.empty(J)
    st = dv.zeros(2, torch.int64)
    nat.call("gb3_box_scale", J, NSUB, wB, dv.ptr(B), dv.ptr(sB), dv.ptr(st), s)
    _check(st, f"B^({k}) scaling")
    lv._B, lv.wB, lv.subband_scale_dev = B, wB, sB
    lv.symmetry_repair = max(lv.symmetry_repair, rep_b)
    op = _Op3(B, Lp, NSUB, wB, sB)
    with dv.phase("3d_spectral"):
        lv.lambda_min_subband, lv.lambda_max_subband = op.eig_extremes(tol=0.1)
    # correction patches -> D^T (row-tail trim fused)
    R3 = (2 * rho + 1) ** 3
    Dt = dv.empty(P * R3 * NSUB)
    nb = nat.query("gb3_correction_workspace", Lp, rho, ctas)
    ws = dv.empty(nb // 8)
    with dv.phase("3d_correction_patches"):
        nat.call("gb3_correction_patches", Lp, wB, dv.ptr(B), dv.ptr(sB), dv.ptr(G), rho,
                 dv.ptr(Dt), dv.ptr(st), dv.ptr(ws), ctas, s)
    _check(st, f"correction patches, level {k}")
    del ws
    Rv = dv.empty(P * R3 * NCH)
    nat.call("gb3_restriction", Lp, rho, dv.ptr(Dt), w8, dv.ptr(Rv), s)
    lv._Dt, lv._R, lv.rho = Dt, Rv, rho
    # split triple product
    wBD = min(wB + rho, Lp - 1)
    wGD = min(wB + rho, Lp - 1)
    wA2 = min(2 * rho + wB, Lp - 1)
    BD = dv.empty(J * slots3(wBD, 1))
    GtD = dv.empty(P * slots3(wGD, 1))
    raw = dv.empty(P * slots3(wA2, 1))
    with dv.phase("3d_triple_product"):
        nat.call("gb3_triple", Lp, wB, dv.ptr(B), dv.ptr(G), dv.ptr(PAPt), rho, dv.ptr(Dt),
                 wBD, dv.ptr(BD), wGD, dv.ptr(GtD), wA2, dv.ptr(raw), s)
        del BD, GtD, G, PAPt
        An, rep_a = _sym_drop(Lp, 1, wA2, raw, f"A^({k - 1}),loc")
    nxt._A, nxt.wA = An, wA2
    nxt.symmetry_repair = rep_a
    return op


def _correction_ctas(Lp, rho):
    """CTAs of the correction-patch launch: 2 per SM (103 KB of shared
    memory each), bounded so their dense workspaces stay below ~8 GB."""
    ld = nat.query("gb3_correction_workspace", Lp, rho, 1)
    return int(max(1, min(148 * 2, (8 << 30) // max(ld, 1), Lp ** 3)))


def fast_transform_3d(M, A, q, radii):
    """Levels q..1 (dict k -> Level3D) and the Krylov operators of k >= 2."""
    for X in (M, A):
        ok = (X.numel() == 8 ** q * 27) if isinstance(X, torch.Tensor) else \
            (X.shape == (8 ** q, 8 ** q))
        if not ok:
            raise InvalidArgumentError(f"M, A must be {8 ** q} x {8 ** q} for q={q} in 3-D")
    W = w_template_3d()
    levels = {q: Level3D(q, q)}
    psi, Aq, wR, rep = _level_q(M, A, q, radii[q - 1])
    levels[q]._psi, levels[q]._A, levels[q].wA = psi, Aq, wR
    levels[q].symmetry_repair = rep
    ops = {}
    for k in range(q, 1, -1):
        nxt = Level3D(k - 1, q)
        rho = radii[k - 2]
        ops[k] = _level_step(levels[k], nxt, rho, W,
                             _correction_ctas(1 << (k - 1), min(rho, (1 << (k - 1)) - 1)))
        levels[k - 1] = nxt
    return levels, ops


# ---------------------------------------------------------------------------
# solve (gamblet_fast.py:677-775)
# ---------------------------------------------------------------------------

def _vmul(a, b):
    out = dv.empty(a.numel())
    nat.call("gb_vmul", a.numel(), dv.ptr(a), dv.ptr(b), dv.ptr(out), dv.stream())
    return out


def solve_with_transform_3d(levels, ops, g_nodal, q, tol):
    W = w_template_3d()
    w8 = W.ctypes.data
    s = dv.stream()
    g = dv.to_dev(np.asarray(g_nodal, dtype=float)) if not isinstance(g_nodal, torch.Tensor) \
        else g_nodal
    coeffs, vts, records, iters = {}, {}, [], {}
    for k in range(q, 1, -1):
        lv = levels[k]
        op = ops[k]
        Lp = 1 << (k - 1)
        rhs = dv.empty(op.n)
        nat.call("gb3_apply_w", Lp, w8, dv.ptr(g), dv.ptr(lv.subband_scale_dev), dv.ptr(rhs), s)
        with dv.phase("3d_subband_cg"):
            z, its, conv, brk = op.cg(rhs, tol)
        if brk:
            raise NumericalError(f"CG breakdown at iteration {brk}: p^T A p <= 0")
        if not conv:
            raise NumericalError(f"subband solve at level {k} did not converge")
        wk = _vmul(z, lv.subband_scale_dev)
        coeffs[k] = wk
        iters[k] = its
        records.append(SolveRecord(k, "subband", op.n, 1, tol, np.array([its]), np.array([0.0])))
        vt = dv.empty(8 * Lp ** 3)
        nat.call("gb3_apply_wt", Lp, w8, dv.ptr(wk), dv.ptr(vt), s)
        vts[k] = vt
        gn = dv.empty(Lp ** 3)
        nat.call("gb3_apply_r", Lp, lv.rho, dv.ptr(lv._R), dv.ptr(g), dv.ptr(gn), s)
        g = gn
    # coarse: CG on S A^(1) S (8 x 8)
    A1 = levels[1]
    s1 = dv.empty(8)
    st = dv.zeros(2, torch.int64)
    nat.call("gb3_box_scale", 8, 1, A1.wA, dv.ptr(A1._A), dv.ptr(s1), dv.ptr(st), s)
    _check(st, "A^(1) scaling")
    op1 = _Op3(A1._A, 2, 1, A1.wA, s1)
    z, its, conv, brk = op1.cg(_vmul(g, s1), tol)
    if brk or not conv:
        raise NumericalError("coarse solve failed")
    U1 = _vmul(z, s1)
    iters[1] = its
    records.append(SolveRecord(1, "coarse", 8, 1, tol, np.array([its]), np.array([0.0])))

    # increments psi^(k)T v_k = psi^(q)T R^(q)T ... R^(k+1)T v_k
    psi, rho_q, wd = levels[q]._psi
    N = 8 ** q

    def lift(vec, k):
        for j in range(k + 1, q + 1):
            lj = levels[j]
            Lp = 1 << (j - 1)
            out = dv.empty(8 * Lp ** 3)
            nat.call("gb3_apply_rt", Lp, lj.rho, dv.ptr(lj._R), dv.ptr(vec), dv.ptr(out), s)
            vec = out
        u = dv.empty(N)
        nat.call("gb3_psi_t_apply", 1 << q, rho_q, wd, dv.ptr(psi), dv.ptr(vec), dv.ptr(u), s)
        return u

    incs = {1: lift(U1, 1)}
    for k in range(2, q + 1):
        incs[k] = lift(vts[k], k)
    partials = {1: incs[1]}
    for k in range(2, q + 1):
        partials[k] = dv.empty(N)
        nat.call("gb_vadd", N, dv.ptr(partials[k - 1]), dv.ptr(incs[k]), dv.ptr(partials[k]), s)
    host = lambda d: {k: dv.to_host(v) for k, v in d.items()}  # noqa: E731
    sol = MultiresSolution(u=dv.to_host(partials[q]), u1_coarse=dv.to_host(U1),
                           subband_coeffs=host(coeffs), increments=host(incs),
                           partials=host(partials), records=records)
    return sol, iters


def fast_solve_3d(M, A, g_nodal, q, epsilon, uniform_rho=None, c_rho=None):
    """Localized transform plus solve in 3-D (gamblet_fast.py:815-837 in
    d = 3, the nodal moment shortcut g^(q) = g): returns FastResult3D."""
    sched = make_schedule(epsilon, q, c_rho=c_rho, uniform_rho=uniform_rho)
    levels, ops = fast_transform_3d(M, A, q, sched.radii)
    sol, iters = solve_with_transform_3d(levels, ops, g_nodal, q, sched.subband_tol())
    return FastResult3D(solution=sol, levels=levels, radii=tuple(sched.radii), iterations=iters,
                        operators=ops)
