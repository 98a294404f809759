"""CPU oracle for the gamblet hot path.  TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 implementation in
`paper_1503_03467_b200`.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it; the
product path never does (it fails loudly when its CUDA library is missing).

It restates, in numpy/scipy, the algorithm of the reference package
`gamblets` (arXiv 1503.03467, `/root/reference/pkg/src/gamblets`) in its
*tight mode* (SURVEY.md section 8(c)): every patch and dense solve is done by a
direct factorization instead of the reference's CG-to-1e-14, which SURVEY.md
measured to agree with the reference to 1e-16..1e-13 on R, A, B, psi and
7e-14..3e-13 on u.  Patch submatrices are gathered in O(patch) instead of the
reference's O(N) fancy indexing, so q <= 8 runs in seconds.

Pinning: `oracle/make_goldens.py` runs the reference itself (tight mode) and
writes `tests/golden/*.npz`; `tests/test_host_and_oracle.py` checks this module
against those fixtures (and against the reference's own pinned values:
goldens.json radii, chi lists, load checksums).

Each function cites the reference file:line it follows (paths relative to
`/root/reference/pkg/src/gamblets/`).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# gamblet_fast.py:65-116, gamblet_exact.py:45-48
DEFAULT_C_RHO = 0.5
TOL_FLOOR = 1e-14
TOL_CEIL = 0.4
TAIL_DROP_REL = 1e-12
ROW_DROP_REL = 1e-11
SYMMETRY_REPAIR_TOL = 1e-12
H = 0.5


class OracleNumericalError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# canonical CSR and the index hierarchy
# --------------------------------------------------------------------------

def canon(m):
    """Canonical CSR: summed duplicates, no explicit zeros, sorted indices
    (sparse_core.py:47-67)."""
    out = sp.csr_array(m).astype(float)
    out.sum_duplicates()
    out.eliminate_zeros()
    out.sort_indices()
    return out


def box_indices(side, flat, rho):
    """Chebyshev index box of half-width floor(rho) around `flat`, clipped,
    row-major ascending (hierarchy.py:187-209)."""
    s, t = divmod(int(flat), side)
    w = int(np.floor(rho))
    ss = np.arange(max(0, s - w), min(side - 1, s + w) + 1)
    tt = np.arange(max(0, t - w), min(side - 1, t + w) + 1)
    return (ss[:, None] * side + tt[None, :]).ravel()


def chi_indices(k, parent, rho):
    """3 subband indices per member of the parent ball (hierarchy.py:211-219)."""
    ball = box_indices(2 ** (k - 1), parent, rho)
    return (3 * ball[:, None] + np.arange(3)[None, :]).ravel()


_W_TEMPLATES = {
    "chain": np.array([[1, -1, 0, 0], [0, 1, -1, 0], [0, 0, 1, -1]], float),
}
_base = np.array([[1, -1, 0, 0], [1, 1, -2, 0], [1, 1, 1, -3]], float)
# integer rows times one reciprocal norm per row (hierarchy.py:35-42)
_W_TEMPLATES["orthonormal"] = _base * (1.0 / np.sqrt((_base ** 2).sum(axis=1)))[:, None]


def children(k, flat):
    """Level-(k+1) children of level-k aggregates, flat-ordered
    (hierarchy.py:109-117)."""
    side = 2 ** k
    s, t = np.divmod(np.asarray(flat), side)
    fs = 2 * side
    base = 2 * s * fs + 2 * t
    return np.stack([base, base + 1, base + fs, base + fs + 1], axis=-1)


def null_basis(k, variant="orthonormal"):
    """W^(k), shape (3*4^(k-1), 4^k) (hierarchy.py:161-183)."""
    tmpl = _W_TEMPLATES[variant]
    npar = 4 ** (k - 1)
    ch = children(k - 1, np.arange(npar))                      # (npar, 4)
    rows = (3 * np.arange(npar)[:, None, None]
            + np.arange(3)[None, :, None] + 0 * ch[:, None, :])
    cols = np.broadcast_to(ch[:, None, :], (npar, 3, 4))
    vals = np.broadcast_to(tmpl[None], (npar, 3, 4))
    return canon(sp.coo_array((vals.ravel(), (rows.ravel(), cols.ravel())),
                              shape=(3 * npar, 4 ** k)))


def pi_step(k):
    """0/1 aggregation pi^(k,k+1) (hierarchy.py:121-134)."""
    side_f = 2 ** (k + 1)
    cols = np.arange(4 ** (k + 1))
    s, t = np.divmod(cols, side_f)
    rows = (s // 2) * (side_f // 2) + t // 2
    return canon(sp.coo_array((np.ones(cols.size), (rows, cols)),
                              shape=(4 ** k, 4 ** (k + 1))))


def phi(k, q, M):
    """Phi^(k) = pi^(k,q) M (hierarchy.py:140-159)."""
    n = 2 ** q
    cols = np.arange(n * n)
    i, j = np.divmod(cols, n)
    step = 2 ** (q - k)
    rows = (i // step) * 2 ** k + j // step
    P = canon(sp.coo_array((np.ones(cols.size), (rows, cols)), shape=(4 ** k, n * n)))
    return canon(P @ M)


def make_radii(epsilon, q, c_rho=None, uniform_rho=None):
    """rho_k, clipped into [1, 2^k] (gamblet_fast.py:240-265)."""
    c = DEFAULT_C_RHO if c_rho is None else float(c_rho)
    out = []
    for k in range(1, q + 1):
        if uniform_rho is not None:
            rho = int(uniform_rho)
        else:
            rho = int(np.ceil(c * (k * (np.log(2.0) + 1.0) + np.log(1.0 / epsilon))))
        out.append(int(min(max(rho, 1), 2 ** k)))
    return tuple(out)


def clamp_tol(tol):
    return float(min(TOL_CEIL, max(TOL_FLOOR, tol)))


def subband_tol(epsilon, q):
    """gamblet_fast.py:235-237."""
    return clamp_tol(epsilon / (2.0 * q))


# --------------------------------------------------------------------------
# scaling, symmetrization and the drop rules
# --------------------------------------------------------------------------

def diag_scale(mat):
    """s = diag^-1/2 and S mat S with (x*s_i)*s_j (gamblet_fast.py:123-139)."""
    mat = canon(mat)
    d = mat.diagonal()
    if d.min() <= 0.0:
        raise OracleNumericalError(f"nonpositive diagonal {d.min():.3e}")
    s = 1.0 / np.sqrt(d)
    row = np.repeat(np.arange(mat.shape[0]), np.diff(mat.indptr))
    out = mat.copy()
    out.data = mat.data * s[row] * s[mat.indices]
    return s, out


def symmetrize(X):
    """(X + X^T)/2 with the rounding-level repair guard
    (gamblet_exact.py:95-103); works on sparse or dense."""
    if sp.issparse(X):
        X = canon(X)
        scale = float(np.abs(X.data).max()) if X.nnz else 0.0
        if scale == 0.0:
            return X, 0.0
        diff = canon(X - X.T)
        repair = (float(np.abs(diff.data).max()) if diff.nnz else 0.0) / scale
    else:
        scale = float(np.abs(X).max())
        if scale == 0.0:
            return X, 0.0
        repair = float(np.abs(X - X.T).max()) / scale
    if repair >= SYMMETRY_REPAIR_TOL:
        raise OracleNumericalError(f"symmetry repair {repair:.3e}")
    out = (X + X.T) * 0.5
    return (canon(out) if sp.issparse(out) else out), repair


def drop_dead_tails(mat):
    """|x| < 1e-12 sqrt(d_i d_j) removed off the diagonal
    (gamblet_fast.py:154-169)."""
    d = mat.diagonal()
    if d.min() <= 0.0:
        return mat
    coo = mat.tocoo()
    keep = np.abs(coo.data) >= TAIL_DROP_REL * np.sqrt(d[coo.row] * d[coo.col])
    keep |= coo.row == coo.col
    return canon(sp.coo_array((coo.data[keep], (coo.row[keep], coo.col[keep])),
                              shape=mat.shape))


def drop_row_tails(mat):
    """|x| < 1e-11 * rowmax removed (gamblet_fast.py:172-190)."""
    mat = canon(mat)
    if mat.nnz == 0:
        return mat
    mag = np.abs(mat.data)
    row = np.repeat(np.arange(mat.shape[0]), np.diff(mat.indptr))
    rmax = np.zeros(mat.shape[0])
    np.maximum.at(rmax, row, mag)
    keep = mag >= ROW_DROP_REL * rmax[row]
    return canon(sp.csr_array((mat.data[keep], (row[keep], mat.indices[keep])),
                              shape=mat.shape))


# --------------------------------------------------------------------------
# CG and spectral extremes
# --------------------------------------------------------------------------

def cg(A, b, rel_tol, max_iter=None, x0=None):
    """Plain CG with the reference's stopping rule and iteration count
    (sparse_core.py:126-165).  Returns (x, iterations, rel_residual)."""
    b = np.asarray(b, float)
    n = b.shape[0]
    if max_iter is None:
        max_iter = max(200, 2 * n)
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return np.zeros(n), 0, 0.0
    x = np.zeros(n) if x0 is None else np.array(x0, float)
    r = b - A @ x if x0 is not None else b.copy()
    rnorm = float(np.linalg.norm(r))
    if rnorm <= rel_tol * bnorm:
        return x, 0, rnorm / bnorm
    p = r.copy()
    rs = rnorm * rnorm
    for it in range(1, max_iter + 1):
        Ap = A @ p
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise OracleNumericalError("CG breakdown")
        alpha = rs / pAp
        x += alpha * p
        r -= alpha * Ap
        rs_new = float(r @ r)
        rnorm = np.sqrt(rs_new)
        if rnorm <= rel_tol * bnorm:
            return x, it, rnorm / bnorm
        p = r + (rs_new / rs) * p
        rs = rs_new
    raise OracleNumericalError("CG did not converge")


def start_vectors(n, seed=24337):
    """The two start vectors eig_extremes draws (sparse_core.py:242-262)."""
    rng = np.random.default_rng(seed)
    x1 = rng.standard_normal(n)
    x2 = rng.standard_normal(n)
    return x1, x2


def eig_extremes(A, tol=0.1, max_iter=500, seed=24337):
    """Power iteration for lambda_max, inverse iteration (inner CG) for
    lambda_min (sparse_core.py:232-278)."""
    n = A.shape[0]
    x1, x2 = start_vectors(n, seed)
    x = x1 / np.linalg.norm(x1)
    lam_max = 0.0
    for _ in range(max_iter):
        y = A @ x
        lam_max = float(x @ y)
        ynorm = float(np.linalg.norm(y))
        if ynorm == 0.0:
            lam_max = 0.0
            break
        res = float(np.linalg.norm(y - lam_max * x))
        x = y / ynorm
        if res <= 0.5 * tol * abs(lam_max):
            break
    inner = max(1e-12, 1e-3 * tol)
    x = x2 / np.linalg.norm(x2)
    lam_min, lam_prev, y_prev = lam_max, np.inf, None
    for _ in range(max_iter):
        y, _, _ = cg(A, x, inner, x0=y_prev)
        ynorm = float(np.linalg.norm(y))
        x = y / ynorm
        y_prev = y / ynorm
        lam_min = float(x @ (A @ x))
        if abs(lam_min - lam_prev) <= 0.5 * tol * abs(lam_min):
            break
        lam_prev = lam_min
    return lam_min, lam_max


# --------------------------------------------------------------------------
# patch gathers and direct batched solves
# --------------------------------------------------------------------------

def principal_dense(mat, idx, pos):
    """Dense mat[idx, idx] in O(patch) (replaces sparse_core.py:99-113).
    `pos` is a scratch array of -1 of size mat.shape[0]."""
    m = idx.size
    pos[idx] = np.arange(m)
    starts = mat.indptr[idx]
    lens = mat.indptr[idx + 1] - starts
    tot = int(lens.sum())
    rows = np.repeat(np.arange(m), lens)
    offs = np.arange(tot) - np.repeat(np.cumsum(lens) - lens, lens) + np.repeat(starts, lens)
    loc = pos[mat.indices[offs]]
    keep = loc >= 0
    out = np.zeros((m, m))
    out[rows[keep], loc[keep]] = mat.data[offs[keep]]
    pos[idx] = -1
    return out


def _batched_solve(mats, rhss):
    """Group equal-size systems and solve them directly."""
    out = [None] * len(mats)
    by_size = {}
    for j, a in enumerate(mats):
        by_size.setdefault(a.shape[0], []).append(j)
    for n, js in by_size.items():
        for c0 in range(0, len(js), 512):
            chunk = js[c0:c0 + 512]
            A = np.stack([mats[j] for j in chunk])
            b = np.stack([rhss[j] for j in chunk])[..., None]
            x = np.linalg.solve(A, b)[..., 0]
            for jj, j in enumerate(chunk):
                out[j] = x[jj]
    return out


# --------------------------------------------------------------------------
# localized transform (Algorithm 2)
# --------------------------------------------------------------------------

def mass_inverse(M, q, rho):
    """psi^(q): per fine node, (S M S)[i^rho, i^rho] z = s_i e_i, row
    s[i^rho] * z (gamblet_fast.py:464-498)."""
    N = 4 ** q
    side = 2 ** q
    s, Ms = diag_scale(M)
    pos = np.full(N, -1)
    mats, rhss, idxs = [], [], []
    for i in range(N):
        idx = box_indices(side, i, rho)
        mats.append(principal_dense(Ms, idx, pos))
        rhs = np.zeros(idx.size)
        rhs[int(np.searchsorted(idx, i))] = s[i]
        rhss.append(rhs)
        idxs.append(idx)
    zs = _batched_solve(mats, rhss)
    rows = np.concatenate([np.full(ix.size, i) for i, ix in enumerate(idxs)])
    cols = np.concatenate(idxs)
    vals = np.concatenate([s[ix] * z for ix, z in zip(idxs, zs)])
    return canon(sp.coo_array((vals, (rows, cols)), shape=(N, N)))


def level_q_stiffness(psi, A):
    """A^(q) = drop(sym(psi A psi^T)) (gamblet_fast.py:658-665)."""
    X = canon(psi @ A)
    Aq, repair = symmetrize(canon(X @ canon(psi.T)))
    return drop_dead_tails(canon(Aq)), repair


def level_step(level, k, rho_coarse, variant="orthonormal", with_psi=True,
               spectral=True):
    """One localized step k -> k-1 with direct correction solves
    (gamblet_fast.py:501-632).  `level` is a dict with psi/stiffness; it is
    updated with W, B, s_b, D, R, lambdas; returns the level-(k-1) dict."""
    W = null_basis(k, variant)
    A_k = canon(level["stiffness"])
    X = canon(W @ A_k)
    B, repair_b = symmetrize(canon(X @ canon(W.T)))
    B = drop_dead_tails(canon(B))
    s_b, Bs = diag_scale(B)
    if spectral:
        lam_min, lam_max = eig_extremes(Bs, tol=0.1)
    else:
        lam_min = lam_max = None
    P = pi_step(k - 1)
    G = canon(X @ canon(P.T * 0.25))
    Gc = sp.csc_array(-G)
    n_coarse = 4 ** (k - 1)
    pos = np.full(B.shape[0], -1)
    mats, rhss, chis, cols_i = [], [], [], []
    for i in range(n_coarse):
        chi = chi_indices(k, i, rho_coarse)
        col = np.zeros(B.shape[0])
        a, b = Gc.indptr[i], Gc.indptr[i + 1]
        col[Gc.indices[a:b]] = Gc.data[a:b]
        rhs = s_b[chi] * col[chi]
        if float(np.linalg.norm(rhs)) == 0.0:
            continue
        mats.append(principal_dense(Bs, chi, pos))
        rhss.append(rhs)
        chis.append(chi)
        cols_i.append(i)
    zs = _batched_solve(mats, rhss)
    if chis:
        rows = np.concatenate(chis)
        cols = np.concatenate([np.full(c.size, i) for c, i in zip(chis, cols_i)])
        vals = np.concatenate([s_b[c] * z for c, z in zip(chis, zs)])
    else:
        rows = cols = np.zeros(0, int)
        vals = np.zeros(0)
    D = canon(sp.coo_array((vals, (rows, cols)), shape=(B.shape[0], n_coarse)))
    Dt = drop_row_tails(canon(D.T))
    D = canon(Dt.T)
    R = canon(P * 0.25 + Dt @ W)
    PAPt = canon(canon(P @ A_k) @ canon(P.T))
    GtD = canon(canon(G.T) @ D)
    DtBD = canon(Dt @ canon(B @ D))
    raw = 0.0625 * PAPt + GtD + canon(GtD.T) + DtBD
    A_next, repair_a = symmetrize(canon(raw))
    A_next = drop_dead_tails(canon(A_next))
    psi_next = None
    if with_psi and level.get("psi") is not None:
        psi = level["psi"]
        psi_next = drop_row_tails(canon(0.25 * canon(P @ psi) + Dt @ canon(W @ psi)))
    level.update(null_w=W, subband=B, subband_scale=s_b, correction=D,
                 restriction=R, lambda_min=lam_min, lambda_max=lam_max,
                 repair=max(level.get("repair", 0.0), repair_b))
    return {"k": k - 1, "psi": psi_next, "stiffness": A_next, "repair": repair_a}


def fast_transform(M, A, q, radii, variant="orthonormal", with_psi=True,
                   spectral=True):
    """Load-independent phase (gamblet_fast.py:635-674)."""
    psi = mass_inverse(canon(M), q, radii[q - 1])
    Aq, repair = level_q_stiffness(psi, canon(A))
    levels = {q: {"k": q, "psi": psi, "stiffness": Aq, "repair": repair}}
    for k in range(q, 1, -1):
        levels[k - 1] = level_step(levels[k], k, radii[k - 2], variant,
                                   with_psi=with_psi, spectral=spectral)
    return levels


def solve_with_transform(levels, g_nodal, q, tol):
    """Load-dependent phase with the nodal moment shortcut
    (gamblet_fast.py:677-775).  Needs psi on every level."""
    g = np.asarray(g_nodal, float).copy()
    coeffs, incs, iters = {}, {}, {}
    for k in range(q, 1, -1):
        L = levels[k]
        W, B, R, s = L["null_w"], L["subband"], L["restriction"], L["subband_scale"]

        class _Op:
            shape = B.shape

            def __matmul__(self, x, B=B, s=s):
                return s * (B @ (s * x))

        z, it, _ = cg(_Op(), s * (W @ g), tol)
        w = s * z
        iters[k] = it
        incs[k] = L["psi"].T @ (W.T @ w)
        coeffs[k] = w
        g = R @ g
    A1 = levels[1]["stiffness"]
    s1 = 1.0 / np.sqrt(A1.diagonal())

    class _Op1:
        shape = A1.shape

        def __matmul__(self, x):
            return s1 * (A1 @ (s1 * x))

    z, it, _ = cg(_Op1(), s1 * g, tol)
    iters[1] = it
    U1 = s1 * z
    incs[1] = levels[1]["psi"].T @ U1
    partials = {1: incs[1]}
    for k in range(2, q + 1):
        partials[k] = partials[k - 1] + incs[k]
    return {"u": partials[q], "u1": U1, "coeffs": coeffs, "increments": incs,
            "partials": partials, "iterations": iters}


def fast_solve(M, A, g_nodal, q, epsilon, uniform_rho=None, c_rho=None,
               variant="orthonormal", spectral=True):
    radii = make_radii(epsilon, q, c_rho, uniform_rho)
    levels = fast_transform(M, A, q, radii, variant, spectral=spectral)
    sol = solve_with_transform(levels, g_nodal, q, subband_tol(epsilon, q))
    return sol, levels, radii


# --------------------------------------------------------------------------
# exact transform (Algorithm 1), dense, direct solves
# --------------------------------------------------------------------------

def _chol_solve(A, B):
    L = np.linalg.cholesky(A)
    import scipy.linalg as la
    return la.cho_solve((L, True), B)


def exact_solve(M, A, b, q, variant="orthonormal"):
    """gamblet_exact.py:115-263 with Cholesky in place of CG."""
    Md = M.toarray()
    Ad = A.toarray()
    psi = _chol_solve(Md, np.eye(Md.shape[0])).T
    a_q, rep = symmetrize(psi @ (A @ psi.T))
    levels = {q: {"k": q, "psi": psi, "stiffness": a_q, "load": psi @ b, "repair": rep}}
    del Ad
    coeffs, incs = {}, {}
    for k in range(q, 1, -1):
        L = levels[k]
        W = null_basis(k, variant)
        A_k = L["stiffness"]
        T = W @ A_k
        B, rep_b = symmetrize(W @ T.T)
        w = _chol_solve(B, W @ L["load"])
        incs[k] = L["psi"].T @ (W.T @ w)
        coeffs[k] = w
        P = pi_step(k - 1)
        rhs_d = -(W @ (P @ A_k).T) * 0.25
        D = _chol_solve(B, rhs_d)
        R = P.toarray() * 0.25 + (W.T @ D).T
        A_next, rep_a = symmetrize(R @ (R @ A_k.T).T)
        L.update(null_w=W, subband=B, correction=D, restriction=R,
                 repair=max(L["repair"], rep_b))
        levels[k - 1] = {"k": k - 1, "psi": R @ L["psi"], "stiffness": A_next,
                         "load": R @ L["load"], "repair": rep_a}
    L1 = levels[1]
    U1 = _chol_solve(L1["stiffness"], L1["load"])
    incs[1] = L1["psi"].T @ U1
    partials = {1: incs[1]}
    for k in range(2, q + 1):
        partials[k] = partials[k - 1] + incs[k]
    return {"u": partials[q], "u1": U1, "coeffs": coeffs, "increments": incs,
            "partials": partials}, levels


# --------------------------------------------------------------------------
# comparison helpers used by the parity tests
# --------------------------------------------------------------------------

def rel_fro(a, b):
    """||a - b||_F / ||b||_F for sparse or dense."""
    if sp.issparse(a) or sp.issparse(b):
        da = sp.csr_array(a) - sp.csr_array(b)
        num = float(np.sqrt((da.data ** 2).sum())) if da.nnz else 0.0
        den = float(np.sqrt((sp.csr_array(b).data ** 2).sum()))
    else:
        num = float(np.linalg.norm(np.asarray(a) - np.asarray(b)))
        den = float(np.linalg.norm(np.asarray(b)))
    return num / den if den > 0 else num


def rel_energy(A, u, u_ref):
    d = np.asarray(u) - np.asarray(u_ref)
    return float(np.sqrt(max(d @ (A @ d), 0.0) / (u_ref @ (A @ u_ref))))


def same_pattern(a, b):
    """Bit-exact structural equality of two canonical CSR matrices."""
    a = canon(a)
    b = canon(b)
    return (a.shape == b.shape and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices))
