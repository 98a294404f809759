"""Dimension-generic CPU oracle (d = 2, 3) for the localized gamblet path.
TEST INFRASTRUCTURE ONLY (same rules as oracle/gamblets_oracle.py: only
tests/, smoke() and bench.py's cpu_baseline leg may import it).

The reference package is 2-D only (grid_fem.py:1-14, hierarchy.py:1-14;
SPEC.md:140 lists 3-D as a non-goal), so BASELINE.json config 4 (3-D unit
cube, Q1 trilinear, 27-point stencil, Haar dyadic-cube measurements, rho=2)
has no reference implementation.  This module restates, for d dimensions:

* grid_fem.py:46-57,189-245 -- tensor-product Q1 elements (the 2-D element
  matrices of the reference are the d=2 instance of the Kronecker forms
  below, in the reference's corner order SW, SE, NE, NW), Dirichlet
  elimination, b = M g;
* hierarchy.py:84-219 -- 2^d children per aggregate (flat ascending),
  pi (0/1), pibar = pi / 2^d, W with 2^d - 1 rows per parent from the
  orthonormalized U^(2^d) of the paper's Lemma 4.14 / Construction 4.15
  (its n=4 instance is the reference's 'orthonormal'
  template, hierarchy.py:35-42), Chebyshev balls and
  chi = (2^d - 1) * ball + c;
* gamblet_fast.py:464-674 and the solve 677-775 -- identical to the 2-D
  oracle with 1/4 -> 1/2^d and 1/16 -> 1/4^d.

Pinning: the d=2 instance is checked against oracle/gamblets_oracle.py and
the reference goldens (tests/test_oracle_nd.py); the d=3 instance is "parity
unpinned" against any reference (there is none) -- it is the specification
the 3-D GPU path will be checked against.
"""

from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

from oracle import gamblets_oracle as O

# 1-D Q1 element matrices on [0, h]: mass h/6 [[2,1],[1,2]], stiffness
# 1/h [[1,-1],[-1,1]]; d-D elements are Kronecker products (lexicographic
# corner order, axis 0 slowest)
_M1 = np.array([[2, 1], [1, 2]], dtype=np.int64)
_K1 = np.array([[1, -1], [-1, 1]], dtype=np.int64)


def _kron_all(mats):
    out = np.array([[1]], dtype=np.int64)
    for m in mats:
        out = np.kron(out, m)
    return out


def element_matrices(d):
    """(mass / h^d, stiffness / h^(d-2)) of the Q1 element in lexicographic
    corner order, formed from exact integers and one division."""
    mass = _kron_all([_M1] * d).astype(float) / float(6 ** d)
    stiff = np.zeros((2 ** d, 2 ** d), dtype=np.int64)
    for ax in range(d):
        stiff += _kron_all([_K1 if a == ax else _M1 for a in range(d)])
    return mass, stiff.astype(float) / float(6 ** (d - 1))


def corner_offsets(d):
    """Lexicographic corner offsets {0,1}^d (axis 0 slowest)."""
    return np.array(list(itertools.product((0, 1), repeat=d)), dtype=np.int64)


class GridND:
    """n = 2^q interior nodes per axis, h = 1/(n+1), nodes (i_1..i_d) in
    {1..n}^d flattened row-major, cells in {0..n}^d (grid_fem.py:60-101)."""

    def __init__(self, q, d):
        self.q, self.d = int(q), int(d)
        self.n = 2 ** self.q
        self.h = 1.0 / (self.n + 1)

    @property
    def num_nodes(self):
        return self.n ** self.d

    @property
    def num_cells(self):
        return (self.n + 1) ** self.d

    def node_positions(self):
        ax = np.arange(1, self.n + 1) * self.h
        g = np.meshgrid(*([ax] * self.d), indexing="ij")
        return np.column_stack([x.ravel() for x in g])

    def cell_index_grid(self):
        m = self.n + 1
        return np.meshgrid(*([np.arange(m)] * self.d), indexing="ij")


def cell_corner_nodes(grid):
    """Flat interior indices of the 2^d corners of every cell (lexicographic
    corner order), -1 on the boundary (grid_fem.py:189-203)."""
    n, d = grid.n, grid.d
    cells = np.stack([c.ravel() for c in grid.cell_index_grid()], axis=1)   # (ncell, d)
    idx = cells[:, None, :] + corner_offsets(d)[None, :, :]                # (ncell, 2^d, d)
    interior = np.all((idx >= 1) & (idx <= n), axis=2)
    flat = np.zeros(idx.shape[:2], dtype=np.int64)
    for a in range(d):
        flat = flat * n + (idx[:, :, a] - 1)
    return np.where(interior, flat, -1)


def _assemble(grid, element, cell_scale):
    """grid_fem.py:206-214 in d dimensions."""
    corners = cell_corner_nodes(grid)
    nc = corners.shape[1]
    rows = np.repeat(corners, nc, axis=1).ravel()
    cols = np.tile(corners, (1, nc)).ravel()
    vals = (cell_scale[:, None, None] * element[None, :, :]).ravel()
    keep = (rows >= 0) & (cols >= 0)
    N = grid.num_nodes
    return O.canon(sp.coo_array((vals[keep], (rows[keep], cols[keep])), shape=(N, N)))


def assemble_mass(grid):
    mass, _ = element_matrices(grid.d)
    return _assemble(grid, mass, np.full(grid.num_cells, grid.h ** grid.d))


def assemble_stiffness(grid, coef):
    _, stiff = element_matrices(grid.d)
    scale = np.asarray(coef, float) * (grid.h ** (grid.d - 2))
    return _assemble(grid, stiff, scale)


def coefficient_example(grid, kmax=None):
    """d=2: the reference's example1 (grid_fem.py:136-155, k = 1..6);
    d=3: BASELINE config 4's prod_{k=1..5} (1 + 0.5 cos(2^k pi (x+y+z)))
    (1 + 0.5 sin(2^k pi (z - 3x + y))), both at the cell's lower corner index
    (c_i / (n+1)) like the reference."""
    m = grid.n + 1
    c = grid.cell_index_grid()
    if grid.d == 2:
        s = (c[0] + c[1]) / m
        t = (c[1] - 3.0 * c[0]) / m
        kmax = 6 if kmax is None else kmax
    else:
        s = (c[0] + c[1] + c[2]) / m
        t = (c[2] - 3.0 * c[0] + c[1]) / m
        kmax = 5 if kmax is None else kmax
    vals = np.ones_like(s, dtype=float)
    for k in range(1, kmax + 1):
        w = (2.0 ** k) * np.pi
        vals *= (1.0 + 0.5 * np.cos(w * s)) * (1.0 + 0.5 * np.sin(w * t))
    return vals.ravel()


def gaussian_load(grid, seed):
    """Nodal g ~ N(0,1) i.i.d. from default_rng(seed) (BASELINE configs 2-4)."""
    return np.random.default_rng(int(seed)).standard_normal(grid.num_nodes)


# --------------------------------------------------------------------------
# index hierarchy (hierarchy.py:84-219) in d dimensions
# --------------------------------------------------------------------------

def _unflat(flat, side, d):
    out = []
    f = np.asarray(flat, dtype=np.int64)
    for _ in range(d):
        f, r = np.divmod(f, side)
        out.append(r)
    return out[::-1]  # axis 0 first


def _flat(coords, side):
    f = np.zeros_like(coords[0])
    for c in coords:
        f = f * side + c
    return f


def box_indices(side, flat, rho, d):
    """Chebyshev box of half-width floor(rho), clipped, flat ascending
    (hierarchy.py:187-209)."""
    w = int(np.floor(rho))
    cs = [int(c) for c in _unflat(flat, side, d)]
    axes = [np.arange(max(0, c - w), min(side - 1, c + w) + 1) for c in cs]
    g = np.meshgrid(*axes, indexing="ij")
    return _flat([x.ravel() for x in g], side)


def nsub(d):
    return 2 ** d - 1


def chi_indices(k, parent, rho, d):
    """(2^d - 1) subband indices per member of the parent ball
    (hierarchy.py:211-219)."""
    ball = box_indices(2 ** (k - 1), parent, rho, d)
    m = nsub(d)
    return (m * ball[:, None] + np.arange(m)[None, :]).ravel()


def children(k, flat, d):
    """Level-(k+1) children of level-k aggregates, flat ascending
    (hierarchy.py:109-117)."""
    side = 2 ** k
    cs = _unflat(flat, side, d)
    offs = corner_offsets(d)
    kids = [_flat([2 * cs[a][..., None] + offs[None, :, a] for a in range(d)], 2 * side)]
    return kids[0]


def helmert(n):
    """Row-orthonormalized U^(n) of Lemma 4.14 without its all-ones row:
    row t (1-based) = (1, .., 1 [t times], -t, 0, ..) / sqrt(t + t^2)."""
    U = np.zeros((n - 1, n))
    for t in range(1, n):
        U[t - 1, :t] = 1.0
        U[t - 1, t] = -float(t)
    return U * (1.0 / np.sqrt((U ** 2).sum(axis=1)))[:, None]


def null_basis(k, d):
    """W^(k): (2^d - 1) rows per parent over its 2^d children
    (hierarchy.py:161-183, Construction 4.15)."""
    m, c = nsub(d), 2 ** d
    tmpl = helmert(c)
    npar = c ** (k - 1)
    ch = children(k - 1, np.arange(npar), d)                        # (npar, c)
    rows = (m * np.arange(npar)[:, None, None] + np.arange(m)[None, :, None]
            + 0 * ch[:, None, :])
    cols = np.broadcast_to(ch[:, None, :], (npar, m, c))
    vals = np.broadcast_to(tmpl[None], (npar, m, c))
    return O.canon(sp.coo_array((vals.ravel(), (rows.ravel(), cols.ravel())),
                                shape=(m * npar, c ** k)))


def pi_step(k, d):
    """0/1 aggregation pi^(k,k+1) (hierarchy.py:121-134)."""
    side_f = 2 ** (k + 1)
    cols = np.arange((2 ** d) ** (k + 1))
    cs = _unflat(cols, side_f, d)
    rows = _flat([c // 2 for c in cs], side_f // 2)
    return O.canon(sp.coo_array((np.ones(cols.size), (rows, cols)),
                                shape=((2 ** d) ** k, (2 ** d) ** (k + 1))))


# --------------------------------------------------------------------------
# localized transform (gamblet_fast.py:464-674) and solve (677-775)
# --------------------------------------------------------------------------

def mass_inverse(M, q, rho, d):
    """psi^(q) (gamblet_fast.py:464-498)."""
    N = (2 ** d) ** q
    side = 2 ** q
    s, Ms = O.diag_scale(M)
    pos = np.full(N, -1)
    mats, rhss, idxs = [], [], []
    for i in range(N):
        idx = box_indices(side, i, rho, d)
        mats.append(O.principal_dense(Ms, idx, pos))
        rhs = np.zeros(idx.size)
        rhs[int(np.searchsorted(idx, i))] = s[i]
        rhss.append(rhs)
        idxs.append(idx)
    zs = O._batched_solve(mats, rhss)
    rows = np.concatenate([np.full(ix.size, i) for i, ix in enumerate(idxs)])
    cols = np.concatenate(idxs)
    vals = np.concatenate([s[ix] * z for ix, z in zip(idxs, zs)])
    return O.canon(sp.coo_array((vals, (rows, cols)), shape=(N, N)))


def level_step(level, k, rho_coarse, d, with_psi=True, spectral=True):
    """One localized step k -> k-1 (gamblet_fast.py:501-632) with direct
    correction solves; pibar = pi / 2^d."""
    c = 2 ** d
    W = null_basis(k, d)
    A_k = O.canon(level["stiffness"])
    X = O.canon(W @ A_k)
    B, repair_b = O.symmetrize(O.canon(X @ O.canon(W.T)))
    B = O.drop_dead_tails(O.canon(B))
    s_b, Bs = O.diag_scale(B)
    lam_min, lam_max = O.eig_extremes(Bs, tol=0.1) if spectral else (None, None)
    P = pi_step(k - 1, d)
    G = O.canon(X @ O.canon(P.T * (1.0 / c)))
    Gc = sp.csc_array(-G)
    n_coarse = c ** (k - 1)
    pos = np.full(B.shape[0], -1)
    mats, rhss, chis, cols_i = [], [], [], []
    for i in range(n_coarse):
        chi = chi_indices(k, i, rho_coarse, d)
        col = np.zeros(B.shape[0])
        a, b = Gc.indptr[i], Gc.indptr[i + 1]
        col[Gc.indices[a:b]] = Gc.data[a:b]
        rhs = s_b[chi] * col[chi]
        if float(np.linalg.norm(rhs)) == 0.0:
            continue
        mats.append(O.principal_dense(Bs, chi, pos))
        rhss.append(rhs)
        chis.append(chi)
        cols_i.append(i)
    zs = O._batched_solve(mats, rhss)
    if chis:
        rows = np.concatenate(chis)
        cols = np.concatenate([np.full(ch.size, i) for ch, i in zip(chis, cols_i)])
        vals = np.concatenate([s_b[ch] * z for ch, z in zip(chis, zs)])
    else:
        rows = cols = np.zeros(0, int)
        vals = np.zeros(0)
    D = O.canon(sp.coo_array((vals, (rows, cols)), shape=(B.shape[0], n_coarse)))
    Dt = O.drop_row_tails(O.canon(D.T))
    D = O.canon(Dt.T)
    R = O.canon(P * (1.0 / c) + Dt @ W)
    PAPt = O.canon(O.canon(P @ A_k) @ O.canon(P.T))
    GtD = O.canon(O.canon(G.T) @ D)
    DtBD = O.canon(Dt @ O.canon(B @ D))
    raw = (1.0 / (c * c)) * PAPt + GtD + O.canon(GtD.T) + DtBD
    A_next, repair_a = O.symmetrize(O.canon(raw))
    A_next = O.drop_dead_tails(O.canon(A_next))
    psi_next = None
    if with_psi and level.get("psi") is not None:
        psi = level["psi"]
        psi_next = O.drop_row_tails(
            O.canon((1.0 / c) * O.canon(P @ psi) + Dt @ O.canon(W @ psi)))
    level.update(null_w=W, subband=B, subband_scale=s_b, correction=D,
                 restriction=R, lambda_min=lam_min, lambda_max=lam_max,
                 repair=max(level.get("repair", 0.0), repair_b))
    return {"k": k - 1, "psi": psi_next, "stiffness": A_next, "repair": repair_a}


def fast_transform(M, A, q, radii, d, with_psi=True, spectral=True):
    """gamblet_fast.py:635-674."""
    psi = mass_inverse(O.canon(M), q, radii[q - 1], d)
    Aq, repair = O.level_q_stiffness(psi, O.canon(A))
    levels = {q: {"k": q, "psi": psi, "stiffness": Aq, "repair": repair}}
    for k in range(q, 1, -1):
        levels[k - 1] = level_step(levels[k], k, radii[k - 2], d, with_psi=with_psi,
                                   spectral=spectral)
    return levels


def fast_solve(M, A, g_nodal, q, d, epsilon, uniform_rho=None, c_rho=None, spectral=True):
    """fast_solve (gamblet_fast.py:815-837) in d dimensions; the solve phase is
    dimension-free (oracle.solve_with_transform)."""
    radii = O.make_radii(epsilon, q, c_rho, uniform_rho)
    levels = fast_transform(M, A, q, radii, d, spectral=spectral)
    sol = O.solve_with_transform(levels, g_nodal, q, O.subband_tol(epsilon, q))
    return sol, levels, radii


def build_problem(q, d, coeff="example", seed_a=0, seed_g=1):
    """(grid, M, A, g_nodal, b) of the d-D benchmark family: 'example'
    coefficient with the example-style load in 2-D or a Gaussian nodal load
    in 3-D (BASELINE config 4), or 'checker' (log-uniform contrast 1e4)."""
    grid = GridND(q, d)
    if coeff == "example":
        a = coefficient_example(grid)
    else:
        u = np.random.default_rng(int(seed_a)).random(grid.num_cells)
        a = np.exp(u * np.log(1e4))
    M = assemble_mass(grid)
    A = assemble_stiffness(grid, a)
    g = gaussian_load(grid, seed_g)
    return grid, M, A, g, M @ g
