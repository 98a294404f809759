"""Generate tests/golden/*.npz by running the REFERENCE package itself.

TEST INFRASTRUCTURE ONLY.  Run in the build container (where the read-only
reference lives at /root/reference):

    python oracle/make_goldens.py

The reference is imported from /root/reference/pkg/src and run in tight mode
(SURVEY.md 8(c)): fast_solve(..., epsilon=1e-13, uniform_rho=3, c_tol=1e-6)
and exact_solve(..., tol_mass=1e-14, tol_subband=1e-14).  The outputs pin both
the CPU oracle (tests/test_host_and_oracle.py) and the GPU path
(tests/test_gpu_parity.py).  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def _ref():
    sys.path.insert(0, REF)
    import gamblets  # noqa: F401  (the reference package)
    return gamblets


def problem(gb, q, coeff):
    grid = gb.build_grid(q)
    if coeff == "example1":
        c = gb.coefficient_example1(grid)
        g = gb.example_load(grid)
    elif coeff == "checker":
        # BASELINE configs 2/3: log-uniform contrast 1e4, seeds S_a=0, S_g=1
        c = gb.coefficient_checkerboard(grid, 1e4, 0)
        g = np.random.default_rng(1).standard_normal(grid.num_nodes)
    else:
        raise ValueError(coeff)
    M = gb.assemble_mass(grid)
    A = gb.assemble_stiffness(grid, c)
    load = gb.assemble_load(grid, g, mass=M)
    return grid, c, M, A, load, gb.build_hierarchy(grid)


def digest(mat):
    mat = sp.csr_array(mat)
    h = hashlib.sha256()
    for arr in (mat.indptr.astype(np.int64), mat.indices.astype(np.int64),
                mat.data.astype(np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def put_csr(d, name, mat):
    mat = sp.csr_array(mat)
    d[name + "/indptr"] = mat.indptr.astype(np.int32)
    d[name + "/indices"] = mat.indices.astype(np.int32)
    d[name + "/data"] = mat.data
    d[name + "/shape"] = np.array(mat.shape, np.int64)


def fast_case(gb, q, coeff, name):
    grid, c, M, A, load, tree = problem(gb, q, coeff)
    res = gb.fast_solve(M, A, load, tree, 1e-13, uniform_rho=3, c_tol=1e-6)
    d = {"q": np.int64(q), "epsilon": 1e-13, "uniform_rho": np.int64(3),
         "radii": np.array(res.schedule.radii, np.int64),
         "subband_tol": res.schedule.subband_tol(),
         "digest_M": np.array(digest(M)), "digest_A": np.array(digest(A)),
         "b": load.b, "g_nodal": load.g_nodal, "coef": c.values}
    for k, lv in res.levels.items():
        put_csr(d, f"A{k}", lv.stiffness)
        put_csr(d, f"psi{k}", lv.psi)
        if k >= 2:
            put_csr(d, f"B{k}", lv.subband)
            put_csr(d, f"D{k}", lv.correction)
            put_csr(d, f"R{k}", lv.restriction)
            d[f"s{k}"] = lv.subband_scale
            d[f"lam{k}"] = np.array([lv.lambda_min_subband, lv.lambda_max_subband])
    sol = res.solution
    d["u"] = sol.u
    d["u1"] = sol.u1_coarse
    for k, w in sol.subband_coeffs.items():
        d[f"w{k}"] = w
    for k, inc in sol.increments.items():
        d[f"inc{k}"] = inc
    its = res.counter.iterations
    d["iters_line8"] = np.array(its.get("line8", []), np.int64)
    d["iters_line16"] = np.array(its.get("line16", []), np.int64)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print("wrote", name)


def sketch(X):
    """X @ Omega with a fixed Gaussian Omega (ncols x 8, seeded by ncols):
    ||(X - Y) Omega||_F / ||Y Omega||_F tracks the relative Frobenius error of
    X against Y entry by entry (E||E Omega||^2 = 8 ||E||_F^2), so the dense
    exact-path levels are pinned without storing them."""
    X = np.asarray(X.toarray() if sp.issparse(X) else X, dtype=float)
    om = np.random.default_rng(1000 + X.shape[1]).standard_normal((X.shape[1], 8))
    return X @ om


def sketch_err(X, sk):
    """Relative error of X against a stored reference sketch X_ref @ Omega."""
    mine = sketch(X)
    return float(np.linalg.norm(mine - sk) / np.linalg.norm(sk))


def exact_case(gb, q, coeff, name, full):
    grid, c, M, A, load, tree = problem(gb, q, coeff)
    sol, levels = gb.exact_solve(M, A, load, tree, tol_mass=1e-14, tol_subband=1e-14)
    d = {"q": np.int64(q), "digest_M": np.array(digest(M)),
         "digest_A": np.array(digest(A)), "u": sol.u, "u1": sol.u1_coarse}
    for k, lv in levels.items():
        d[f"fro_A{k}"] = np.linalg.norm(lv.stiffness)
        d[f"fro_psi{k}"] = np.linalg.norm(lv.psi)
        d[f"sk_A{k}"] = sketch(lv.stiffness)
        d[f"sk_psi{k}"] = sketch(lv.psi)
        if k >= 2:
            d[f"sk_B{k}"] = sketch(lv.subband)
            d[f"sk_R{k}"] = sketch(lv.restriction)
            d[f"sk_D{k}"] = sketch(lv.correction)
        if full or k <= 2:
            d[f"A{k}"] = lv.stiffness
            d[f"psi{k}"] = lv.psi
        if k >= 2:
            d[f"fro_B{k}"] = np.linalg.norm(lv.subband)
            d[f"fro_R{k}"] = np.linalg.norm(lv.restriction)
            d[f"fro_D{k}"] = np.linalg.norm(lv.correction)
            if full or k <= 2:
                d[f"B{k}"] = lv.subband
                d[f"R{k}"] = lv.restriction
                d[f"D{k}"] = lv.correction
            d[f"w{k}"] = sol.subband_coeffs[k]
    for k, inc in sol.increments.items():
        d[f"inc{k}"] = inc
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print("wrote", name)


def pins(gb):
    """Values the reference's own tests pin (copied as numbers, computed here
    by calling the reference)."""
    tree = gb.IndexTree(3)
    d = {
        "chi_q3_k3_c5_r1": tree.chi_neighborhood(3, 5, 1),
        "radii_1e-3_q5": np.array(gb.make_schedule(1e-3, 5).radii),
        "radii_1e-4_q5": np.array(gb.make_schedule(1e-4, 5).radii),
        "radii_1e-3_q7": np.array(gb.make_schedule(1e-3, 7).radii),
        "radii_u3_q4": np.array(gb.make_schedule(1e-3, 4, uniform_rho=3).radii),
    }
    grid = gb.build_grid(6)
    load = gb.assemble_load(grid, gb.example_load(grid))
    d["load_q6_norm"] = np.linalg.norm(load.b)
    d["load_q6_abs"] = np.abs(load.b).sum()
    coef = gb.coefficient_example1(grid)
    d["ex1_q6_minmax"] = np.array([coef.lambda_min, coef.lambda_max])
    for q in (3, 5, 7, 10):
        grid = gb.build_grid(q)
        d[f"digest_M_q{q}"] = np.array(digest(gb.assemble_mass(grid)))
        d[f"digest_Aex1_q{q}"] = np.array(digest(
            gb.assemble_stiffness(grid, gb.coefficient_example1(grid))))
        d[f"digest_Achk_q{q}"] = np.array(digest(
            gb.assemble_stiffness(grid, gb.coefficient_checkerboard(grid, 1e4, 0))))
    np.savez_compressed(OUT / "pins.npz", **d)
    print("wrote pins")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    gb = _ref()
    if sys.argv[1:] == ["exact"]:  # regenerate only the exact-path fixtures
        exact_case(gb, 3, "example1", "exact_q3_example1", full=True)
        exact_case(gb, 5, "example1", "exact_q5_example1", full=False)
        return
    pins(gb)
    fast_case(gb, 4, "example1", "fast_q4_example1")
    fast_case(gb, 5, "checker", "fast_q5_checker")
    fast_case(gb, 5, "example1", "fast_q5_example1")
    exact_case(gb, 3, "example1", "exact_q3_example1", full=True)
    exact_case(gb, 5, "example1", "exact_q5_example1", full=False)


if __name__ == "__main__":
    main()
