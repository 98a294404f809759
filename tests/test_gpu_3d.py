"""BASELINE config 4 (3-D, Q1 trilinear, 27-point stencil, rho = 2): the
GPU path (paper_1503_03467_b200.gamblet_3d, csrc/gb_3d.cu) against the
dimension-generic CPU restatement oracle/gamblets_oracle_nd.py (its d = 2
instance is pinned to the reference; the reference itself has no 3-D, so
d = 3 parity is against the restatement -- "parity unpinned" upstream of it).

Bars: BASELINE's 1e-10 relative Frobenius on A^(k), B^(k), R (D and s_B held
to the same), identical sparsity patterns, 1e-9 relative energy norm on u.
"""

import numpy as np
import pytest

from oracle import gamblets_oracle as O
from oracle import gamblets_oracle_nd as ND

pytestmark = pytest.mark.gpu

TOL_OP = 1e-10
TOL_U = 1e-9


def _inputs(q, coeff="example"):
    from paper_1503_03467_b200 import gamblet_3d as g3
    grid = g3.build_grid_3d(q)
    c = (g3.coefficient_example_3d(grid) if coeff == "example"
         else g3.coefficient_checkerboard_3d(grid, 1e4, 0))
    M = g3.assemble_mass_3d(grid)
    A = g3.assemble_stiffness_3d(grid, c)
    g = g3.gaussian_load_3d(grid, 1)
    return grid, M, A, g


def _check(got, ref, what):
    err = O.rel_fro(got, ref)
    assert err <= TOL_OP, f"{what}: rel Frobenius {err:.3e}"
    assert O.same_pattern(got, ref), f"{what}: sparsity pattern differs"


def test_3d_inputs_match_the_restatement():
    from oracle.make_goldens import digest
    from paper_1503_03467_b200 import gamblet_3d as g3
    G = np.load("tests/golden/fast3d_q3_example.npz")
    grid, M, A, g = _inputs(3)
    assert digest(M) == str(G["digest_M"]) and digest(A) == str(G["digest_A"])
    np.testing.assert_array_equal(g, G["g"])
    np.testing.assert_array_equal(g3.w_template_3d(), ND.helmert(8))


@pytest.mark.parametrize("q,coeff", [(3, "example"), (4, "example"), (4, "checker")])
def test_3d_fast_solve_matches_restatement(q, coeff):
    from paper_1503_03467_b200 import gamblet_3d as g3
    grid, M, A, g = _inputs(q, coeff)
    res = g3.fast_solve_3d(M, A, g, q, 1e-13, uniform_rho=2)
    sol, lv, radii = ND.fast_solve(M, A, g, q, 3, 1e-13, uniform_rho=2)
    assert tuple(res.radii) == tuple(radii)
    _check(res.levels[q].psi, lv[q]["psi"], f"psi^({q})")
    for k in range(q, 0, -1):
        gl, ol = res.levels[k], lv[k]
        _check(gl.stiffness, ol["stiffness"], f"A^({k})")
        assert gl.symmetry_repair < 1e-12
        if k >= 2:
            _check(gl.subband, ol["subband"], f"B^({k})")
            _check(gl.correction, ol["correction"], f"D^({k},{k - 1})")
            _check(gl.restriction, ol["restriction"], f"R^({k - 1},{k})")
            np.testing.assert_allclose(gl.subband_scale, ol["subband_scale"], rtol=TOL_OP)
            # the reference's eig_extremes on both sides (inner CG to 1e-4)
            np.testing.assert_allclose(gl.lambda_max_subband, ol["lambda_max"], rtol=1e-6)
            np.testing.assert_allclose(gl.lambda_min_subband, ol["lambda_min"], rtol=1e-4)
    err = O.rel_energy(A, res.solution.u, sol["u"])
    assert err <= TOL_U, f"u: rel energy {err:.3e}"
    for k in range(2, q + 1):
        w_ref = sol["coeffs"][k]
        np.testing.assert_allclose(res.solution.subband_coeffs[k], w_ref, rtol=0,
                                   atol=1e-9 * np.abs(w_ref).max())
        e = O.rel_fro(res.solution.increments[k], sol["increments"][k])
        assert e <= 1e-8, f"increment {k}: {e:.3e}"


def test_3d_golden_q3():
    """The committed 3-D fixture (oracle/make_goldens_nd.py): operators at
    every level and u."""
    from paper_1503_03467_b200 import gamblet_3d as g3
    G = np.load("tests/golden/fast3d_q3_example.npz")

    def csr(key):
        import scipy.sparse as sp
        return sp.csr_array((G[f"{key}/data"], G[f"{key}/indices"], G[f"{key}/indptr"]),
                            shape=tuple(G[f"{key}/shape"]))

    grid, M, A, g = _inputs(3)
    res = g3.fast_solve_3d(M, A, g, 3, 1e-13, uniform_rho=int(G["rho"]))
    for k in range(3, 0, -1):
        _check(res.levels[k].stiffness, csr(f"A{k}"), f"A^({k})")
        if k >= 2:
            _check(res.levels[k].subband, csr(f"B{k}"), f"B^({k})")
            _check(res.levels[k].restriction, csr(f"R{k}"), f"R^({k - 1},{k})")
            _check(res.levels[k].correction, csr(f"D{k}"), f"D^({k},{k - 1})")
    assert O.rel_energy(A, res.solution.u, G["u"]) <= TOL_U


def test_3d_solution_is_linear_and_converges_with_rho():
    """Size-independent properties: linearity of u in the load, and rho = 2
    closer than rho = 1 to the exact FE solution."""
    import scipy.sparse.linalg as spla
    from paper_1503_03467_b200 import gamblet_3d as g3
    q = 4
    grid, M, A, g = _inputs(q)
    g2 = np.random.default_rng(9).standard_normal(grid.num_nodes)
    r1 = g3.fast_solve_3d(M, A, g, q, 1e-13, uniform_rho=2)
    r2 = g3.fast_solve_3d(M, A, g2, q, 1e-13, uniform_rho=2)
    r12 = g3.fast_solve_3d(M, A, g + g2, q, 1e-13, uniform_rho=2)
    assert O.rel_energy(A, r1.solution.u + r2.solution.u, r12.solution.u) <= 1e-9
    exact = spla.spsolve(A.tocsc(), M @ g)
    errs = [O.rel_energy(A, g3.fast_solve_3d(M, A, g, q, 1e-13, uniform_rho=r).solution.u, exact)
            for r in (1, 2)]
    assert errs[0] > 2 * errs[1]
    # the shared-memory mass-patch kernel covers rho <= 2 in 3-D (BASELINE: 2)
    with pytest.raises(g3.InvalidArgumentError):
        g3.fast_solve_3d(M, A, g, q, 1e-13, uniform_rho=3)


def test_3d_lanczos_lambda_min_is_the_inverse_iteration():
    """The default lambda_min (Lanczos moments of the start vector) against
    the reference's inverse iteration run verbatim on the same device
    operator (inner CG to 1e-4), at every level of q = 4."""
    from paper_1503_03467_b200 import gamblet_3d as g3
    grid, M, A, g = _inputs(4, "checker")
    res = g3.fast_solve_3d(M, A, g, 4, 1e-13, uniform_rho=2)
    for k, op in res.operators.items():
        lam_min, lam_max = op.eig_extremes(method="cg")
        np.testing.assert_allclose(res.levels[k].lambda_max_subband, lam_max, rtol=1e-12)
        np.testing.assert_allclose(res.levels[k].lambda_min_subband, lam_min, rtol=1e-4)


def test_3d_tiled_products_are_bitwise_the_per_entry_kernels():
    """The register-tiled / column-enumerated split triple product
    (k3_bd_tiled, k3_gtd_bycol, k3_coarse_raw_tiled; gb_tune(6) = 1, default)
    keeps every entry's summation order, so A^(k-1) at every level equals the
    per-entry kernels' bit for bit (clipped patches, odd run lengths: q = 4)."""
    from paper_1503_03467_b200 import _native as nat, gamblet_3d as g3
    grid, M, A, g = _inputs(4, "checker")
    lib = nat.load()
    old = lib.gb_tune(6, -1)
    try:
        lib.gb_tune(6, 0)
        a = g3.fast_solve_3d(M, A, g, 4, 1e-13, uniform_rho=2)
        lib.gb_tune(6, 1)
        b = g3.fast_solve_3d(M, A, g, 4, 1e-13, uniform_rho=2)
    finally:
        lib.gb_tune(6, old)
    for k in range(4, 0, -1):
        sa, sb = a.levels[k].stiffness, b.levels[k].stiffness
        assert O.same_pattern(sa, sb) and np.array_equal(sa.data, sb.data), f"A^({k})"
    assert np.array_equal(a.solution.u, b.solution.u)
