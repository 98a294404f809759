"""Device diagnostics against the reference's own
diagnostics.py outputs on its tight-mode q=5 contrast-1e4 solve
(tests/golden/diag_q5_checker.npz, oracle/make_goldens_diag.py), plus
size-independent properties at q=10.  Our solve agrees with the reference's
to ~1e-13 (test_gpu_parity.py), so the tables agree to the tolerances below."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import diagnostics as D

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def solved(problem):
    p = problem(5, "checker")
    res = gb.fast_solve(p.M, p.A, p.load, p.tree, 1e-13, uniform_rho=3, c_tol=1e-6)
    return p, res


def test_cell_energies_and_decay(golden, solved):
    G = golden("diag_q5_checker")
    p, res = solved
    en = D.cell_energies(p.grid, p.coef, res.solution.u)
    ref = G["energies_u"]
    np.testing.assert_allclose(en, ref, rtol=0, atol=RTOL * np.abs(ref).max())
    # sums to u^T A u (diagnostics.py:41)
    uAu = float(res.solution.u @ (p.A @ res.solution.u))
    assert abs(en.sum() - uAu) <= 1e-12 * uAu
    dec = D.decay_profile(p.grid, p.coef, G["psi_row"], G["center"], G["radii"])
    np.testing.assert_allclose(dec, G["decay"], rtol=0, atol=1e-12)
    assert dec[0] == 1.0 and np.all(np.diff(dec) <= 0)
    # the decay of OUR psi row (same row index) matches too
    row = 3 * 32 + 5
    ours = res.levels[5].psi[[row], :].toarray().ravel()
    dec2 = D.decay_profile(p.grid, p.coef, ours, G["center"], G["radii"])
    np.testing.assert_allclose(dec2, G["decay"], rtol=0, atol=1e-9)
    slope = D.fit_log_slope(G["radii"], dec2)
    assert slope < 0


def test_coefficient_spectrum(golden, solved):
    G = golden("diag_q5_checker")
    p, res = solved
    spec = D.coefficient_spectrum(res.solution, res.levels)
    assert sorted(spec) == list(range(1, 6))
    for k, v in spec.items():
        ref = G[f"spec{k}"]
        np.testing.assert_allclose(v, ref, rtol=0, atol=1e-8 * np.abs(ref).max())


@pytest.mark.parametrize("frac", [1.0, 0.25, 0.05])
def test_compress(golden, solved, frac):
    G = golden("diag_q5_checker")
    p, res = solved
    u_c, rel = D.compress(res.solution, res.levels, p.A, frac)
    ref_u, ref_rel = G[f"compress_u_{frac}"], float(G[f"compress_rel_{frac}"])
    if frac == 1.0:
        assert rel <= 1e-12
    else:
        assert abs(rel - ref_rel) <= 1e-8 * ref_rel
    np.testing.assert_allclose(u_c, ref_u, rtol=0, atol=1e-9 * np.abs(ref_u).max())
    # a device-assembled stiffness gives the same number
    Ad = gb.assemble_stiffness(p.grid, p.coef, device=True)
    _, rel2 = D.compress(res.solution, res.levels, Ad, frac)
    assert rel2 == rel
    with pytest.raises(gb.InvalidArgumentError):
        D.compress(res.solution, res.levels, p.A, 0.0)


def test_convergence_and_conditioning(golden, solved):
    G = golden("diag_q5_checker")
    p, res = solved
    rows = D.convergence_table(res.solution, G["u_ref"], p.A, float(G["lam_a"]),
                               float(G["g_l2"]))
    ref = G["convergence"]
    got = np.array(rows)
    np.testing.assert_array_equal(got[:, 0], ref[:, 0])
    np.testing.assert_allclose(got[:, 1:], ref[:, 1:], rtol=1e-8)
    named = []
    for k in (5, 4):
        shape = tuple(G[f"SBS{k}/shape"])
        named.append((f"SBS{k}", sp.csr_array(
            (G[f"SBS{k}/data"], G[f"SBS{k}/indices"], G[f"SBS{k}/indptr"]), shape=shape)))
    tab = D.conditioning_table(named)
    got = np.array([r[1:] for r in tab], float)
    np.testing.assert_allclose(got, G["conditioning"], rtol=1e-6)
    assert D.config_hash({"q": 5, "a": "x"}) == D.config_hash({"a": "x", "q": 5})


def test_diagnostics_at_full_size():
    """q=10 (config 2): energies sum to the energy, full compression is the
    solution, the convergence table ends at the solution."""
    q = 10
    grid = gb.build_grid(q)
    c = gb.coefficient_checkerboard(grid, 1e4, 0)
    g = np.random.default_rng(1).standard_normal(grid.num_nodes)
    Md = gb.assemble_mass(grid, device=True)
    Ad = gb.assemble_stiffness(grid, c, device=True)
    load = gb.assemble_load(grid, g, mass=Md)
    res = gb.fast_solve(Md, Ad, load, gb.build_hierarchy(grid), 1e-13, uniform_rho=3)
    u = res.solution.u
    en = D.cell_energies(grid, c, u)
    A = Ad.to_csr()
    uAu = float(u @ (A @ u))
    assert abs(en.sum() - uAu) <= 1e-11 * uAu
    _, rel = D.compress(res.solution, res.levels, Ad, 1.0)
    assert rel <= 1e-12
    _, rel_half = D.compress(res.solution, res.levels, Ad, 0.5)
    assert 0.0 < rel_half < 1.0
    rows = D.convergence_table(res.solution, u, Ad, c.lambda_min, 1.0)
    assert rows[-1][1] <= 1e-12 * np.sqrt(uAu)
    errs = [r[1] for r in rows]
    assert errs[0] > errs[-2]
