"""The dimension-generic oracle (oracle/gamblets_oracle_nd.py, BASELINE config
4's 3-D restatement): its d=2 instance is pinned to the 2-D oracle, the
package's reference-bitwise builders and the reference goldens; its d=3
instance is checked for the structural identities of the hierarchy and, with
covering radii, for exactness against a direct FE solve."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import paper_1503_03467_b200 as gb
from oracle import gamblets_oracle as O
from oracle import gamblets_oracle_nd as ND


def test_element_matrices_d2_are_the_reference_elements():
    from paper_1503_03467_b200 import grid_fem as gf
    mass, stiff = ND.element_matrices(2)
    # lexicographic corners (0,0),(0,1),(1,0),(1,1) -> reference SW, SE, NE, NW
    perm = [0, 2, 3, 1]
    np.testing.assert_array_equal(mass[np.ix_(perm, perm)], gf.MASS_ELEMENT)
    np.testing.assert_array_equal(stiff[np.ix_(perm, perm)], gf.STIFFNESS_ELEMENT)


def test_element_matrices_d3_identities():
    mass, stiff = ND.element_matrices(3)
    assert abs(mass.sum() - 1.0) < 1e-15            # integrates 1 over the unit cell
    np.testing.assert_allclose(stiff.sum(axis=1), 0.0, atol=1e-15)  # constants in kernel
    np.testing.assert_allclose(stiff, stiff.T)
    assert np.linalg.eigvalsh(stiff)[1] > 0          # one-dimensional kernel


@pytest.mark.parametrize("q", [3, 4])
def test_assembly_d2_matches_reference_builders(q):
    grid2 = gb.build_grid(q)
    coef = gb.coefficient_example1(grid2)
    g = ND.GridND(q, 2)
    np.testing.assert_array_equal(ND.coefficient_example(g), coef.values)
    for mine, ref in ((ND.assemble_mass(g), gb.assemble_mass(grid2)),
                      (ND.assemble_stiffness(g, coef.values),
                       gb.assemble_stiffness(grid2, coef))):
        assert O.same_pattern(mine, ref)
        assert O.rel_fro(mine, ref) <= 1e-15


def test_hierarchy_d2_is_the_2d_hierarchy():
    for k in (2, 3, 4):
        assert (ND.null_basis(k, 2) != O.null_basis(k)).nnz == 0
        assert (ND.pi_step(k - 1, 2) != O.pi_step(k - 1)).nnz == 0
        np.testing.assert_array_equal(ND.children(k - 1, np.arange(4 ** (k - 1)), 2),
                                      O.children(k - 1, np.arange(4 ** (k - 1))))
        for p in (0, 3, 4 ** (k - 1) - 1):
            np.testing.assert_array_equal(ND.chi_indices(k, p, 2, 2), O.chi_indices(k, p, 2))


@pytest.mark.parametrize("k", [1, 2, 3])
def test_hierarchy_d3_identities(k):
    W = ND.null_basis(k + 1, 3)
    P = ND.pi_step(k, 3)
    assert W.shape == (7 * 8 ** k, 8 ** (k + 1))
    np.testing.assert_allclose((W @ W.T).toarray(), np.eye(W.shape[0]), atol=1e-15)
    assert abs(W @ P.T).max() < 1e-15              # W annihilates the aggregate indicators
    np.testing.assert_array_equal(np.asarray(P.sum(axis=1)).ravel(), 8.0)
    ch = ND.children(k, np.arange(8 ** k), 3)
    assert sorted(ch.ravel().tolist()) == list(range(8 ** (k + 1)))


def test_fast_solve_d2_matches_2d_oracle_and_reference_golden(golden, problem):
    q = 4
    p = problem(q, "example1")
    sol, lv, _ = ND.fast_solve(p.M, p.A, p.load.g_nodal, q, 2, 1e-13, uniform_rho=3)
    sol2, lv2, _ = O.fast_solve(p.M, p.A, p.load.g_nodal, q, 1e-13, uniform_rho=3)
    G = golden("fast_q4_example1")
    for k in range(q, 0, -1):
        assert O.rel_fro(lv[k]["stiffness"], lv2[k]["stiffness"]) <= 1e-14
        assert O.rel_fro(lv[k]["stiffness"], G[f"A{k}"]) <= 1e-10
        if k >= 2:
            assert O.rel_fro(lv[k]["restriction"], G[f"R{k}"]) <= 1e-10
            assert O.rel_fro(lv[k]["subband"], G[f"B{k}"]) <= 1e-10
    assert O.rel_energy(p.A, sol["u"], G["u"]) <= 1e-9


@pytest.mark.parametrize("q", [2, 3])
def test_fast_solve_d3_covering_radius_is_the_fe_solution(q):
    """With balls covering every level (rho = 2^q) the localized transform is
    exact: u equals the Q1 finite-element solution A^-1 b to solver tolerance."""
    grid, M, A, g, b = ND.build_problem(q, 3, "example")
    sol, lv, _ = ND.fast_solve(M, A, g, q, 3, 1e-13, uniform_rho=2 ** q, spectral=False)
    # the nodal shortcut g^(q) = g means the reference's measured right-hand
    # side is M g = b with psi^(q) = M^-1 (exact under full cover)
    u_ref = spla.spsolve(sp.csc_array(A), b)
    assert O.rel_energy(A, sol["u"], u_ref) <= 1e-9
    for k in range(2, q + 1):
        assert lv[k]["subband"].shape[0] == 7 * 8 ** (k - 1)


def test_fast_solve_d3_localization_error_decays_with_radius():
    """BASELINE config 4's radius (rho=2) at q=3 runs localized; the error
    against the FE solution is the gamblets' localization error and decays
    exponentially with rho (the 2-D reference shows the same: ~7% at rho=3,
    q=4 for example1) until full cover makes it exact."""
    q = 3
    grid, M, A, g, b = ND.build_problem(q, 3, "example")
    u_ref = spla.spsolve(sp.csc_array(A), b)
    errs = []
    for rho in (1, 2, 3):
        sol, lv, radii = ND.fast_solve(M, A, g, q, 3, 1e-13, uniform_rho=rho,
                                       spectral=(rho == 2))
        errs.append(O.rel_energy(A, sol["u"], u_ref))
        if rho == 2:
            assert radii == (2, 2, 2)
            for k in range(2, q + 1):
                assert 0 < lv[k]["lambda_min"] <= lv[k]["lambda_max"]
    assert errs[0] > 3 * errs[1] > 9 * errs[2]
    assert errs[1] < 0.15


def test_fast_solve_d3_reproduces_committed_golden(golden):
    """tests/golden/fast3d_q3_example.npz (oracle/make_goldens_nd.py) pins the
    3-D restatement: rebuilt inputs bitwise, operators and u unchanged."""
    from oracle.make_goldens import digest
    G = golden("fast3d_q3_example")
    q = int(G["q"])
    grid, M, A, g, b = ND.build_problem(q, 3, "example")
    assert digest(M) == str(G["digest_M"]) and digest(A) == str(G["digest_A"])
    sol, lv, radii = ND.fast_solve(M, A, g, q, 3, 1e-13, uniform_rho=int(G["rho"]))
    for k in range(q, 0, -1):
        assert O.rel_fro(lv[k]["stiffness"], G[f"A{k}"]) <= 1e-13
        assert O.same_pattern(lv[k]["stiffness"], G[f"A{k}"])
        if k >= 2:
            assert O.rel_fro(lv[k]["subband"], G[f"B{k}"]) <= 1e-13
            assert O.rel_fro(lv[k]["restriction"], G[f"R{k}"]) <= 1e-13
    assert O.rel_energy(A, sol["u"], G["u"]) <= 1e-12
