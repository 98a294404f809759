"""GPU Krylov API (sparse_core.cg_solve / cg_solve_block / eig_extremes),
ported from the reference's test_sparse_core.py contracts."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gamblets_oracle as O
from paper_1503_03467_b200 import krylov
from paper_1503_03467_b200.errors import InvalidArgumentError, NumericalError

pytestmark = pytest.mark.gpu


def _spd(n, seed):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((n, n))
    return Q @ Q.T + n * np.eye(n)


def test_cg_identity_one_iteration():
    x, rep = krylov.cg_solve(sp.eye_array(5, format="csr"), np.arange(1.0, 6.0))
    np.testing.assert_allclose(x, np.arange(1.0, 6.0))
    assert rep.iterations == 1 and rep.converged


def test_cg_finite_termination_two_eigenvalues():
    A = sp.diags_array(np.array([1.0, 1.0, 3.0, 3.0]), format="csr")
    _, rep = krylov.cg_solve(A, np.ones(4), rel_tol=1e-14)
    assert rep.iterations <= 2 and rep.converged


def test_cg_zero_rhs():
    x, rep = krylov.cg_solve(sp.eye_array(3, format="csr") * 2.0, np.zeros(3))
    assert np.all(x == 0.0) and rep.iterations == 0 and rep.converged


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_cg_matches_oracle_and_residual_contract(seed):
    A = _spd(40, seed)
    b = np.random.default_rng(seed + 10).standard_normal(40)
    x, rep = krylov.cg_solve(A, b, rel_tol=1e-10)
    assert np.linalg.norm(b - A @ x) <= 1e-10 * np.linalg.norm(b) * 1.0001
    xo, it, _ = O.cg(A, b, 1e-10)
    assert abs(rep.iterations - it) <= 1
    np.testing.assert_allclose(x, xo, rtol=0, atol=1e-9 * np.abs(xo).max())


def test_cg_max_iter_reported_not_fatal():
    A = _spd(30, 3)
    _, rep = krylov.cg_solve(A, np.ones(30), rel_tol=1e-15, max_iter=2)
    assert rep.iterations == 2 and not rep.converged


def test_cg_breakdown_on_indefinite():
    with pytest.raises(NumericalError):
        krylov.cg_solve(-sp.eye_array(4, format="csr"), np.ones(4))


def test_cg_warm_start_and_guards():
    A = _spd(20, 4)
    b = np.ones(20)
    x_exact = np.linalg.solve(A, b)
    _, rep = krylov.cg_solve(A, b, x0=x_exact)
    assert rep.iterations == 0
    with pytest.raises(InvalidArgumentError):
        krylov.cg_solve(A, np.ones(3))


def test_block_cg_matches_columnwise():
    A = _spd(25, 5)
    B = np.random.default_rng(6).standard_normal((25, 4))
    B[:, 2] = 0.0
    X, its, rel, ok = krylov.cg_solve_block(A, B, rel_tol=1e-11)
    for j in range(4):
        x, rep = krylov.cg_solve(A, B[:, j], rel_tol=1e-11)
        np.testing.assert_array_equal(X[:, j], x)
        assert its[j] == rep.iterations
    assert its[2] == 0 and ok.all()


def test_eig_extremes_match_oracle_and_dense():
    A = sp.csr_array(_spd(60, 7))
    lo, hi = krylov.eig_extremes(A, tol=1e-3)
    lo_o, hi_o = O.eig_extremes(A, tol=1e-3)
    np.testing.assert_allclose([lo, hi], [lo_o, hi_o], rtol=1e-8)
    w = np.linalg.eigvalsh(A.toarray())
    # the reference algorithm stops on a relative change of 0.5 tol, so its
    # estimate of a clustered lower spectrum is only a few percent accurate
    assert lo == pytest.approx(w[0], rel=5e-2) and hi == pytest.approx(w[-1], rel=1e-2)
