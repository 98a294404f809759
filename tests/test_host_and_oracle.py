"""CPU tests: the oracle pinned against the reference's golden outputs, the
package's host-side input builders and index maps against the reference
(bitwise), and the C ABI library's exported symbols (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1503_03467_b200 as gb
from oracle import gamblets_oracle as O
from oracle.make_goldens import digest

ROOT = Path(__file__).resolve().parents[1]


# --- oracle pinned to the reference -----------------------------------------

@pytest.mark.parametrize("name,q,coeff", [
    ("fast_q4_example1", 4, "example1"),
    ("fast_q5_checker", 5, "checker"),
])
def test_oracle_fast_matches_reference(golden, problem, oracle_fast, name, q, coeff):
    G = golden(name)
    sol, lv, radii = oracle_fast(q, coeff)
    assert tuple(radii) == tuple(G["radii"])
    for k in range(q, 0, -1):
        assert O.rel_fro(lv[k]["stiffness"], G[f"A{k}"]) <= 1e-12
        assert O.same_pattern(lv[k]["stiffness"], G[f"A{k}"])
        assert O.rel_fro(lv[k]["psi"], G[f"psi{k}"]) <= 1e-12
        assert O.same_pattern(lv[k]["psi"], G[f"psi{k}"])
        if k >= 2:
            for key, g in (("subband", "B"), ("restriction", "R"), ("correction", "D")):
                assert O.rel_fro(lv[k][key], G[f"{g}{k}"]) <= 1e-12, (key, k)
                assert O.same_pattern(lv[k][key], G[f"{g}{k}"]), (key, k)
            np.testing.assert_allclose([lv[k]["lambda_min"], lv[k]["lambda_max"]],
                                       G[f"lam{k}"], rtol=1e-9)
    p = problem(q, coeff)
    assert O.rel_energy(p.A, sol["u"], G["u"]) <= 1e-12


def test_oracle_exact_matches_reference(golden, problem):
    G = golden("exact_q3_example1")
    p = problem(3)
    sol, lv = O.exact_solve(p.M, p.A, p.load.b, 3)
    for k in range(3, 0, -1):
        assert O.rel_fro(lv[k]["stiffness"], G[f"A{k}"]) <= 1e-12
        assert O.rel_fro(lv[k]["psi"], G[f"psi{k}"]) <= 1e-12
    assert O.rel_energy(p.A, sol["u"], G["u"]) <= 1e-12


def test_oracle_exact_q5_matches_reference_every_level(golden, problem):
    """Config 0 (q = 5): the oracle's exact sweep against the reference's
    A, psi, B, R, D at every level (sketches) and u."""
    from oracle.make_goldens import sketch_err
    G = golden("exact_q5_example1")
    p = problem(5)
    sol, lv = O.exact_solve(p.M, p.A, p.load.b, 5)
    for k in range(5, 0, -1):
        assert sketch_err(lv[k]["stiffness"], G[f"sk_A{k}"]) <= 1e-12, k
        assert sketch_err(lv[k]["psi"], G[f"sk_psi{k}"]) <= 1e-12, k
        if k >= 2:
            assert sketch_err(lv[k]["subband"], G[f"sk_B{k}"]) <= 1e-12, k
            assert sketch_err(lv[k]["restriction"], G[f"sk_R{k}"]) <= 1e-12, k
            assert sketch_err(lv[k]["correction"], G[f"sk_D{k}"]) <= 1e-12, k
    assert O.rel_energy(p.A, sol["u"], G["u"]) <= 1e-12


def test_oracle_reproduces_reference_goldens_json(problem):
    """The reference's own pinned values (pkg/tests/golden/goldens.json:
    fast/q4/relerr and fast/q4/biorth_defect, rtol 1e-3), reproduced by the
    oracle at the reference's default schedule."""
    gold_relerr = [9.597639903617125e-4, 8.017142494668527e-6]
    gold_biorth = [2.6573471127002216e-5, 7.159738350518316e-6]
    p = problem(4)
    ex, _ = O.exact_solve(p.M, p.A, p.load.b, 4)
    errs, defs = [], []
    for eps in (1e-3, 1e-4):
        sol, lv, _ = O.fast_solve(p.M, p.A, p.load.g_nodal, 4, eps, spectral=False)
        errs.append(O.rel_energy(p.A, sol["u"], ex["u"]))
        worst = 0.0
        for k in (1, 2, 3, 4):
            Gm = (O.phi(k, 4, p.M) @ lv[k]["psi"].T).toarray()
            worst = max(worst, float(np.abs(Gm - np.eye(Gm.shape[0])).max()))
        defs.append(worst)
    np.testing.assert_allclose(errs, gold_relerr, rtol=1e-3)
    np.testing.assert_allclose(defs, gold_biorth, rtol=1e-3)


def test_pinned_index_maps_and_schedules(golden):
    P = golden("pins")
    tree = gb.IndexTree(3)
    np.testing.assert_array_equal(tree.chi_neighborhood(3, 5, 1), P["chi_q3_k3_c5_r1"])
    np.testing.assert_array_equal(O.chi_indices(3, 5, 1), P["chi_q3_k3_c5_r1"])
    assert gb.make_schedule(1e-3, 5).radii == tuple(P["radii_1e-3_q5"])
    assert gb.make_schedule(1e-4, 5).radii == tuple(P["radii_1e-4_q5"])
    assert gb.make_schedule(1e-3, 7).radii == tuple(P["radii_1e-3_q7"])
    assert gb.make_schedule(1e-3, 4, uniform_rho=3).radii == tuple(P["radii_u3_q4"])
    assert O.make_radii(1e-3, 7) == tuple(P["radii_1e-3_q7"])


# --- host-side builders reproduce the reference bitwise --------------------

@pytest.mark.parametrize("q", [3, 5, 7, 10])
def test_assembly_is_bitwise_reference(golden, q):
    P = golden("pins")
    grid = gb.build_grid(q)
    assert digest(gb.assemble_mass(grid)) == str(P[f"digest_M_q{q}"])
    assert digest(gb.assemble_stiffness(grid, gb.coefficient_example1(grid))) == \
        str(P[f"digest_Aex1_q{q}"])
    assert digest(gb.assemble_stiffness(grid, gb.coefficient_checkerboard(grid, 1e4, 0))) \
        == str(P[f"digest_Achk_q{q}"])


def test_load_and_coefficient_pins(golden):
    P = golden("pins")
    grid = gb.build_grid(6)
    load = gb.assemble_load(grid, gb.example_load(grid))
    assert np.linalg.norm(load.b) == P["load_q6_norm"]
    assert np.abs(load.b).sum() == P["load_q6_abs"]
    coef = gb.coefficient_example1(grid)
    np.testing.assert_array_equal([coef.lambda_min, coef.lambda_max], P["ex1_q6_minmax"])


def test_hierarchy_maps_match_oracle():
    tree = gb.IndexTree(5)
    for k in range(2, 6):
        for variant in ("orthonormal", "chain"):
            W = tree.null_basis(k, variant)
            assert O.same_pattern(W, O.null_basis(k, variant))
            assert O.rel_fro(W, O.null_basis(k, variant)) == 0.0
        P = tree.pi_step(k - 1)
        assert O.rel_fro(P, O.pi_step(k - 1)) == 0.0
        for i in sorted({0, min(7, 4 ** (k - 1) - 1), 4 ** (k - 1) - 1}):
            np.testing.assert_array_equal(tree.neighborhood(k - 1, i, 3),
                                          O.box_indices(2 ** (k - 1), i, 3))
            np.testing.assert_array_equal(tree.chi_neighborhood(k, i, 3),
                                          O.chi_indices(k, i, 3))
    W = tree.null_basis(4)
    assert np.all(np.abs((W @ np.ones(W.shape[1]))) == 0.0)
    assert np.allclose((W @ W.T).toarray(), np.eye(W.shape[0]))


def test_tree_and_schedule_guards():
    for bad in (0, -2, 1.5, True, "3"):
        with pytest.raises(gb.InvalidArgumentError):
            gb.IndexTree(bad)
    for eps in (0.0, 1.0, -0.5):
        with pytest.raises(gb.InvalidArgumentError):
            gb.make_schedule(eps, 4)
    with pytest.raises(gb.InvalidArgumentError):
        gb.make_schedule(1e-3, 4, uniform_rho=0)
    with pytest.raises(gb.InvalidArgumentError):
        gb.make_schedule(1e-3, 4).rho(5)
    with pytest.raises(gb.InvalidArgumentError):
        gb.build_grid(13)


# --- the C ABI ----------------------------------------------------------------

def test_library_exports_every_header_symbol():
    from paper_1503_03467_b200 import _native
    header = (ROOT / "include" / "gamblets_b200.h").read_text()
    declared = set(re.findall(r"^(?:int|size_t|const char\*|unsigned long long)\s+(gb3?_\w+)\(", header, re.M))
    assert len(declared) > 40
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.EXPORTED)
    assert lib.gb_abi_version() == 7


def _lanczos_ab(A, v0, m):
    """m plain Lanczos steps (no reorthogonalization, as on the GPU)."""
    v = v0 / np.linalg.norm(v0)
    vp = np.zeros_like(v)
    beta = 0.0
    ab = []
    for _ in range(m):
        w = A @ v - beta * vp
        alpha = float(v @ w)
        w -= alpha * v
        beta = float(np.linalg.norm(w))
        ab += [alpha, beta]
        vp, v = v, w / beta
    return np.array(ab)


def _emulate(ab, tol=0.1, max_outer=500):
    from paper_1503_03467_b200 import _native
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    lam, rmin, rmax = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    outer = ctypes.c_int()
    buf = np.ascontiguousarray(ab, dtype=np.float64)
    rc = lib.gb_lanczos_emulate(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(len(ab) // 2),
                                ctypes.c_double(tol), ctypes.c_int(max_outer), ctypes.byref(lam),
                                ctypes.byref(outer), ctypes.byref(rmin), ctypes.byref(rmax))
    return rc, lam.value, outer.value, rmin.value, rmax.value


@pytest.mark.parametrize("n,cond", [(60, 50.0), (300, 3e3)])
def test_lanczos_emulation_reproduces_inverse_iteration(n, cond):
    """Level engine spectral mode 1 (csrc/gb_lanczos.h): the inverse-iteration
    sequence of sparse_core.py:258-277 evaluated from the Lanczos moments of
    its start vector equals the iteration run with exact solves -- estimate
    and stopping index -- and matches the reference restatement (inner CG at
    1e-4) to its inner tolerance."""
    rng = np.random.default_rng(7)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.geomspace(1.0 / cond, 1.0, n) * (1 + 0.01 * rng.standard_normal(n))
    A = (Q * ev) @ Q.T
    A = 0.5 * (A + A.T)
    x1, x2 = O.start_vectors(n)
    # the reference's iteration with exact inner solves
    x = x2 / np.linalg.norm(x2)
    lam_prev, outer_exact = np.inf, None
    for j in range(1, 501):
        y = np.linalg.solve(A, x)
        x = y / np.linalg.norm(y)
        lam = float(x @ (A @ x))
        if abs(lam - lam_prev) <= 0.05 * abs(lam):
            outer_exact = j
            break
        lam_prev = lam
    rc, lz, outer, rmin, rmax = _emulate(_lanczos_ab(A, x2, 2 * n))
    assert rc == 0
    assert outer == outer_exact
    assert abs(lz - lam) <= 1e-9 * lam
    assert abs(rmin - ev.min()) <= 1e-3 * ev.min() and abs(rmax - ev.max()) <= 1e-6
    lam_ref, _ = O.eig_extremes(sp.csr_array(A), tol=0.1)
    assert abs(lz - lam_ref) <= 1e-3 * lam_ref


def test_lanczos_emulation_flags_indefinite_operator():
    A = np.diag([-1.0, 1.0, 2.0, 3.0])
    with np.errstate(divide="ignore", invalid="ignore"):
        ab = _lanczos_ab(A, np.ones(4), 4)
    rc = _emulate(ab)[0]
    assert rc == 2


def _check(ab, lz_tol=1e-4, tol=0.1, max_outer=500):
    from paper_1503_03467_b200 import _native
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    lam, outer, stop = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    buf = np.ascontiguousarray(ab, dtype=np.float64)
    rc = lib.gb_lanczos_check(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(len(ab) // 2),
                              ctypes.c_double(tol), ctypes.c_int(max_outer),
                              ctypes.c_double(lz_tol), ctypes.byref(lam), ctypes.byref(outer),
                              ctypes.byref(stop))
    return rc, lam.value, outer.value, stop.value


def test_lanczos_check_matches_emulation_and_stops_when_converged():
    """gb_lanczos_check (the engines' convergence test): its O(m) evaluation
    equals the eigen-decomposition one on every leading T_m, and walking the
    engine's check points (64, 96, 128, ...) it stops at a point whose
    estimate is within lz_tol of the converged one, not before the estimates
    have settled."""
    rng = np.random.default_rng(11)
    n = 700
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.geomspace(2e-4, 1.0, n)
    A = (Q * ev) @ Q.T
    A = 0.5 * (A + A.T)
    ab = _lanczos_ab(A, rng.standard_normal(n), 640)
    lam_final = _emulate(ab)[1]
    for m in (1, 2, 17, 64, 333, 640):
        rc, lam, outer, _, _ = _emulate(ab[:2 * m])
        rc2, lam2, outer2, _ = _check(ab[:2 * m])
        assert rc == 0 and rc2 == 0
        assert outer2 == outer
        assert abs(lam2 - lam) <= 1e-11 * lam
    stops = []
    for lz_tol in (1e-2, 1e-4, 1e-6):
        for m in range(64, 641, 32):
            rc, lam, outer, stop = _check(ab[:2 * m], lz_tol=lz_tol)
            assert rc == 0
            if stop:
                break
        assert stop, "the sequence converges well inside 640 steps"
        assert abs(lam - lam_final) <= 2 * lz_tol * lam_final
        stops.append(m)
    assert stops[0] < stops[1] < stops[2]
    assert _check(ab[:2 * 64], lz_tol=1e-6)[3] == 0


def test_lanczos_check_flags_indefinite_operator():
    A = np.diag([-1.0, 1.0, 2.0, 3.0])
    with np.errstate(divide="ignore", invalid="ignore"):
        ab = _lanczos_ab(A, np.ones(4), 4)
    assert _check(ab)[0] == 2


def test_matrix_market_roundtrip_and_bad_transform_file(tmp_path):
    from paper_1503_03467_b200.persistence import load_transform, mm_read, mm_write
    rng = np.random.default_rng(3)
    m = sp.random_array((40, 30), density=0.2, random_state=rng, format="csr")
    mm_write(tmp_path / "m.mtx", m)
    back = mm_read(tmp_path / "m.mtx")
    assert np.array_equal(back.toarray(), m.toarray())
    np.savez(tmp_path / "bad.npz", x=np.zeros(3))
    with pytest.raises(gb.InvalidArgumentError):
        load_transform(tmp_path / "bad.npz")
