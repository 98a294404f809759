"""Parity at BASELINE.json config 2's full size (q = 10, 1 048 576 fine DOFs,
contrast 1e4) -- where the oracle cannot run end to end -- through checks
that do not depend on the size:

* windowed: finest-level correction patches and restriction rows at chosen
  coarse nodes (corners, edges, interior) recomputed on the host from the
  GPU's own A^(10) and B^(10) rows with a dense solve (gamblet_fast.py:546-591);
* per level: the oracle's level step on the GPU's A^(k) for coarse levels;
* the solve: linearity in the load and bitwise repeatability of
  solve_with_transform on the stored transform (test_gamblet_fast.py:230-244).
"""

import numpy as np
import pytest

from oracle import gamblets_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

Q = 10
RHO = 3


@pytest.fixture(scope="module")
def c2():
    import torch
    import paper_1503_03467_b200 as gb
    from bench import build_inputs
    grid, M, A, load, tree = build_inputs(Q, "checker")
    res = gb.fast_solve(M, A, load, tree, 1e-13, uniform_rho=RHO, c_tol=1e-6)
    torch.cuda.synchronize()
    return grid, M, A, load, tree, res


def _rows(box, rows):
    import torch
    from paper_1503_03467_b200 import device as dv
    v = box.vals.view(-1, box.slots)
    idx = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=v.device)
    return dv.to_host(v.index_select(0, idx))


def _vec(t, idx):
    import torch
    from paper_1503_03467_b200 import device as dv
    return dv.to_host(t.index_select(0, torch.as_tensor(np.asarray(idx, np.int64),
                                                        device=t.device)))


@pytest.mark.parametrize("node", [(0, 0), (0, 255), (511, 511), (256, 257), (3, 400), (137, 63)])
def test_finest_correction_patch_and_restriction_windows(c2, node):
    from paper_1503_03467_b200.hierarchy import w_template
    grid, M, A, load, tree, res = c2
    lv = res.levels[Q]
    Bb, Ab = lv.raw("subband"), lv.raw("stiffness")
    Dtb, Rb = lv.raw("correction"), lv.raw("restriction")
    sB = lv.raw("subband_scale")
    Lp, L = 2 ** (Q - 1), 2 ** Q
    wB, wA = Bb.w, Ab.w
    W = w_template("orthonormal")
    si, ti = node
    i = si * Lp + ti
    ps = np.arange(max(0, si - RHO), min(Lp - 1, si + RHO) + 1)
    pt = np.arange(max(0, ti - RHO), min(Lp - 1, ti + RHO) + 1)
    ball = [(a, b) for a in ps for b in pt]
    chi = [((a * Lp + b) * 3 + c, a, b, c) for a, b in ball for c in range(3)]
    rows = [r for r, *_ in chi]
    Brows = _rows(Bb, rows)
    s = _vec(sB, rows)
    m = len(chi)
    K = np.zeros((m, m))
    W2 = 2 * wB + 1
    for l1, (r1, a1, b1, c1) in enumerate(chi):
        for l2, (r2, a2, b2, c2_) in enumerate(chi):
            ds, dt = a2 - a1, b2 - b1
            if abs(ds) <= wB and abs(dt) <= wB:
                K[l1, l2] = Brows[l1, ((ds + wB) * W2 + dt + wB) * 3 + c2_] * s[l1] * s[l2]
    # G[(p,c), i] = sum_{a in children(p)} W[c, a] sum_{b in children(i)} A[a, b] / 4
    kids = lambda a, b: [(2 * a + u, 2 * b + v) for u in (0, 1) for v in (0, 1)]
    ki = kids(si, ti)
    WA2 = 2 * wA + 1
    G = np.zeros(m)
    for l, (r, a, b, c) in enumerate(chi):
        ka = kids(a, b)
        Arows = _rows(Ab, [x * L + y for x, y in ka])
        acc = 0.0
        for j, (x, y) in enumerate(ka):
            sa = 0.0
            for (u, v) in ki:
                dx, dy = u - x, v - y
                if abs(dx) <= wA and abs(dy) <= wA:
                    sa += Arows[j, (dx + wA) * WA2 + dy + wA]
            acc += W[c, j] * sa * 0.25
        G[l] = acc
    z = np.linalg.solve(K, s * (-G))
    d = s * z
    d[np.abs(d) < 1e-11 * np.abs(d).max()] = 0.0          # row-tail trim of D^T
    Dt = _rows(Dtb, [i])[0]
    R1 = 2 * RHO + 1
    got = np.array([Dt[((a - si + RHO) * R1 + (b - ti + RHO)) * 3 + c] for _, a, b, c in chi])
    assert np.linalg.norm(got - d) <= 1e-10 * np.linalg.norm(d)
    assert np.array_equal(got != 0.0, d != 0.0)
    # R row i: pibar + D^T W on the children of each ball parent
    Rrow = _rows(Rb, [i])[0]
    for (a, b) in ball:
        for j in range(4):
            want = (0.25 if (a, b) == (si, ti) else 0.0) + sum(
                got[[l for l, (_, aa, bb, _c) in enumerate(chi) if (aa, bb) == (a, b)][c]]
                * W[c, j] for c in range(3))
            have = Rrow[((a - si + RHO) * R1 + (b - ti + RHO)) * 4 + j]
            assert abs(have - want) <= 1e-12 * max(1.0, abs(want))


@pytest.mark.parametrize("k", [7, 6])
def test_coarse_levels_match_oracle_level_step(c2, k):
    grid, M, A, load, tree, res = c2
    lv = res.levels[k]
    ref = {"k": k, "stiffness": lv.stiffness}
    nxt = O.level_step(ref, k, RHO, with_psi=False, spectral=False)
    for name, got, want in (("B", lv.subband, ref["subband"]),
                            ("R", lv.restriction, ref["restriction"]),
                            ("D", lv.correction, ref["correction"]),
                            ("A", res.levels[k - 1].stiffness, nxt["stiffness"])):
        assert O.rel_fro(got, want) <= 1e-10, (name, O.rel_fro(got, want))
        assert O.same_pattern(got, want), name


def test_solve_is_linear_and_repeatable_at_full_size(c2):
    import paper_1503_03467_b200 as gb
    grid, M, A, load, tree, res = c2
    sched = res.schedule
    rng = np.random.default_rng(7)
    g1 = rng.standard_normal(grid.num_nodes)
    g2 = rng.standard_normal(grid.num_nodes)
    sol = {}
    for name, g in (("1", g1), ("2", g2), ("12", g1 + g2)):
        ld = gb.assemble_load(grid, g, mass=M)
        sol[name], _ = gb.solve_with_transform(res.levels, ld, tree, sched)
    u1, u2, u12 = sol["1"].u, sol["2"].u, sol["12"].u
    assert O.rel_energy(A, u1 + u2, u12) <= 1e-9
    again, _ = gb.solve_with_transform(res.levels, gb.assemble_load(grid, g1, mass=M), tree,
                                       sched)
    assert np.array_equal(again.u, u1)
