"""Generate tests/golden/diag_q5_checker.npz by running the REFERENCE
package's diagnostics (diagnostics.py) on its own tight-mode fast_solve.

TEST INFRASTRUCTURE ONLY (build container; /root/reference is read-only and
absent on the GPU box):

    python oracle/make_goldens_diag.py

Pins the device diagnostics of paper_1503_03467_b200.diagnostics
(tests/test_gpu_diagnostics.py): cell energies of u, the energy-decay
profile of one psi^(q) row, the coefficient spectrum, compress at three keep
fractions, the convergence table against a direct solve, and the
conditioning table of S B^(k) S.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as sla

from make_goldens import OUT, _ref, problem


def main():
    gb = _ref()
    from gamblets import diagnostics as D
    q = 5
    grid, c, M, A, load, tree = problem(gb, q, "checker")
    res = gb.fast_solve(M, A, load, tree, 1e-13, uniform_rho=3, c_tol=1e-6)
    sol, levels = res.solution, res.levels
    d = {"q": np.int64(q)}
    d["energies_u"] = D.cell_energies(grid, c, sol.u)
    row = 3 * (1 << q) + 5                      # one interior fine node
    psi_row = levels[q].psi[[row], :].toarray().ravel()
    d["psi_row"] = psi_row
    center = grid.node_positions()[row]
    radii = np.arange(0, 12) * grid.h
    d["center"] = np.asarray(center, float)
    d["radii"] = radii
    d["decay"] = D.decay_profile(grid, c, psi_row, center, radii)
    # the reference's spectrum / compress read np.diag of the level operators
    # (dense in its exact path); hand it dense copies of the fast-path levels
    from types import SimpleNamespace
    dense = {}
    for k, lv in levels.items():
        dense[k] = SimpleNamespace(
            k=k, psi=lv.psi.toarray(), stiffness=lv.stiffness.toarray(),
            subband=lv.subband.toarray() if k >= 2 else None,
            null_w=lv.null_w.toarray() if k >= 2 else None)
    levels = dense
    spec = D.coefficient_spectrum(sol, levels)
    for k, v in spec.items():
        d[f"spec{k}"] = v
    for frac in (1.0, 0.25, 0.05):
        u_c, rel = D.compress(sol, levels, A, frac)
        d[f"compress_u_{frac}"] = u_c
        d[f"compress_rel_{frac}"] = np.float64(rel)
    u_ref = sla.spsolve(A.tocsc(), load.b)
    d["u_ref"] = u_ref
    lam_a = c.lambda_min
    g_l2 = gb.l2_norm(M, load.g_nodal)
    d["lam_a"], d["g_l2"] = np.float64(lam_a), np.float64(g_l2)
    d["convergence"] = np.array(D.convergence_table(sol, u_ref, A, lam_a, g_l2))
    import scipy.sparse as sp
    named = [(f"SBS{k}", sp.csr_array(res.levels[k].subband.multiply(
        np.outer(res.levels[k].subband_scale, res.levels[k].subband_scale))))
        for k in (q, q - 1)]
    for k, (_, m) in zip((q, q - 1), named):
        d[f"SBS{k}/indptr"] = m.indptr
        d[f"SBS{k}/indices"] = m.indices
        d[f"SBS{k}/data"] = m.data
        d[f"SBS{k}/shape"] = np.array(m.shape, np.int64)
    d["conditioning"] = np.array([r[1:] for r in D.conditioning_table(named)], float)
    np.savez_compressed(OUT / "diag_q5_checker.npz", **d)
    print("wrote diag_q5_checker")


if __name__ == "__main__":
    main()
