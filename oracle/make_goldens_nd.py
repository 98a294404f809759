"""Generate tests/golden/fast3d_*.npz from the dimension-generic oracle.

TEST INFRASTRUCTURE ONLY.  The reference package has no 3-D path (SURVEY.md
8(c)), so these fixtures come from oracle/gamblets_oracle_nd.py, whose d=2
instance is pinned to the reference (tests/test_oracle_nd.py).  They pin the
3-D restatement against regressions and are the parity target of the 3-D GPU
path (BASELINE config 4 family: example coefficient, Gaussian nodal load
seed 1, rho = 2, tight mode epsilon = 1e-13).

    python oracle/make_goldens_nd.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import gamblets_oracle_nd as ND  # noqa: E402
from oracle.make_goldens import digest, put_csr  # noqa: E402

OUT = ROOT / "tests" / "golden"


def make(q, rho=2, d=3):
    grid, M, A, g, b = ND.build_problem(q, d, "example")
    sol, lv, radii = ND.fast_solve(M, A, g, q, d, 1e-13, uniform_rho=rho)
    out = {"q": q, "d": d, "rho": rho, "radii": np.array(radii),
           "digest_M": digest(M), "digest_A": digest(A), "g": g, "u": sol["u"]}
    for k in range(q, 0, -1):
        put_csr(out, f"A{k}", lv[k]["stiffness"])
        put_csr(out, f"psi{k}", lv[k]["psi"])
        if k >= 2:
            put_csr(out, f"B{k}", lv[k]["subband"])
            put_csr(out, f"R{k}", lv[k]["restriction"])
            put_csr(out, f"D{k}", lv[k]["correction"])
            out[f"s{k}"] = lv[k]["subband_scale"]
            out[f"lam{k}"] = np.array([lv[k]["lambda_min"], lv[k]["lambda_max"]])
            out[f"w{k}"] = sol["coeffs"][k]
    name = f"fast3d_q{q}_example"
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print("wrote", OUT / f"{name}.npz")


if __name__ == "__main__":
    make(3)
