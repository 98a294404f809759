"""Small-size check of the patch kernels against dense numpy solves."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import gamblet_fast as gf
from oracle import gamblets_oracle as O
from conftest import build_problem
for q, rho in ((2, 4), (3, 1), (3, 3), (4, 3)):
    p = build_problem(q, "example1")
    psi = gf.local_mass_inverse(p.M, p.tree, rho=rho, tol=1e-12)
    ref = O.mass_inverse(p.M, q, rho)
    print("mass", q, rho, O.rel_fro(psi, ref), O.same_pattern(psi, ref), flush=True)
gf.SPECTRAL = False
for q, coeff in ((4, "example1"), (5, "checker")):
    p = build_problem(q, coeff)
    sched = gb.make_schedule(1e-13, q, uniform_rho=3)
    lv = O.fast_transform(p.M, p.A, q, sched.radii, spectral=False, with_psi=False)
    lvl = gb.LocalGambletLevel(q, None, lv[q]["stiffness"])
    nxt = gf.local_level_step(lvl, p.tree, sched)
    print("corr", q, coeff, O.rel_fro(lvl.correction, lv[q]["correction"]),
          O.rel_fro(nxt.stiffness, lv[q - 1]["stiffness"]), flush=True)
