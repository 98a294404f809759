"""psi^(k-1): tensor-core block GEMM vs the gather kernel (reference summation
order) -- values and row-drop patterns per level, plus timing."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import _native as nat
from oracle import gamblets_oracle as O
from conftest import build_problem

for q, coeff in [(int(a.split(":")[0]), a.split(":")[1]) for a in (sys.argv[1:] or ["6:checker", "8:checker"])]:
    p = build_problem(q, coeff)
    sched = gb.make_schedule(1e-13, q, uniform_rho=3)
    out = {}
    for mode in (0, 1):
        nat.load().gb_products_mode(mode)
        gb.fast_transform(p.M, p.A, p.tree, sched)  # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        lv, _ = gb.fast_transform(p.M, p.A, p.tree, sched)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        out[mode] = {(k, f): getattr(lv[k], f) for k in range(1, q + 1)
                     for f in ("psi", "stiffness", "subband", "correction")
                     if getattr(lv[k], f, None) is not None}
        print(f"q={q} {coeff} mode={mode} transform {dt * 1e3:.1f} ms", flush=True)
    for k in sorted(out[0]):
        a, b = out[0][k], out[1][k]
        print(f"  {k}: nnz {a.nnz} vs {b.nnz} same_pattern={O.same_pattern(a, b)} "
              f"rel={O.rel_fro(b, a):.2e}", flush=True)
