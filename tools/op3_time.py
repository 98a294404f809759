"""3-D level operator: time the separate CG / lambda solves against the paired engine."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1503_03467_b200 import device as dv, gamblet_3d as g3
from paper_1503_03467_b200.gamblet_fast import make_schedule
from bench import build_inputs_3d

q = int(sys.argv[1]) if len(sys.argv) > 1 else 5
grid, M, A, g = build_inputs_3d(q)
sched = make_schedule(1e-13, q, uniform_rho=2)
levels, ops = g3.fast_transform_3d(M, A, q, sched.radii)
op = ops[q]
print("level", q, "rows", op.n, "w", op.w, "matrix GB", op.n * (2 * op.w + 1) ** 3 * op.nr * 8 / 1e9)
rhs = dv.to_dev(np.random.default_rng(5).standard_normal(op.n))
tol = sched.subband_tol()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, out
for _ in range(2):
    a, r1 = t(lambda: op.cg(rhs, tol))
    b, r2 = t(lambda: op.eig_extremes(tol=0.1))
    c = 0.0
    print(f"cg {a:.1f} ms ({r1[1]} its)  eig {b:.1f} ms ({op.spectral_passes} passes)")
x = dv.to_dev(np.random.default_rng(6).standard_normal(op.n)); y = dv.empty(op.n)
d, _ = t(lambda: [op.apply(x, y) for _ in range(50)])
print(f"single sweep {d / 50 * 1e3:.1f} us")
