"""The finest level's engine (PCG + power + Lanczos) timed alone on the GPU:
time per operator pass including the vector updates between passes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
levels, counter = gf.fast_transform(M, A, tree, sched)
lv = levels[q]
op = lv._op
rng = np.random.default_rng(3)
rhs = op.pad(dv.to_dev(rng.standard_normal(op.n)))
tol = sched.subband_tol()
for rep in range(3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gf.ENGINE_TIMING = {"n": op.n, "cap": 512, "ms": []}
    a.record()
    out = gf._paired_level(op, rhs, tol)
    b.record()
    torch.cuda.synchronize()
    t = gf.ENGINE_TIMING["ms"]
    gf.ENGINE_TIMING = None
    nd, ns = out["passes"]
    print(f"engine alone: {a.elapsed_time(b):.1f} ms, PCG its {out['its']}, passes dual {nd} "
          f"single {ns} -> {a.elapsed_time(b) / (nd + ns) * 1e3:.1f} us per pass incl. updates; "
          f"dual pass kernel {np.mean(t) * 1e3:.1f} us (n={len(t)})")
