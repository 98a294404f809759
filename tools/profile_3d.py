"""Per-phase CUDA-event times of one 3-D fast_solve_3d step (config 4)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1503_03467_b200 import device as dv, gamblet_3d as g3
from bench import build_inputs_3d, EPS, RHO3

ap = argparse.ArgumentParser()
ap.add_argument("--q", type=int, default=6)
ap.add_argument("--tiled", type=int, default=-1, help="gb_tune(6): 3-D product kernels (0 per-entry, 1 tiled)")
a = ap.parse_args()
if a.tiled >= 0:
    from paper_1503_03467_b200 import _native as nat
    nat.load().gb_tune(6, a.tiled)
grid, M, A, g = build_inputs_3d(a.q)
Md, Ad = g3.box3_from_csr(M, 1 << a.q), g3.box3_from_csr(A, 1 << a.q)
gd = dv.to_dev(g)
g3.fast_solve_3d(Md, Ad, gd, a.q, EPS, uniform_rho=RHO3)
torch.cuda.synchronize()
dv.Prof.reset(enabled=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = g3.fast_solve_3d(Md, Ad, gd, a.q, EPS, uniform_rho=RHO3)
e1.record()
torch.cuda.synchronize()
ph = dv.Prof.times_ms()
import hashlib
import numpy as np
digest = hashlib.sha256(np.ascontiguousarray(np.asarray(res.solution.u)).tobytes()).hexdigest()[:16]
print(json.dumps({"u_digest": digest, "q": a.q, "step_ms": round(e0.elapsed_time(e1), 2),
                  "phases_ms": {k: round(v, 2) for k, v in sorted(ph.items(), key=lambda x: -x[1])},
                  "iterations": {str(k): v for k, v in res.iterations.items()},
                  "peak_gib": round(torch.cuda.max_memory_allocated() / 2**30, 2)}))
