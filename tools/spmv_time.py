"""Isolated timing of the finest-level S B S application (the Krylov SpMV)
after one q=10 fast_solve: CUDA events over `reps` back-to-back applications
on the launching stream.  --profile brackets 3 applications with
cudaProfilerStart/Stop for `ncu --profile-from-start off`."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import argparse
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO

ap = argparse.ArgumentParser()
ap.add_argument("--q", type=int, default=10)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
grid, M, A, load, tree = build_inputs(a.q, "checker")
sched = gb.make_schedule(EPS, a.q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
levels, parts, U1, counter = gf._fast_solve_device(Md, Ad, gd, tree, sched)
torch.cuda.synchronize()
op = levels[a.q]._op
x, y = op.vec(), op.vec()
x.normal_()
for _ in range(3):
    op.apply(x, y)
torch.cuda.synchronize()
if a.profile:
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(3):
        op.apply(x, y)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    op.apply(x, y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
mat = 8 * op.n * op.stored_slots
print(f"L={op.L} w={op.w} layout={op.layout}: {ms * 1e3:.1f} us per apply, "
      f"matrix {mat / 1e9:.3f} GB -> {mat / ms / 1e6:.0f} GB/s")
