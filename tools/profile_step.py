"""One device-resident fast_solve step (for ncu captures)."""
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
ap.add_argument("--coeff", default="checker")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--profile-last", action="store_true",
                help="bracket only the last step with cudaProfilerStart/Stop "
                     "(use with ncu --profile-from-start off)")
a = ap.parse_args()
grid, M, A, load, tree = build_inputs(a.q, a.coeff)
sched = gb.make_schedule(EPS, a.q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
for i in range(a.steps):
    last = i == a.steps - 1
    if last and a.profile_last:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    gf._fast_solve_device(Md, Ad, gd, tree, sched)
    if last and a.profile_last:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
torch.cuda.synchronize()
print("ok")
