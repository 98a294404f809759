"""Per-step device time of the lean q=12 step (config 3), synchronized steps."""
import sys, time, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
q = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
del M, A
for i in range(n):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = gf._fast_solve_device(Md, Ad, gd, tree, sched, lean=True)
    b.record()
    torch.cuda.synchronize()
    out = None
    print(f"step {i}: {a.elapsed_time(b):.0f} ms, reserved {torch.cuda.memory_reserved() / 2**30:.0f} GiB",
          flush=True)
