"""Where does the e2e (host-input) step spend time beyond the device step?"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
grid, M, A, load, tree = build_inputs(10, "checker")
sched = gb.make_schedule(EPS, 10, uniform_rho=RHO)
for _ in range(2):
    gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO, c_tol=1e-6)
torch.cuda.synchronize()
for name, fn in [("upload M", lambda: dv.DeviceCSR.from_scipy(M)),
                 ("upload g", lambda: dv.to_dev(load.g_nodal)),
                 ("canon check", lambda: gf._canon(M)),
                 ("fast_solve e2e", lambda: gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO, c_tol=1e-6)),
                 ]:
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:16s} {np.median(ts):9.2f} ms")
Md, Ad, gd = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A), dv.to_dev(load.g_nodal)
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); gf._fast_solve_device(Md, Ad, gd, tree, sched); torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"{'device step':16s} {np.median(ts):9.2f} ms")
res = gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO, c_tol=1e-6)
print({k: round(v*1e3, 1) for k, v in res.counter.seconds.items()})
