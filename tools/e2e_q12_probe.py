"""Where does the config-3 (q=12, lean) e2e step spend time beyond the device step?"""
import os, sys, time
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
os.environ.setdefault("GB_SPECTRAL_WORKERS", "3")
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
Q = int(sys.argv[1]) if len(sys.argv) > 1 else 12
grid, M, A, load, tree = build_inputs(Q, "checker")
sched = gb.make_schedule(EPS, Q, uniform_rho=RHO)
Md, Ad, gd = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A), dv.to_dev(load.g_nodal)
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = gf._fast_solve_device(Md, Ad, gd, tree, sched, lean=True)
    torch.cuda.synchronize(); print(f"device step {(time.perf_counter() - t0) * 1e3:9.1f} ms", flush=True)
    out = None
del Md, Ad, gd
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO, c_tol=1e-6, lean=True)
    torch.cuda.synchronize(); print(f"e2e step    {(time.perf_counter() - t0) * 1e3:9.1f} ms", flush=True)
    print({k: round(v * 1e3, 1) for k, v in res.counter.seconds.items()}, flush=True)
    res = None
print("max mem GiB", torch.cuda.max_memory_allocated() / 2**30)
