"""Where the host sits during an outlier step: wall-clock spans of every
device->host read (device.to_host) and of the step, over many steps."""
import sys, time, traceback
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
q = int(sys.argv[1]) if len(sys.argv) > 1 else 7
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
log = []
orig = dv.to_host


def timed_to_host(t):
    t0 = time.perf_counter()
    out = orig(t)
    dt = time.perf_counter() - t0
    if dt > 0.03:
        fr = traceback.extract_stack(limit=3)[0]
        log.append((dt * 1e3, f"{Path(fr.filename).name}:{fr.lineno}"))
    return out


dv.to_host = timed_to_host
for _ in range(5):
    out = gf._fast_solve_device(Md, Ad, gd, tree, sched); out = None
dv.reserve(1.5 * torch.cuda.max_memory_allocated())
torch.cuda.synchronize()
walls = []
for i in range(steps):
    n0 = len(log)
    t0 = time.perf_counter()
    out = gf._fast_solve_device(Md, Ad, gd, tree, sched)
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) * 1e3
    out = None
    walls.append(w)
    if len(log) > n0:
        print(f"step {i}: wall {w:.1f} ms; slow reads: {log[n0:]}", flush=True)
walls = np.array(walls)
med = np.median(walls)
print("median", round(float(med), 2), "outliers(>1.5x):", [(int(i), round(float(w), 1)) for i, w in enumerate(walls) if w > 1.5 * med])
