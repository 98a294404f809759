"""Which phase of a slow q=10 step is slow: per-phase CUDA-event spans of every
step, printed for the steps above 1.15x the median."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
grid, M, A, load, tree = build_inputs(10, "checker")
sched = gb.make_schedule(EPS, 10, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
for _ in range(3):
    out = gf._fast_solve_device(Md, Ad, gd, tree, sched); out = None
dv.reserve(1.5 * torch.cuda.max_memory_allocated())
steps = []
for i in range(30):
    torch.cuda.synchronize()
    dv.Prof.reset(enabled=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = gf._fast_solve_device(Md, Ad, gd, tree, sched)
    e1.record(); torch.cuda.synchronize(); out = None
    ph = [(lbl, e0.elapsed_time(a), a.elapsed_time(b)) for lbl, a, b in dv.Prof.events]
    steps.append((e0.elapsed_time(e1), ph))
dv.Prof.reset(enabled=False)
tot = np.array([s[0] for s in steps])
med = np.median(tot)
print("median step", round(float(med), 1), "slow steps:", [round(float(t), 1) for t in tot if t > 1.15 * med])
base = {}
for t, ph in steps:
    if t <= 1.05 * med:
        for j, (lbl, st, du) in enumerate(ph):
            base.setdefault(j, []).append(du)
for t, ph in steps:
    if t > 1.15 * med:
        print(f"--- slow step {t:.1f} ms")
        for j, (lbl, st, du) in enumerate(ph):
            b = float(np.median(base.get(j, [du])))
            if du > b + 15:
                print(f"   phase #{j} {lbl:20s} start {st:7.1f}  took {du:7.1f} ms (typ. {b:.1f})")
