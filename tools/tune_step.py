"""Step-time sweep of the concurrency knobs of the q-level pipeline: Krylov
worker threads (level engines / small-level solves running beside the setup)
and the CTA cap of the persistent symmetric-band SpMV pass (gb_tune(3)).
Prints one JSON line per setting: median step ms over --steps device-resident
fast_solve steps (CUDA events)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import _native as nat, device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO

ap = argparse.ArgumentParser()
ap.add_argument("--q", type=int, default=10)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--workers", default="2,3,4")
ap.add_argument("--ctas", default="0,96,74")
ap.add_argument("--ws", default="1", help="phase-1 kernel: 1 warp-specialized, 0 register-pipelined")
ap.add_argument("--prio", default="-1", help="stream priority of the level tasks")
ap.add_argument("--mainprio", type=int, default=0, help="run the steps on a side stream of this priority (0: current stream)")
a = ap.parse_args()
grid, M, A, load, tree = build_inputs(a.q, "checker")
sched = gb.make_schedule(EPS, a.q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
lib = nat.load()
main = torch.cuda.Stream(priority=a.mainprio) if a.mainprio else None
if main is not None:
    torch.cuda.set_stream(main)
for ws, prio in ((w_, p_) for w_ in map(int, a.ws.split(",")) for p_ in map(int, a.prio.split(","))):
  lib.gb_tune(5, ws)
  gf.SPECTRAL_PRIORITY = prio
  for w in map(int, a.workers.split(",")):
    gf.SPECTRAL_WORKERS = w
    if gf._LevelTasks._pool is not None:
        gf._LevelTasks._pool.shutdown(wait=True)
        gf._LevelTasks._pool = None
    for c in map(int, a.ctas.split(",")):
        lib.gb_tune(3, c)
        ts = []
        for i in range(a.steps + 2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = gf._fast_solve_device(Md, Ad, gd, tree, sched)
            e1.record()
            torch.cuda.synchronize()
            out = None
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        print(json.dumps({"ws": ws, "prio": prio, "workers": w, "sym_ctas": c,
                          "ms": round(float(np.median(ts)), 2),
                          "all": [round(t, 1) for t in ts]}), flush=True)
