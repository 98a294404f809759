"""Time the partitioned program on ONE rank (a single strip, no exchange)
against the single-GPU pipeline: the cost of its Python-driven, non-overlapped
Krylov loop."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_dist as gd, gamblet_fast as gf
from bench import EPS, RHO

q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
grid = gb.build_grid(q)
tree = gb.build_hierarchy(grid)
c = gb.coefficient_checkerboard(grid, 1e4, 0)
g = np.random.default_rng(1).standard_normal(grid.num_nodes)
Mb = gb.assemble_mass(grid, device=True)
Ab = gb.assemble_stiffness(grid, c, device=True)
gdv = dv.to_dev(g)
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
for name, fn in (("single-GPU pipeline", lambda: gf._fast_solve_device(Mb, Ab, gdv, tree, sched)),
                 ("strip program, 1 rank", lambda: gd.fast_solve_dist(
                     gb.SelfComm(), Mb, Ab, gdv, tree, EPS, uniform_rho=RHO, force_strips=True))):
    ts = []
    for i in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        out = None
    print(f"{name}: {np.median(ts[2:]):.1f} ms per q={q} solve  {['%.0f' % t for t in ts]}")
