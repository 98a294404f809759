import sys, cProfile, pstats
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
grid, M, A, load, tree = build_inputs(7, "example1")
sched = gb.make_schedule(EPS, 7, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
for _ in range(5):
    gf._fast_solve_device(Md, Ad, gd, tree, sched)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    gf._fast_solve_device(Md, Ad, gd, tree, sched)
    torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
