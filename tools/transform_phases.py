"""Per-phase CUDA-event times of the transform alone (no Krylov side streams:
gamblet_fast.SPECTRAL off, no load), for A/B tests of the setup kernels."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO

q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gf.SPECTRAL = False
for _ in range(2):
    levels, _ = gb.fast_transform(Md, Ad, tree, sched)
    levels = None
torch.cuda.synchronize()
dv.Prof.reset(enabled=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    levels, _ = gb.fast_transform(Md, Ad, tree, sched)
    levels = None
b.record()
torch.cuda.synchronize()
print(f"transform alone: {a.elapsed_time(b) / reps:.2f} ms per q={q} transform")
for k, v in sorted(dv.Prof.times_ms().items(), key=lambda x: -x[1]):
    print(f"  {k:22s} {v / reps:8.3f} ms")
