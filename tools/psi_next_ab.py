"""A/B of two builds of the library on the q-level transform: phase times and a
bitwise comparison of every psi^(k) (GB_LIB selects the build per process)."""
import sys, hashlib
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gf.SPECTRAL = False
levels, _ = gb.fast_transform(Md, Ad, tree, sched)
torch.cuda.synchronize()
hh = hashlib.sha256()
for k in sorted(levels):
    hh.update(levels[k].raw("psi").vals.cpu().numpy().tobytes())
    hh.update(levels[k].raw("stiffness").vals.cpu().numpy().tobytes())
print("digest of every psi^(k), A^(k):", hh.hexdigest()[:24])
levels = None
dv.Prof.reset(enabled=True)
for _ in range(3):
    levels, _ = gb.fast_transform(Md, Ad, tree, sched); levels = None
torch.cuda.synchronize()
t = dv.Prof.times_ms()
print({k: round(v / 3, 2) for k, v in sorted(t.items(), key=lambda x: -x[1])[:4]})
