"""lambda estimates of S B S per level: reference inner CG vs block-Jacobi PCG
vs the Lanczos-moment evaluation (level engine spectral mode 1)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import gamblet_fast as gf
from bench import build_inputs, EPS, RHO

q = int(sys.argv[1]) if len(sys.argv) > 1 else 8
grid, M, A, load, tree = build_inputs(q, "checker")
out = {}
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["cg", "lanczos"]
for inner in modes + modes:
    gf.SPECTRAL_INNER = inner
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    out[inner] = {k: (res.levels[k].lambda_min_subband, res.levels[k].lambda_max_subband)
                  for k in range(2, q + 1)}
    print(f"{inner}: {dt * 1e3:.1f} ms", flush=True)
for k in range(2, q + 1):
    a, b = out[modes[0]][k], out[modes[1]][k]
    print(k, a, b, abs(b[0] - a[0]) / abs(a[0]), abs(b[1] - a[1]) / abs(a[1]))
