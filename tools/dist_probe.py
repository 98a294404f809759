"""Run the partitioned solve on in-process ranks and compare with one GPU."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_dist as T
from paper_1503_03467_b200 import comm as cm, device as dv

q, world = int(sys.argv[1]), int(sys.argv[2])
grid, M, A, g, tree = T._inputs(q)
levels, u_ref, counter = T._single(M, A, g, tree)
t0 = time.time()
out = cm.run_threads(world, T._rank_body, M, A, g, tree, device=dv.device())
torch.cuda.synchronize()
print("dist run", time.time() - t0, "s; first replicated", out[0].first_replicated)
print("rel err u", float((out[0].u - u_ref).norm() / u_ref.norm()))
print("iterations", out[0].iterations, counter.iterations["line8"])
print("lambdas", {k: out[0].lambdas[k] for k in out[0].lambdas})
print("ref lam", {k: (levels[k].lambda_min_subband, levels[k].lambda_max_subband) for k in levels if k >= 2})
print("halo bytes", [o.halo_bytes for o in out], "passes", out[0].krylov_passes)
