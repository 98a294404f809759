"""Per-step device time of the device-resident step + allocator activity."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO

import os
import subprocess
q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
smi = None
if os.environ.get("SV_SMI"):
    smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm", "--format=csv",
                            "-lms", os.environ["SV_SMI"]], stdout=subprocess.DEVNULL)
if os.environ.get("SV_PROF"):
    dv.Prof.reset(enabled=True)
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
for i in range(n):
    if i == 1:
        dv.reserve(1.25 * torch.cuda.max_memory_allocated())
    s0 = torch.cuda.memory_stats()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record()
    gf._fast_solve_device(Md, Ad, gd, tree, sched)
    b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3
    s1 = torch.cuda.memory_stats()
    print(f"step {i}: {a.elapsed_time(b):.1f} ms (wall {wall:.1f}) "
          f"device_allocs +{s1['num_device_alloc'] - s0['num_device_alloc']} "
          f"frees +{s1['num_device_free'] - s0['num_device_free']} "
          f"retries +{s1['num_alloc_retries'] - s0['num_alloc_retries']} "
          f"peak {s1['allocated_bytes.all.peak'] / 2**30:.1f} GiB "
          f"reserved {s1['reserved_bytes.all.current'] / 2**30:.1f} GiB", flush=True)
if smi is not None:
    smi.terminate()
