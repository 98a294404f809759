"""Step-time noise of the q=10 device-resident solve, with the caching
allocator's counters per step (segments allocated / freed, alloc retries)."""
import sys, gc, json, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import os
if os.environ.get("GB_SPIN"):
    # cudaDeviceScheduleSpin before the context exists: stream / event waits
    # poll instead of blocking on an interrupt
    import ctypes, glob
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
        glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*") + \
        ["/usr/local/cuda/lib64/libcudart.so"]
    rt = ctypes.CDLL(cands[0])
    print("cudart:", cands[0])
    rc = rt.cudaSetDeviceFlags(int(os.environ["GB_SPIN"]))
    print("cudaSetDeviceFlags ->", rc)
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
grid, M, A, load, tree = build_inputs(10, "checker")
sched = gb.make_schedule(EPS, 10, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
def stats():
    s = torch.cuda.memory_stats()
    return (s.get("segment.all.allocated", 0), s.get("segment.all.freed", 0), s.get("num_alloc_retries", 0),
            s.get("reserved_bytes.all.current", 0) >> 20)
def run(n, tag):
    rows = []
    for i in range(n):
        torch.cuda.synchronize()
        s0 = stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        out = gf._fast_solve_device(Md, Ad, gd, tree, sched)
        t_enq = (time.perf_counter() - t0) * 1e3
        e1.record(); torch.cuda.synchronize(); out = None
        s1 = stats()
        rows.append((round(e0.elapsed_time(e1), 1), round(t_enq, 1), s1[0] - s0[0], s1[1] - s0[1], s1[2] - s0[2], s1[3]))
    print(tag, "median", np.median([r[0] for r in rows]))
    for r in rows:
        if r[0] > 270 or r[2] or r[3] or r[4]:
            print("   step ms %.1f, host-return ms %.1f, segments +%d -%d, retries %d, reserved MiB %d" % r)
import os
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "loadavg", os.getloadavg())
if len(sys.argv) > 1:
    gf.SPECTRAL_WORKERS = int(sys.argv[1])
run(3, "warm")
dv.reserve(1.5 * torch.cuda.max_memory_allocated())
run(2, "after reserve")
run(40, "timed")
print("loadavg", os.getloadavg())
