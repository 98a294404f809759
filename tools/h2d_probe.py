"""Host->device upload rates for the API's pageable inputs (e2e leg)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1503_03467_b200 import _native as nat, device as dv

x = np.random.default_rng(0).standard_normal(75 * 2 ** 20 // 8)
t = torch.from_numpy(x)
def timed(name, fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:28s} {np.median(ts):8.2f} ms  {x.nbytes / np.median(ts) / 1e6:6.1f} GB/s", flush=True)
timed("np.copy", lambda: x.copy())
timed("pageable .to(cuda)", lambda: t.to("cuda"))
pin = torch.empty_like(t).pin_memory()
timed("pinned .to(cuda)", lambda: pin.to("cuda", non_blocking=True))
timed("copy into pinned (1 thr)", lambda: pin.copy_(t))
out = torch.empty(t.shape, dtype=t.dtype, device="cuda")
for th in (1, 2, 4, 8, 16):
    timed(f"gb_h2d_staged {th} thr", lambda: nat.call("gb_h2d_staged", out.data_ptr(), t.data_ptr(),
                                                       x.nbytes, th, dv.stream()))
import os
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
from bench import build_inputs
grid, M, A, load, tree = build_inputs(10, "checker")
print("dtypes", M.indptr.dtype, M.indices.dtype, M.data.dtype, M.data.flags["C_CONTIGUOUS"])
timed("from_scipy(M)", lambda: dv.DeviceCSR.from_scipy(M))
timed("to_dev(M.data)", lambda: dv.to_dev(M.data))
timed("to_dev(M.indices)", lambda: dv.to_dev(M.indices))
timed("to_dev(M.indptr)", lambda: dv.to_dev(M.indptr))
timed("astype idx", lambda: M.indices.astype(np.int32, copy=False))
