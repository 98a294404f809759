"""Device memory per level of one fast_solve (allocated after each level step,
peak so far), to plan q=12 on one GPU."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO

q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
lean = len(sys.argv) > 2 and sys.argv[2] == "lean"
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
G = 2 ** 30
orig = gf.local_level_step


def wrapped(level, *a, **kw):
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    out = orig(level, *a, **kw)
    torch.cuda.synchronize()
    print(f"level {level.k}: before {before / G:6.1f} GiB, peak in step "
          f"{torch.cuda.max_memory_allocated() / G:6.1f}, after {torch.cuda.memory_allocated() / G:6.1f}",
          flush=True)
    return out


gf.local_level_step = wrapped
from contextlib import contextmanager
_orig_phase = dv.phase


@contextmanager
def phase_log(label):
    with _orig_phase(label):
        yield
    if torch.cuda.current_stream() == torch.cuda.default_stream():
        print(f"    {label:20s} allocated {torch.cuda.memory_allocated() / G:6.1f} GiB", flush=True)


dv.phase = phase_log
torch.cuda.reset_peak_memory_stats()
import time
t0 = time.perf_counter()
levels, parts, U1, counter = gf._fast_solve_device(Md, Ad, gd, tree, sched, lean=lean)
torch.cuda.synchronize()
print(f"end: allocated {torch.cuda.memory_allocated() / G:.1f} GiB, step {time.perf_counter() - t0:.2f} s")
tot = 0
for k, lv in sorted(levels.items()):
    psi = lv.raw("psi")
    nb = psi.vals.numel() * 8 if psi is not None and hasattr(psi, "vals") else 0
    tot += nb
    print(f"  psi^({k}) {nb / G:6.2f} GiB")
print(f"  psi total {tot / G:.1f} GiB")
