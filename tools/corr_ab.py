"""A/B harness of the 2-D correction-patch kernel: the finest level of a
q-level instance, launched alone on the level's own B and a seeded G; prints
the time per launch and a digest of D^T (load a variant with GB_LIB=...)."""
import hashlib, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import _native as nat, device as dv, gamblet_fast as gf
from bench import build_inputs, EPS, RHO
q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
grid, M, A, load, tree = build_inputs(q, "checker")
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
gf.SPECTRAL = False
levels = gf.fast_transform(M, A, tree, sched)[0]
for k in (q, q - 2):
    lv = levels[k]
    B = lv.raw("subband")
    rho = min(3, B.L - 1)
    s = dv.stream()
    Dt = dv.empty(B.L * B.L * dv.box_slots(rho, 3))
    st = dv.zeros(2, torch.int64)
    rng = np.random.default_rng(5)
    G = dv.to_dev(rng.standard_normal(B.rows * dv.box_slots(B.w, 1)))
    ws, nb = gf._correction_ws(B.L, rho, 0, B.L)
    args = (B.L, B.w, dv.ptr(B.vals), dv.ptr(lv.raw("subband_scale")), B.w, dv.ptr(G), rho,
            dv.ptr(Dt), dv.ptr(st), dv.ptr(ws), nb, s)
    nat.call("gb_correction_patches_v2", *args)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nat.call("gb_correction_patches_v2", *args)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h = hashlib.sha256(Dt.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"level {k}: L={B.L} wB={B.w} min {min(ts):.3f} ms median {sorted(ts)[2]:.3f} ms "
          f"status {st.tolist()} digest {h}")
