"""Standalone timing of phase 1 of the symmetric band SpMV for one and two
vectors (k_symb_apply_ws<1|2>) on a level-10-sized operator (L=512, w=4),
through gb_dist_apply over the whole level (raw reductions, no solver)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1503_03467_b200 import _native as nat, device as dv

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
R = L * L * 3
S = (2 * w + 1) ** 2 * 3
g = torch.Generator(device="cuda").manual_seed(0)
B = torch.rand(R * S, dtype=torch.float64, device="cuda", generator=g)
s = torch.rand(R, dtype=torch.float64, device="cuda", generator=g) + 0.5
st = dv.stream()
U = dv.empty(nat.query("gb_boxsym_elems", L, w))
nat.call("gb_scale_box_symT", L, w, dv.ptr(B), dv.ptr(s), dv.ptr(U), st)
del B
npad = (L + 2 * w) ** 2 * 3
tail = nat.query("gb_sym_overflow_elems", L, w)
xs = [torch.rand(npad, dtype=torch.float64, device="cuda", generator=g) for _ in range(2)]
ys = [dv.zeros(npad + tail) for _ in range(2)]
nb = nat.query("gb_kstate_bytes")
sts = [dv.empty(nb, torch.uint8) for _ in range(2)]
parts = [dv.empty(3 * nat.query("gb_red_blocks")) for _ in range(2)]
for t in sts:
    nat.call("gb_state_reset", dv.ptr(t), 0, st)
red = dv.zeros(2)
mat = U.numel() * 8


def run(nv):
    nat.call("gb_dist_apply", L, w, dv.ptr(U), nv, dv.ptr(xs[0]), dv.ptr(ys[0]), dv.ptr(sts[0]),
             dv.ptr(parts[0]), dv.ptr(xs[1]) if nv == 2 else None,
             dv.ptr(ys[1]) if nv == 2 else None, dv.ptr(sts[1]) if nv == 2 else None,
             dv.ptr(parts[1]) if nv == 2 else None, dv.ptr(red), 0, L, st)


for nv in (1, 2):
    for _ in range(3):
        run(nv)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run(nv)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    nbytes = mat + nv * 2 * 8 * npad
    print(f"nv={nv} L={L} w={w}: {ms * 1e3:.1f} us per pass, {nbytes / 1e9:.3f} GB -> "
          f"{nbytes / ms / 1e6:.0f} GB/s")
