"""Standalone timing of the symmetric band SpMV on a synthetic level-10-sized
operator (L=512, w=4; random symmetric box built on the device), no solver --
for A/B tests of kernel variants (GB_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1503_03467_b200 import _native as nat, device as dv

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = 20
R = L * L * 3
S = (2 * w + 1) ** 2 * 3
g = torch.Generator(device="cuda").manual_seed(0)
B = torch.rand(R * S, dtype=torch.float64, device="cuda", generator=g)  # values only matter
s = torch.rand(R, dtype=torch.float64, device="cuda", generator=g) + 0.5
st = dv.stream()
U = dv.empty(nat.query("gb_boxsym_elems", L, w))
nat.call("gb_scale_box_symT", L, w, dv.ptr(B), dv.ptr(s), dv.ptr(U), st)
del B
npad = (L + 2 * w) ** 2 * 3
tail = nat.query("gb_sym_overflow_elems", L, w)
x = torch.rand(npad, dtype=torch.float64, device="cuda", generator=g)
y = dv.zeros(npad + tail)
for _ in range(3):
    nat.call("gb_tbox_apply", L, 3, w, dv.ptr(U), dv.ptr(x), dv.ptr(y), st, 1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    nat.call("gb_tbox_apply", L, 3, w, dv.ptr(U), dv.ptr(x), dv.ptr(y), st, 1)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
mat = U.numel() * 8
print(f"L={L} w={w}: {ms * 1e3:.1f} us per apply (phase 1 + 2), matrix {mat / 1e9:.3f} GB "
      f"-> {mat / ms / 1e6:.0f} GB/s")
