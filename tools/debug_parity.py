"""Stage-by-stage GPU vs oracle comparison (development aid)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import scipy.sparse as sp
import torch
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import gamblet_fast as gf, device as dv, _native as nat
from oracle import gamblets_oracle as O
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from conftest import build_problem

q = int(sys.argv[1]) if len(sys.argv) > 1 else 4
coeff = sys.argv[2] if len(sys.argv) > 2 else "example1"
p = build_problem(q, coeff)
gf.SPECTRAL = False
gf.STRICT = False
sched = gb.make_schedule(1e-13, q, uniform_rho=3)
levels, _ = gb.fast_transform(p.M, p.A, p.tree, sched)
lv = O.fast_transform(p.M, p.A, q, sched.radii, spectral=False)
def cmp(name, a, b):
    try:
        e = O.rel_fro(a, b); pat = O.same_pattern(a, b)
        print(f"{name:12s} rel {e:.3e} pattern {'ok' if pat else 'DIFF'} nnz {sp.csr_array(a).nnz} vs {sp.csr_array(b).nnz}")
    except Exception as ex:
        print(name, "ERR", ex)
for k in range(q, 0, -1):
    g, o = levels[k], lv[k]
    cmp(f"A{k}", g.stiffness, o["stiffness"])
    if o.get("psi") is not None: cmp(f"psi{k}", g.psi, o["psi"])
    if k >= 2:
        cmp(f"B{k}", g.subband, o["subband"])
        print("   sB", np.abs(g.subband_scale / o["subband_scale"] - 1).max())
        cmp(f"D{k}", g.correction, o["correction"])
        cmp(f"R{k}", g.restriction, o["restriction"])
# CG on our B^(q)
B = levels[q].raw("subband"); sB = levels[q].raw("subband_scale")
op = gf._POp(B, sB)
n = B.rows
x = np.random.default_rng(0).standard_normal(n)
xp = op.pad(dv.to_dev(x)); yp = op.vec()
op.apply(xp, yp)
_, Bs = O.diag_scale(lv[q]["subband"])
y = op.unpad(yp).cpu().numpy()
print("pbox_apply err", np.abs(y - Bs @ x).max() / np.abs(Bs @ x).max())
z, its, rel, conv, brk, h = gf._cg(op, xp, 1e-10)
print("cg", its, rel, conv, brk, "err", np.abs(Bs @ op.unpad(z).cpu().numpy() - x).max())
print("eig", gf._eig_extremes(op)[:2], O.eig_extremes(Bs))
z, its, rel, conv, brk, h = gf._pcg(op, xp, 1e-10)
print("pcg", its, rel, conv, brk, "err", np.abs(Bs @ op.unpad(z).cpu().numpy() - x).max())
inv = op.bj_inv().cpu().numpy().reshape(-1, 12, 12)
L = B.L
bs, bt = 1, 1
idx = []
for i in range(2):
    for j in range(2):
        p_ = (2*bs+i)*L + 2*bt+j
        idx += [3*p_, 3*p_+1, 3*p_+2]
blk = Bs[idx][:, idx].toarray()
print("bj inv err", np.abs(inv[bs*(L//2)+bt] @ blk - np.eye(12)).max())
