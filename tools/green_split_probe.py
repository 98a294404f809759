"""How the dual-vector SpMV pass and the setup kernels scale with an SM
partition (CUDA green contexts): the inputs of the overlap model."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from cuda.bindings import driver as cu
from paper_1503_03467_b200 import _native as nat, device as dv

def chk(r):
    err, *rest = r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"driver error {err}")
    return rest[0] if len(rest) == 1 else rest

torch.zeros(1, device="cuda"); dv.device()
dev = chk(cu.cuDeviceGet(0))
res = chk(cu.cuDeviceGetDevResource(dev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))

def split(n_sm):
    err, groups, nb, rem = cu.cuDevSmResourceSplitByCount(1, res, 0, n_sm)
    out = []
    for r in (groups[0], rem):
        desc = chk(cu.cuDevResourceGenerateDesc([r], 1))
        g = chk(cu.cuGreenCtxCreate(desc, dev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        st = chk(cu.cuGreenCtxStreamCreate(g, cu.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
        out.append((torch.cuda.ExternalStream(int(st)), r.sm.smCount))
    return out

L, w = 512, 4
R = L * L * 3; S = (2 * w + 1) ** 2 * 3
g = torch.Generator(device="cuda").manual_seed(0)
B = torch.rand(R * S, dtype=torch.float64, device="cuda", generator=g)
s = torch.rand(R, dtype=torch.float64, device="cuda", generator=g) + 0.5
U = dv.empty(nat.query("gb_boxsym_elems", L, w))
nat.call("gb_scale_box_symT", L, w, dv.ptr(B), dv.ptr(s), dv.ptr(U), dv.stream())
del B
npad = (L + 2 * w) ** 2 * 3; tail = nat.query("gb_sym_overflow_elems", L, w)
xs = [torch.rand(npad, dtype=torch.float64, device="cuda", generator=g) for _ in range(2)]
ys = [dv.zeros(npad + tail) for _ in range(2)]
nb = nat.query("gb_kstate_bytes")
sts = [dv.empty(nb, torch.uint8) for _ in range(2)]
parts = [dv.empty(3 * nat.query("gb_red_blocks")) for _ in range(2)]
for t in sts:
    nat.call("gb_state_reset", dv.ptr(t), 0, dv.stream())
red = dv.zeros(2)
torch.cuda.synchronize()

def dual(es, nv, reps=40):
    def run():
        nat.call("gb_dist_apply", L, w, dv.ptr(U), nv, dv.ptr(xs[0]), dv.ptr(ys[0]), dv.ptr(sts[0]),
                 dv.ptr(parts[0]), dv.ptr(xs[1]) if nv == 2 else None, dv.ptr(ys[1]) if nv == 2 else None,
                 dv.ptr(sts[1]) if nv == 2 else None, dv.ptr(parts[1]) if nv == 2 else None,
                 dv.ptr(red), 0, L, es.cuda_stream)
    with torch.cuda.stream(es):
        for _ in range(3): run()
        es.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(es)
        for _ in range(reps): run()
        b.record(es); es.synchronize()
    return a.elapsed_time(b) / reps * 1e3

print("full device: nv=1 %.1f us, nv=2 %.1f us" % (dual(torch.cuda.current_stream(), 1), dual(torch.cuda.current_stream(), 2)))
for n in (32, 48, 64, 96):
    (ek, ck), (et, ct) = split(n)
    print(f"{ck} SMs: nv=1 {dual(ek, 1):.1f} us, nv=2 {dual(ek, 2):.1f} us")
