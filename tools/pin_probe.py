import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from bench import build_inputs
grid, M, A, load, tree = build_inputs(10, "checker")
dev = torch.device('cuda', 0)
torch.zeros(1, device=dev)
cr = torch.cuda.cudart()
def up_plain(a):
    return torch.from_numpy(a).to(dev)
def up_reg(a):
    t = torch.from_numpy(a)
    ptr, nb = a.ctypes.data, a.nbytes
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(ptr, nb, 0)
    t1 = time.perf_counter()
    out = torch.empty(a.shape, dtype=t.dtype, device=dev)
    out.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(ptr)
    t3 = time.perf_counter()
    return out, (t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, int(r)
for rep in range(3):
    torch.cuda.synchronize(); t0=time.perf_counter()
    for a in (M.data, M.indices, M.indptr): up_plain(a)
    torch.cuda.synchronize(); print('plain', (time.perf_counter()-t0)*1e3)
    torch.cuda.synchronize(); t0=time.perf_counter()
    for a in (M.data, M.indices, M.indptr): print('  reg', up_reg(a)[1:])
    print('registered total', (time.perf_counter()-t0)*1e3)
