"""Convergence of the emulated inverse-iteration lambda_min with the number of
Lanczos steps, per level of a q-level instance: runs the engine to a long
fixed length and evaluates the estimate on every leading T_m."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1503_03467_b200 as gb
from paper_1503_03467_b200 import device as dv, gamblet_fast as gf, _native as nat
from bench import build_inputs, EPS, RHO
q = int(sys.argv[1]) if len(sys.argv) > 1 else 10
medium = sys.argv[2] if len(sys.argv) > 2 else "checker"
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 704
grid, M, A, load, tree = build_inputs(q, medium)
sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
gd = dv.to_dev(load.g_nodal)
gf.LANCZOS_TOL = 0.0
gf.LANCZOS_CAP = cap
gf._LANCZOS_DUMP = []
out = gf._fast_solve_device(Md, Ad, gd, tree, sched)
lib = ctypes.CDLL(str(nat.LIB_PATH))


def emulate(ab, m):
    lam, outer = ctypes.c_double(), ctypes.c_int()
    buf = np.ascontiguousarray(ab[:2 * m])
    rc = lib.gb_lanczos_emulate(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(m),
                                ctypes.c_double(0.1), ctypes.c_int(500), ctypes.byref(lam),
                                ctypes.byref(outer), None, None)
    return rc, lam.value, outer.value


def check(ab, m, lz_tol=1e-4):
    lam, outer, stop = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    buf = np.ascontiguousarray(ab[:2 * m])
    rc = lib.gb_lanczos_check(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(m),
                              ctypes.c_double(0.1), ctypes.c_int(500), ctypes.c_double(lz_tol),
                              ctypes.byref(lam), ctypes.byref(outer), ctypes.byref(stop))
    return rc, lam.value, outer.value, stop.value


for n, ab in sorted(gf._LANCZOS_DUMP, key=lambda t: -t[0]):
    mtot = len(ab) // 2
    rc, lam_f, out_f = emulate(ab, mtot)
    print(f"n={n} steps={mtot} final lam={lam_f:.12e} outer={out_f}")
    for m in [64] + list(range(96, mtot + 1, 32)):  # the engine's check points
        rc, lam, outer, stop = check(ab, m)
        if stop:
            print(f"   engine stops at m={m}: lam/lam_final - 1 = {lam / lam_f - 1.0:+.2e}, outer {outer}")
            break
    else:
        print("   engine does not stop within", mtot)
    row = []
    for m in range(16, mtot + 1, 16):
        rc, lam, outer = emulate(ab, m)
        row.append((m, lam / lam_f - 1.0, outer))
    if "-v" in sys.argv:
        print("   " + "  ".join(f"{m}:{d:+.1e}/{o}" for m, d, o in row))
