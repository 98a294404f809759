"""Spatially partitioned localized gamblet transform and solve (multi-GPU).

SURVEY.md 8(e) / BASELINE north_star: the fine grid is split into `world`
row strips, one per rank (one process per GPU over torch.distributed / NCCL;
`comm.ThreadComm` runs the same program on in-process ranks of one GPU for
the parity tests).  The arithmetic is gamblet_fast's, kernel for kernel: every
level-step kernel has a row-range form that computes the rank's rows of its
output from inputs addressed by global row (csrc `*_rows` entry points), so
the union of the strips is bitwise the single-GPU transform.

Levels k with parent grids of at least max(64, 16 world) rows are
*distributed*: a rank allocates only its rows (plus the halo it reads) of
A^(k), B^(k), G, D^T, R, psi^(k), the Krylov copy of S B S and its
block-Jacobi inverses -- 1/world of every operator -- and exchanges per step

    bdiag, s_B                       halo  w_B rows         (tiny)
    B^(k), G                         halo  rho / max(rho, w_B) rows
    D^T                              halo  w_B + rho rows
    B D, G^T D, raw A^(k-1)          halo  rho, w_B + rho, 2 rho + w_B rows
    W psi^(k)                        halo  rho rows
    min diag, repair statistics      all-reduce (min / max)

(patches are independent given the level operator: gamblet_fast.py:546-580,
464-498).  The subband systems of those levels are solved by a
distributed block-Jacobi PCG that shares every pass over the strip's rows of
S B S with the lambda estimates (power iteration, then the Lanczos moments of
the inverse iteration, as gb_level_engine does on one GPU): per iteration the
w rows of the operator inputs below the strip and the spill-over tiles of the
rows above it go to the neighbour, and two small all-reduces carry the CG /
Lanczos scalars (csrc/gb_dist.cuh).

Coarser levels are *replicated* (every rank runs gamblet_fast's level step on
the whole small level -- identical bits on every rank); their subband systems
are independent, so each is solved by one owner rank (levels
dealt round-robin, the owners work concurrently) and broadcast.  The
exception to replication is psi, whose rows
get wider as the level gets coarser: there a rank keeps the *column strip* of
every psi^(k) row (the window points whose fine row it owns), which makes
psi^(k-1), W psi and the increments psi^T W^T w local; only the row maxima of
the tail drop are max-reduced.

The solution is assembled from the ranks' increments: distributed levels
add psi^(k)T W^T w over the rank's own psi rows (a halo_add hands the
overhang to the neighbours), column-strip levels are exact on the rank's fine
rows; an all-gather returns u on every rank.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from . import device as dv
from . import gamblet_fast as gf
from .comm import Comm, SelfComm
from .device import BoxMatrix, PsiWindows, box_slots
from .errors import InvalidArgumentError, NumericalError
from .hierarchy import w_template

__all__ = ["fast_solve_dist", "Rows", "DistResult", "min_distributed_rows"]

# live timing of the strip's dual-vector operator passes (bench.py): {"n": rows
# of the level to time, "cap": launches} -> CUDA events on the launching stream
# around the first `cap` two-vector gb_dist_apply calls of that level; their
# durations (ms) are appended to DIST_TIMING["ms"], the strip's matrix bytes
# are stored under "matrix_bytes" and the vector bytes under "vector_bytes"
DIST_TIMING = None


def min_distributed_rows(world):
    """Smallest parent grid side that is split into strips: strips must be
    whole 4-row tile rows with room for every halo, and the tiled Krylov
    kernels need L % 64 == 0."""
    return max(64, 16 * int(world))


class Rows:
    """Grid rows [a, b) of a row-major (L rows x row_elems) device array,
    addressed by global row: `vptr` is the base pointer the row-range kernels
    take (the address row 0 would have), `x[lo:hi]` slices by global element
    offsets (what comm.Comm's exchanges index with)."""

    def __init__(self, L, row_elems, a, b, dtype=torch.float64, zero=False):
        self.L, self.row_elems = int(L), int(row_elems)
        self.a, self.b = max(int(a), 0), min(int(b), int(L))
        n = (self.b - self.a) * self.row_elems
        self.t = dv.zeros(n, dtype) if zero else dv.empty(n, dtype)

    @property
    def vptr(self):
        return self.t.data_ptr() - self.a * self.row_elems * self.t.element_size()

    def __getitem__(self, sl):
        off = self.a * self.row_elems
        if sl.start - off < 0 or sl.stop - off > self.t.numel():
            raise IndexError(f"rows {sl.start // self.row_elems}..{sl.stop // self.row_elems} "
                             f"outside the held range [{self.a}, {self.b})")
        return self.t[sl.start - off:sl.stop - off]

    def rows(self, x0, x1):
        return self[x0 * self.row_elems:x1 * self.row_elems]

    dtype = property(lambda self: self.t.dtype)
    device = property(lambda self: self.t.device)
    is_cuda = property(lambda self: self.t.is_cuda)

    def element_size(self):
        return self.t.element_size()

    @property
    def nbytes(self):
        return self.t.numel() * self.t.element_size()


class DistResult:
    """What fast_solve_dist returns on every rank."""

    def __init__(self):
        self.u = None                # device tensor, the whole solution (all-gathered)
        self.strips = {}             # k -> {"A", "B", "Dt", "R", "psi", "sB"}: Rows of this rank
        self.levels = {}             # replicated levels: gamblet_fast.LocalGambletLevel
        self.lambdas = {}            # k -> (lambda_min, lambda_max) of S B^(k) S
        self.iterations = {}         # k -> subband PCG iterations
        self.first_replicated = None
        self.peak_bytes = 0
        self.halo_bytes = 0
        self.krylov_passes = {}


def _ptr(x):
    if x is None:
        return None
    return x.vptr if isinstance(x, Rows) else x.data_ptr()


def _box_scale_rows(rows_count_per_grid_row, nr, w, box, out, status, a, b, s):
    """gb_box_scale over grid rows [a, b) (flat entry, offset pointers)."""
    per = rows_count_per_grid_row
    S = box_slots(w, nr)
    nat.call("gb_box_scale", (b - a) * per, nr, w, _ptr(box) + a * per * S * 8,
             _ptr(out) + a * per * 8, status, s)


def _diag_min_rows(per, nr, w, box, dmin_ptr, a, b, s):
    S = box_slots(w, nr)
    nat.call("gb_box_diag_min", (b - a) * per, nr, w, _ptr(box) + a * per * S * 8, dmin_ptr, s)


def _window_reach(n, L, lo, wd, world):
    """(up, down): how many rows above / below a rank's strip of the L-row
    level have psi windows (origin clamp(i h + lo, 0, n - wd), width wd) that
    reach into the strip's fine rows -- the maximum over the ranks, since the
    halo widths of an exchange are the same on every rank."""
    h = n // L
    org = np.clip(np.arange(L) * h + lo, 0, n - wd)
    up = dn = 0
    for r in range(world):
        p0, p1 = L * r // world, L * (r + 1) // world
        f0, f1 = p0 * h, p1 * h
        above = np.nonzero(org[:p0] + wd > f0)[0]
        below = np.nonzero(org[p1:] < f1)[0]
        if above.size:
            up = max(up, p0 - int(above[0]))
        if below.size:
            dn = max(dn, int(below[-1]) + 1)
    return up, dn


class _StripOp:
    """This rank's rows of the symmetric band Krylov copy of S B^(k) S and of
    the block-Jacobi inverses; vectors keep the global padded layout."""

    def __init__(self, comm, Lp, wB, Bv, sB, p0, p1):
        self.comm, self.L, self.w, self.nr = comm, Lp, wB, 3
        self.p0, self.p1 = p0, p1
        self.n = 3 * Lp * Lp
        self.Lpad = Lp + 2 * wB
        self.npad = self.Lpad * self.Lpad * 3
        self.vtail = nat.query("gb_sym_overflow_elems", Lp, wB)
        s = dv.stream()
        ns = nat.query("gb_boxsym_elems", Lp, wB) // (Lp * Lp)  # slots per parent
        self.slots_per_parent = ns
        self.BsT = Rows(Lp, Lp * ns, p0, p1)
        nat.call("gb_scale_box_symT_rows", Lp, wB, _ptr(Bv), _ptr(sB), self.BsT.vptr, p0, p1, s)
        Lb = Lp // 2
        self.inv = Rows(Lb, Lb * 144, p0 // 2, p1 // 2, dtype=torch.float32)
        nat.call("gb_bj_setup_rows", Lp, wB, _ptr(Bv), _ptr(sB), self.inv.vptr, p0, p1, s)
        # geometry of the per-iteration exchanges
        self.tile_rows = Lp // 4
        self.tile_row_elems = (Lp // 64) * (4 + wB) * (64 + 2 * wB) * 3
        self.KI = (wB + 3) // 4
        self.matrix_bytes = self.BsT.nbytes

    def vec(self):
        return dv.zeros(self.npad + self.vtail)

    # the operator input needs the w rows below the strip
    def halo_x(self, *vecs):
        re = self.Lpad * 3
        self.comm.halo_many([(_PaddedView(v, self.w, self.L, re), self.L, re, 0, self.w)
                             for v in vecs])

    # the neighbour above sends the spill-over of its last KI tile rows
    def halo_spill(self, *vecs):
        self.comm.halo_many([(v[self.npad:], self.tile_rows, self.tile_row_elems, self.KI, 0)
                             for v in vecs])


class _PaddedView:
    """Grid row r of a padded vector = padded row r + w (all padded columns)."""

    def __init__(self, v, w, L, row_elems):
        self.v, self.off = v, w * row_elems
        self.dtype, self.device, self.is_cuda = v.dtype, v.device, v.is_cuda

    def __getitem__(self, sl):
        return self.v[sl.start + self.off:sl.stop + self.off]

    def element_size(self):
        return self.v.element_size()


class _KState:
    def __init__(self):
        nb = nat.query("gb_kstate_bytes")
        self.state = dv.empty(nb, torch.uint8)
        self.host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        self.part = dv.empty(3 * nat.query("gb_red_blocks"))
        nat.call("gb_state_reset", dv.ptr(self.state), 0, dv.stream())

    def read(self):
        nat.call("gb_sync_read", dv.ptr(self.state), self.host.data_ptr(), self.host.numel(),
                 dv.stream())
        return self.host.numpy().view(gf._KSTATE)[0]


def _dist_krylov(op, rhs_pad, tol, spectral=True, eig_tol=0.1, max_outer=500, seed=24337):
    """Distributed gb_level_engine: block-Jacobi PCG for (S B S) z = rhs on
    the rank's strip, paired with the lambda estimates of S B S (power
    iteration, then the Lanczos moments of the inverse iteration's start
    vector; same start vectors, stopping tests and host evaluation as the
    single-GPU engine, gamblet_fast._paired_level).  Returns a dict like it."""
    comm, L, w = op.comm, op.L, op.w
    p0, p1 = op.p0, op.p1
    s = dv.stream()
    n = op.n
    Lpad = op.Lpad
    off = (p0 + w) * Lpad * 3
    cnt = (p1 - p0) * Lpad * 3
    U, inv = op.BsT.vptr, op.inv.vptr
    # --- A: PCG ---------------------------------------------------------
    ka = _KState()
    xa, ra, pa, apa, za = (op.vec() for _ in range(5))
    red = dv.zeros(2)       # all-reduced after phase 1: (p.Ap, x.y of the B half)
    outs = dv.zeros(4)      # all-reduced after the updates, one message:
    outa = outs[0:3]        #   A (rr, rz[, bb at the start])
    outb = outs[3:4]        #   B: y.y / |u|^2
    outr = dv.zeros(1)      # B: power residual
    max_a = min(max(200, 2 * n), gf.MAX_ITER_CAP)
    nat.call("gb_dist_pcg_init", L, w, dv.ptr(rhs_pad), dv.ptr(xa), dv.ptr(ra), dv.ptr(pa),
             dv.ptr(za), inv, dv.ptr(ka.state), dv.ptr(ka.part), dv.ptr(outa), p0, p1, s)
    comm.allreduce(outa, "sum")
    nat.call("gb_dist_pcg_init_commit", dv.ptr(ka.state), dv.ptr(outa), float(tol), int(max_a), s)
    passes = [0, 0]
    timing = DIST_TIMING if (DIST_TIMING is not None and DIST_TIMING.get("n") == n) else None
    evs = []

    def a_post():
        nat.call("gb_dist_pcg_update", L, w, dv.ptr(xa), dv.ptr(ra), dv.ptr(pa), dv.ptr(apa),
                 dv.ptr(za), inv, dv.ptr(ka.state), dv.ptr(red), dv.ptr(ka.part), dv.ptr(outa),
                 p0, p1, s)

    def a_commit():
        nat.call("gb_dist_pcg_commit_dir", L, w, dv.ptr(ka.state), dv.ptr(red), dv.ptr(outa),
                 dv.ptr(za), dv.ptr(pa), p0, p1, s)

    def apply(a_live, xb=None, yb=None, kb=None):
        """One pass over the strip's rows of S B S for the live halves."""
        if a_live and xb is not None:
            op.halo_x(pa, xb)
            timed = timing is not None and len(evs) < int(timing.get("cap", 64))
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            nat.call("gb_dist_apply", L, w, U, 2, dv.ptr(pa), dv.ptr(apa), dv.ptr(ka.state),
                     dv.ptr(ka.part), dv.ptr(xb), dv.ptr(yb), dv.ptr(kb.state), dv.ptr(kb.part),
                     dv.ptr(red), p0, p1, s)
            if timed:
                e1.record()
                evs.append((e0, e1))
            op.halo_spill(apa, yb)
            passes[0] += 1
        elif a_live:
            op.halo_x(pa)
            nat.call("gb_dist_apply", L, w, U, 1, dv.ptr(pa), dv.ptr(apa), dv.ptr(ka.state),
                     dv.ptr(ka.part), None, None, None, None, dv.ptr(red), p0, p1, s)
            op.halo_spill(apa)
            passes[1] += 1
        else:
            # the B half alone: it rides in vector slot 0, its sum lands in red[0]
            op.halo_x(xb)
            nat.call("gb_dist_apply", L, w, U, 1, dv.ptr(xb), dv.ptr(yb), dv.ptr(kb.state),
                     dv.ptr(kb.part), None, None, None, None, dv.ptr(red), p0, p1, s)
            red[1:2].copy_(red[0:1])
            op.halo_spill(yb)
            passes[1] += 1
        comm.allreduce(red, "sum")

    out = {"lam_min": None, "lam_max": None, "calls": 0}
    ha = ka.read()
    if spectral:
        # --- B: start vectors drawn exactly as eig_extremes draws them ----
        x1, x2 = gf._start_vectors(n, seed)
        kb = _KState()
        xb, yb, xs, vp = (op.vec() for _ in range(4))
        nrm = dv.zeros(1)
        for src, dst in ((x1, xb), (x2, xs)):
            # the strip's rows of the unit start vector (global norm)
            nat.call("gb_pad_rows", L, 3, w, dv.ptr(src), None, dv.ptr(dst), p0, p1, s)
            nat.call("gb_dist_dot", cnt, dv.ptr(dst) + off * 8, dv.ptr(dst) + off * 8,
                     dv.ptr(kb.state), dv.ptr(kb.part), dv.ptr(nrm), s)
            comm.allreduce(nrm, "sum")
            nat.call("gb_scale_by_norm", cnt, dv.ptr(dst) + off * 8, dv.ptr(nrm), 0,
                     dv.ptr(dst) + off * 8, None, s)
        nat.call("gb_state_reset", dv.ptr(kb.state), int(max_outer), s)
        # power iteration paired with the PCG (sparse_core.py:244-257)
        chunk = 8
        while True:
            a_live = not ha["done"]
            for _ in range(chunk):
                apply(a_live, xb, yb, kb)
                if a_live:
                    a_post()
                nat.call("gb_dist_fix_yy", L, w, dv.ptr(yb), dv.ptr(kb.state), dv.ptr(kb.part),
                         dv.ptr(outb), p0, p1, s)
                comm.allreduce(outs, "sum")
                if a_live:
                    a_commit()
                nat.call("gb_dist_pow_step", L, w, dv.ptr(xb), dv.ptr(yb), dv.ptr(kb.state),
                         dv.ptr(red), dv.ptr(outb), dv.ptr(outr), dv.ptr(kb.part),
                         float(eig_tol), p0, p1, 0, s)
                comm.allreduce(outr, "sum")
                nat.call("gb_dist_pow_step", L, w, dv.ptr(xb), dv.ptr(yb), dv.ptr(kb.state),
                         dv.ptr(red), dv.ptr(outb), dv.ptr(outr), dv.ptr(kb.part),
                         float(eig_tol), p0, p1, 1, s)
            ha = ka.read()
            hb = kb.read()
            if hb["done"]:
                break
            chunk = min(chunk * 2, 128)
        out["lam_max"] = float(hb["lam"])
        out["power_its"] = int(hb["it"])
        out["calls"] = int(hb["it"]) + (0 if hb["ynorm"] != 0 else 1)
        # Lanczos moments of the inverse iteration's start vector (gb_lanczos.h)
        cap = int(min(n, gf.LANCZOS_CAP))
        lz = dv.empty(2 * cap)
        hlz = np.empty(2 * cap)
        v, wv = xs, yb
        nat.call("gb_dist_lz_begin", dv.ptr(kb.state), cap, s)
        chunk, lam, m = 64, None, 0
        lamc = nat.ctypes.c_double(0.0)
        outc = nat.ctypes.c_int(0)
        stopc = nat.ctypes.c_int(0)
        while True:
            a_live = not ha["done"]
            for _ in range(chunk):
                apply(a_live, v, wv, kb)
                if a_live:
                    a_post()
                nat.call("gb_dist_lz_update", L, w, dv.ptr(v), dv.ptr(wv), dv.ptr(vp),
                         dv.ptr(kb.state), dv.ptr(red), dv.ptr(kb.part), dv.ptr(outb), p0, p1, s)
                comm.allreduce(outs, "sum")
                if a_live:
                    a_commit()
                nat.call("gb_dist_lz_commit", dv.ptr(kb.state), dv.ptr(red), dv.ptr(outb),
                         dv.ptr(lz), s)
                v, wv = wv, v
            ha = ka.read()
            hb = kb.read()
            m = int(hb["it"])
            if m > 0:
                hlz[:2 * m] = dv.to_host(lz[:2 * m])
                rc = nat.query("gb_lanczos_check", hlz.ctypes.data, m, float(eig_tol),
                               int(max_outer), float(gf.LANCZOS_TOL), nat.ctypes.byref(lamc),
                               nat.ctypes.byref(outc), nat.ctypes.byref(stopc))
                if rc:
                    raise NumericalError(
                        f"Lanczos moments of S B S at n={n}: "
                        + ("nonpositive pivot (matrix is not SPD)" if rc == 2
                           else "evaluation failed"))
                lam = float(lamc.value)
                if hb["done"] or stopc.value:
                    break
            elif hb["done"]:
                raise NumericalError("inverse iteration broke down: A^{-1} x = 0")
            chunk = 32
        out["lam_min"] = lam
        out["lanczos"] = m
        out["calls"] += m
    # --- the PCG alone until it converges -------------------------------
    chunk = 8
    while not ha["done"]:
        for _ in range(chunk):
            apply(True)
            a_post()
            comm.allreduce(outa, "sum")
            a_commit()
        ha = ka.read()
        chunk = min(chunk * 2, 128)
    if ha["breakdown"]:
        raise NumericalError(f"CG breakdown at iteration {int(ha['breakdown'])}: p^T A p <= 0 "
                             "(matrix is not SPD)")
    if ha["aux0"] != 0.0:  # zero right-hand side: the solution is zero
        xa.zero_()
    if timing is not None and evs:
        evs[-1][1].synchronize()
        timing.setdefault("ms", []).extend(a.elapsed_time(b) for a, b in evs)
        timing["matrix_bytes"] = op.matrix_bytes
        timing["vector_bytes"] = 4 * 8 * (p1 - p0 + w) * Lpad * 3
    rel = float(ha["rnorm"] / ha["bnorm"]) if ha["bnorm"] > 0 else 0.0
    out.update(x=xa, its=int(ha["it"]), rel=rel, conv=bool(ha["converged"]),
               passes=tuple(passes))
    return out


class _NoTasks:
    """Level-step spool that runs nothing: the replicated levels' solves are
    assigned to owner ranks afterwards."""

    def submit(self, level, op, k, g=None):
        return

    def join(self, counter):
        return


def _psi_next_cols(comm, level, psiw, n, k, sched, w12, f0, f1, s):
    """psi^(k-1) from psi^(k) and the level's D^T on this rank's column strip
    (the window points with fine row in [f0, f1)): the psi part of
    gamblet_fast.local_level_step (gamblet_fast.py:615-624), row maxima of the
    tail drop max-reduced over the ranks."""
    Lk, Lp = 1 << k, 1 << (k - 1)
    P, J = Lp * Lp, 3 * Lp * Lp
    rho = int(min(sched.rho(k - 1), Lp - 1))
    Dt = level.raw("correction").vals
    h = n // Lk
    lo, hi, wd = psiw.lo, psiw.hi, psiw.wd
    wdw = min(hi - lo + 1 + h, n)
    Wpsi = dv.empty(J * wdw * wdw)
    lo2, hi2 = -2 * rho * h + lo, (2 * rho + 1) * h + hi
    wd2 = PsiWindows.window(n, lo2, hi2)
    pv = dv.empty(P * wd2 * wd2)
    rmax = dv.empty(P)
    nat.call("gb_wpsi_rows", n, Lk, lo, wd, w12, dv.ptr(psiw.vals), wdw, dv.ptr(Wpsi), 0, Lp,
             f0, f1, s)
    nat.call("gb_psi_next_raw_rows", n, Lk, lo, hi, wd, dv.ptr(psiw.vals), wdw, dv.ptr(Wpsi),
             rho, dv.ptr(Dt), lo2, wd2, dv.ptr(pv), dv.ptr(rmax), 0, Lp, f0, f1, s)
    comm.allreduce(rmax, "max")
    nat.call("gb_psi_drop_rows", n, Lp, lo2, wd2, dv.ptr(pv), dv.ptr(rmax), 0, Lp, f0, f1, s)
    return PsiWindows(pv, n, Lp, lo2, hi2)


def fast_solve_dist(comm: Comm, M, A, g_nodal, tree, epsilon, uniform_rho=None, c_rho=None,
                    w_variant="orthonormal", lean=True, keep=False, spectral=True,
                    force_strips=False):
    """gamblet_fast.fast_solve (nodal load) on `comm.world` ranks, this rank's
    part.  M, A: the whole mass / stiffness matrix on every rank (BoxMatrix
    from grid_fem.assemble_*(device=True), DeviceCSR or canonical scipy CSR:
    9 values per row, the one replicated input); g_nodal: the whole nodal load.

    Returns a DistResult; `u` is the whole solution on every rank.  keep=True
    retains this rank's strips of every distributed level (parity tests);
    lean=True releases each operator once consumed.  force_strips=True runs the
    strip program even on one rank (a single strip, no exchange): the
    single-GPU measurement of the partitioned code path."""
    comm = comm if comm is not None else SelfComm()
    q = tree.q
    n = 1 << q
    N = n * n
    world, rank = comm.world, comm.rank
    if world & (world - 1):
        raise InvalidArgumentError(f"the spatial partition needs a power-of-two world, got {world}")
    sched = gf.make_schedule(epsilon, q, c_rho=c_rho, uniform_rho=uniform_rho)
    tol = sched.subband_tol()
    tmpl = w_template(w_variant)
    w12 = tmpl.ctypes.data
    s = dv.stream()
    ctx = gf._Ctx()
    ctx.comm = comm
    counter = gf.FlopCounter()
    res = DistResult()
    Lmin = min_distributed_rows(world)
    torch.cuda.reset_peak_memory_stats()
    bytes0 = getattr(comm, "bytes_sent", 0)

    def strip(L):
        return comm.strip(L)

    # replicated inputs -> boxes (half-width 1)
    Mb = M if isinstance(M, BoxMatrix) else dv.csr_to_box(gf._canon(M), n)[0]
    Ab = A if isinstance(A, BoxMatrix) else dv.csr_to_box(gf._canon(A), n)[0]
    gfull = dv.to_dev(g_nodal if isinstance(g_nodal, torch.Tensor)
                      else np.asarray(g_nodal, dtype=float))
    uacc = dv.zeros(N)           # this rank's increments (own fine rows + overhang)
    over = [0, 0]                # fine rows of overhang above / below the strip
    f0, f1 = strip(n)

    # ------------------------------------------------------------------
    # level q: psi^(q) by mass patches, A^(q) = psi A psi^T (gamblet_fast._level_q)
    # ------------------------------------------------------------------
    dist_q = (world > 1 or force_strips) and n // 2 >= Lmin
    if not dist_q:
        # nothing to split at this size: the single-GPU program on every rank
        # (world == 1, or a grid too small for strips)
        levels, parts, U1, _ = gf._fast_solve_device(Mb, Ab, gfull, tree, sched,
                                                     w_variant=w_variant, lean=q >= 12)
        res.u = parts["partials"].device(q)
        res.levels = levels
        res.first_replicated = q
        for k, lv in levels.items():
            if k >= 2:
                res.lambdas[k] = (lv.lambda_min_subband, lv.lambda_max_subband)
        res.peak_bytes = torch.cuda.max_memory_allocated()
        return res

    rho = int(min(sched.rho(q), n - 1))
    lo, hi = -rho, rho
    wd = PsiWindows.window(n, lo, hi)
    wX = min(rho + Ab.w, n - 1)
    wR = min(wX + rho, n - 1)
    SX, SR = box_slots(wX, 1), box_slots(wR, 1)
    a, b = max(f0 - rho, 0), min(f1 + rho, n)
    sM = Rows(n, n, a, b)
    _box_scale_rows(n, 1, Mb.w, Mb.vals, sM, ctx.st(ctx.slot("scale", "mass")), a, b, s)
    psi = Rows(n, n * wd * wd, f0 - wR, f1 + wR)
    nat.call("gb_mass_patches_rows", n, Mb.w, dv.ptr(Mb.vals), sM.vptr, rho, wd, psi.vptr,
             ctx.st(ctx.slot("mass", "mass")), f0, f1, s)
    X = Rows(n, n * SX, f0, f1)
    nat.call("gb_psi_stencil_rows", n, lo, wd, rho, psi.vptr, Ab.w, dv.ptr(Ab.vals), wX, X.vptr,
             f0, f1, s)
    comm.halo(psi, n, n * wd * wd, wR, wR)
    raw = Rows(n, n * SR, f0 - wR, f1 + wR)
    work = dv.empty(nat.query("gb_psi_galerkin_workspace_rows", n, wd, wX, wR, f0, f1) // 8)
    nat.call("gb_psi_galerkin_t_rows", n, lo, wd, rho, psi.vptr, wX, X.vptr, wR, raw.vptr,
             dv.ptr(work), f0, f1, s)
    del work, X, sM
    ia = ctx.slot("sym", "A^(q),loc")
    _diag_min_rows(n, 1, wR, raw, ctx.dm(ia), f0, f1, s)
    comm.allreduce(ctx.dmin[ia:ia + 1], "min")
    comm.halo(raw, n, n * SR, wR, wR)
    Ak = Rows(n, n * SR, f0, f1)
    nat.call("gb_box_sym_drop_rows", n, 1, wR, raw.vptr, Ak.vptr, ctx.dm(ia), ctx.sp(ia), f0, f1,
             s)
    del raw
    wA = wR
    psi_lo, psi_hi, psi_wd = lo, hi, wd
    # psi^(q) rows of this rank only from here on (the halo rows are not needed again)
    gk = Rows(n, n, f0 - 2 * int(min(sched.rho(q - 1), n // 2 - 1)),
              f1 + 2 * int(min(sched.rho(q - 1), n // 2 - 1)))
    gk.rows(f0, f1).copy_(gfull[f0 * n:f1 * n])
    del gfull
    if keep:
        res.strips[q] = {"A": Ak, "psi": psi, "wA": wA, "psi_lo": lo, "psi_hi": hi}

    # ------------------------------------------------------------------
    # distributed level steps k -> k-1 (gamblet_fast.local_level_step on strips)
    # ------------------------------------------------------------------
    k = q
    while k >= 2 and (1 << (k - 1)) >= Lmin:
        Lk, Lp = 1 << k, 1 << (k - 1)
        p0, p1 = strip(Lp)
        P = Lp * Lp
        wB = min((wA + 1) // 2, Lp - 1)
        rho = int(min(sched.rho(k - 1), Lp - 1))
        SB3, SG, SD = box_slots(wB, 3), box_slots(wB, 1), box_slots(rho, 3)
        # K3: B (sym + dead-tail drop fused), G, P A P^T
        ib = ctx.slot("sym", f"B^({k}),loc")
        bdiag = Rows(Lp, Lp * 3, p0 - wB, p1 + wB)
        nat.call("gb_level_diag_rows", Lk, wA, Ak.vptr, w12, bdiag.vptr, ctx.dm(ib), p0, p1, s)
        comm.halo(bdiag, Lp, Lp * 3, wB, wB)
        comm.allreduce(ctx.dmin[ib:ib + 1], "min")
        hG = max(rho, wB)
        Bv = Rows(Lp, Lp * 3 * SB3, p0 - rho, p1 + rho)
        Gv = Rows(Lp, Lp * 3 * SG, p0 - hG, p1 + hG)
        PAPt = Rows(Lp, Lp * SG, p0, p1)
        nat.call("gb_level_blocks_rows", Lk, wA, Ak.vptr, w12, wB, bdiag.vptr, ctx.dm(ib),
                 Bv.vptr, Gv.vptr, PAPt.vptr, ctx.sp(ib), p0, p1, s)
        del bdiag
        if lean and not keep:
            Ak = None
        sB = Rows(Lp, Lp * 3, p0 - hG, p1 + hG)
        _box_scale_rows(Lp * 3, 3, wB, Bv, sB, ctx.st(ctx.slot("scale", f"B^({k}),loc")), p0, p1,
                        s)
        comm.halo(sB, Lp, Lp * 3, hG, hG)
        # the Krylov copy of the strip's rows and the level's solve run first
        # (the single-GPU path overlaps them with the patches on a side stream)
        op = _StripOp(comm, Lp, wB, Bv, sB, p0, p1)
        rhs = Rows(Lp, Lp * 3, p0, p1)
        nat.call("gb_apply_w_rows", Lp, w12, gk.vptr, sB.vptr, rhs.vptr, p0, p1, s)
        bp = op.vec()
        nat.call("gb_pad_rows", Lp, 3, wB, rhs.vptr, None, dv.ptr(bp), p0, p1, s)
        kr = _dist_krylov(op, bp, tol, spectral=spectral)
        if not kr["conv"]:
            raise NumericalError(f"subband solve at level {k} did not converge")
        res.iterations[k] = kr["its"]
        res.lambdas[k] = (kr["lam_min"], kr["lam_max"])
        res.krylov_passes[k] = kr["passes"]
        wk = Rows(Lp, Lp * 3, p0, p1)
        nat.call("gb_unpad_rows", Lp, 3, wB, dv.ptr(kr["x"]), sB.vptr, wk.vptr, p0, p1, s)
        vk = Rows(Lk, Lk, 2 * p0, 2 * p1)
        nat.call("gb_apply_wt_rows", Lp, w12, wk.vptr, vk.vptr, p0, p1, s)
        # increment psi^(k)T W^T w over this rank's psi rows -> uacc
        h = n // Lk
        F0 = int(np.clip(2 * p0 * h + psi_lo, 0, n - psi_wd))
        F1 = int(np.clip((2 * p1 - 1) * h + psi_lo, 0, n - psi_wd)) + psi_wd
        inc = dv.empty((F1 - F0) * n)
        nat.call("gb_psi_t_apply_rows", n, Lk, psi_lo, psi_wd, psi.vptr, vk.vptr,
                 dv.ptr(inc) - F0 * n * 8, F0, F1, 2 * p0, 2 * p1, s)
        nat.call("gb_vadd", (F1 - F0) * n, dv.ptr(uacc) + F0 * n * 8, dv.ptr(inc),
                 dv.ptr(uacc) + F0 * n * 8, s)
        over[0], over[1] = max(over[0], f0 - F0), max(over[1], F1 - f1)
        del inc, vk, wk, kr, bp, rhs, op
        # K4: correction patches -> D^T rows (trim fused)
        comm.halo(Bv, Lp, Lp * 3 * SB3, rho, rho)
        comm.halo(Gv, Lp, Lp * 3 * SG, hG, hG)
        hD = min(wB + rho, Lp - 1)
        Dt = Rows(Lp, Lp * SD, p0 - hD, p1 + hD)
        wsb = nat.query("gb_correction_patches_workspace", Lp, rho, p0, p1)
        ws = dv.empty((wsb + 7) // 8) if wsb else None
        nat.call("gb_correction_patches_rows", Lp, wB, Bv.vptr, sB.vptr, wB, Gv.vptr, rho,
                 Dt.vptr, ctx.st(ctx.slot("corr", f"level {k}", detail=k)), p0, p1, dv.ptr(ws),
                 wsb, s)
        del ws
        Rv = Rows(Lp, Lp * box_slots(rho, 4), p0, p1)
        nat.call("gb_restriction_rows", Lp, rho, Dt.vptr, w12, Rv.vptr, p0, p1, s)
        comm.halo(Dt, Lp, Lp * SD, hD, hD)
        # K6: split triple product
        wBD = wGD = hD
        wA2 = min(2 * rho + wB, Lp - 1)
        SBD, SA2 = box_slots(wBD, 1), box_slots(wA2, 1)
        BD = Rows(Lp, Lp * 3 * SBD, p0 - rho, p1 + rho)
        nat.call("gb_bd_rows", Lp, wB, Bv.vptr, rho, Dt.vptr, wBD, BD.vptr, p0, p1, s)
        comm.halo(BD, Lp, Lp * 3 * SBD, rho, rho)
        GtD = Rows(Lp, Lp * SBD, p0 - wGD, p1 + wGD)
        nat.call("gb_gtd_rows", Lp, wB, Gv.vptr, rho, Dt.vptr, wGD, GtD.vptr, p0, p1, s)
        comm.halo(GtD, Lp, Lp * SBD, wGD, wGD)
        raw = Rows(Lp, Lp * SA2, p0 - wA2, p1 + wA2)
        nat.call("gb_coarse_raw_rows", Lp, wB, PAPt.vptr, wGD, GtD.vptr, rho, Dt.vptr, wBD,
                 BD.vptr, wA2, raw.vptr, p0, p1, s)
        del BD, GtD, PAPt, Gv
        ia = ctx.slot("sym", f"A^({k - 1}),loc")
        _diag_min_rows(Lp, 1, wA2, raw, ctx.dm(ia), p0, p1, s)
        comm.allreduce(ctx.dmin[ia:ia + 1], "min")
        comm.halo(raw, Lp, Lp * SA2, wA2, wA2)
        An = Rows(Lp, Lp * SA2, p0, p1)
        nat.call("gb_box_sym_drop_rows", Lp, 1, wA2, raw.vptr, An.vptr, ctx.dm(ia), ctx.sp(ia),
                 p0, p1, s)
        del raw
        # psi^(k-1) = drop_row(0.25 P psi + D^T (W psi)) on the rank's parent rows
        wdw = min(psi_hi - psi_lo + 1 + h, n)
        Wpsi = Rows(Lp, Lp * 3 * wdw * wdw, p0 - rho, p1 + rho)
        nat.call("gb_wpsi_rows", n, Lk, psi_lo, psi_wd, w12, psi.vptr, wdw, Wpsi.vptr, p0, p1, 0,
                 n, s)
        comm.halo(Wpsi, Lp, Lp * 3 * wdw * wdw, rho, rho)
        lo2, hi2 = -2 * rho * h + psi_lo, (2 * rho + 1) * h + psi_hi
        wd2 = PsiWindows.window(n, lo2, hi2)
        last = not (k - 1 >= 2 and (1 << (k - 2)) >= Lmin)
        # the last distributed step hands psi^(k-1) to the column strips: its
        # rows whose windows reach into the neighbours' fine rows travel once
        Hup, Hdn = _window_reach(n, Lp, lo2, wd2, world) if last else (0, 0)
        pv = Rows(Lp, Lp * wd2 * wd2, p0 - Hup, p1 + Hdn)
        rmax = Rows(Lp, Lp, p0, p1)
        nat.call("gb_psi_next_raw_rows", n, Lk, psi_lo, psi_hi, psi_wd, psi.vptr, wdw, Wpsi.vptr,
                 rho, Dt.vptr, lo2, wd2, pv.vptr, rmax.vptr, p0, p1, 0, n, s)
        nat.call("gb_psi_drop_rows", n, Lp, lo2, wd2, pv.vptr, rmax.vptr, p0, p1, 0, n, s)
        del Wpsi, rmax
        # g^(k-1) = R g^(k)
        comm.halo(gk, Lk, Lk, 2 * rho, 2 * rho)
        rho_n = int(min(sched.rho(k - 2), Lp // 2 - 1)) if k - 2 >= 1 else 0
        gn = Rows(Lp, Lp, p0 - 2 * rho_n, p1 + 2 * rho_n)
        nat.call("gb_apply_r_rows", Lp, rho, Rv.vptr, gk.vptr, gn.vptr, p0, p1, s)
        if keep:
            res.strips[k].update({"B": Bv, "sB": sB, "Dt": Dt, "R": Rv, "wB": wB, "rho": rho})
            res.strips[k - 1] = {"A": An, "psi": pv, "wA": wA2, "psi_lo": lo2, "psi_hi": hi2}
        del Bv, sB, Dt, Rv
        psi, psi_lo, psi_hi, psi_wd = pv, lo2, hi2, wd2
        Ak, wA, gk = An, wA2, gn
        k -= 1

    # ------------------------------------------------------------------
    # hand-over to the replicated levels: A^(k) and g^(k) are gathered whole,
    # psi^(k) keeps its rows near the strip (column strips from here on)
    # ------------------------------------------------------------------
    res.first_replicated = k
    Lk = 1 << k
    p0, p1 = strip(Lk)
    SA = box_slots(wA, 1)
    Afull = dv.empty(Lk * Lk * SA)
    Afull[p0 * Lk * SA:p1 * Lk * SA].copy_(Ak.rows(p0, p1))
    comm.allgather_rows(Afull, Lk, Lk * SA)
    gfull = dv.empty(Lk * Lk)
    gfull[p0 * Lk:p1 * Lk].copy_(gk.rows(p0, p1))
    comm.allgather_rows(gfull, Lk, Lk)
    per = psi_wd * psi_wd
    comm.halo(psi, Lk, Lk * per, Hup, Hdn)
    # full-size window array (only the rows near the strip are ever read: the
    # column mask keeps every kernel inside them)
    psifull = dv.empty(Lk * Lk * per)
    psifull[psi.a * Lk * per:psi.b * Lk * per].copy_(psi.t)
    if not keep:
        del psi, Ak, gk
    # (R1) the operators of the replicated levels -- B^(k), D, R, A^(k-1), no
    # psi yet: every rank, identical bits (the levels are small)
    level = gf.LocalGambletLevel(k, None, BoxMatrix(Afull, Lk, 1, wA, 1))
    level._repair_slot_a = -1
    levels = {k: level}
    records = []
    solver = gf._LevelSolver(levels, tree, tol, counter, records)
    solver.fine_rows = (f0, f1)
    gs = {k: gfull}
    for kk in range(k, 1, -1):
        levels[kk - 1] = gf.local_level_step(levels[kk], tree, sched, w_variant=w_variant,
                                             counter=counter, _ctx=ctx, _spool=_NoTasks(),
                                             _g=None, _lean=False)
        gs[kk - 1] = solver.restrict(kk, gs[kk])
    # (R2) the independent subband systems of those levels (SPEC.md:401,
    # PAPER.md:1515), one owner rank each: the owners solve concurrently,
    # then every rank receives every w^(k) (and the lambda estimates)
    prep, sols = {}, {}
    for kk in range(k, 1, -1):
        owner = (k - kk) % world
        op, sBk, rhs = solver.subband_rhs(kk, gs[kk])
        prep[kk] = (op, sBk)
        zp = op.vec()
        sc = dv.zeros(6)
        if owner == rank:
            if spectral and gf.PAIRED_ENGINE and gf._engine_ok(op):
                out = gf._paired_level(op, op.pad(rhs), tol)
                z, vals = out["x"], (out["its"], out["rel"], out["conv"], out["brk"],
                                     out["lam_min"], out["lam_max"])
            else:
                lmin = lmax = float("nan")
                if spectral:
                    lmin, lmax, _ = gf._eig_extremes(op)
                z, its, rel, conv, brk, _ = gf._pcg(op, op.pad(rhs), tol)
                vals = (its, rel, conv, brk, lmin, lmax)
            zp.copy_(z)
            sc.copy_(torch.tensor([float(v) for v in vals], dtype=torch.float64))
        sols[kk] = (owner, zp, sc)
        del rhs
    for kk in range(k, 1, -1):
        owner, zp, sc = sols[kk]
        comm.broadcast(zp, owner)
        comm.broadcast(sc, owner)
    # (R3) psi^(k-1) = drop_row(0.25 P psi + D^T W psi) down the replicated
    # levels on this rank's column strip, each level's increment formed before
    # its psi^(k) is released
    psik = PsiWindows(psifull, n, Lk, psi_lo, psi_hi)
    for kk in range(k, 1, -1):
        owner, zp, sc = sols[kk]
        its, rel, conv, brk, lmin, lmax = dv.to_host(sc).tolist()
        levels[kk].psi = psik
        if spectral:
            levels[kk].lambda_min_subband, levels[kk].lambda_max_subband = lmin, lmax
        res.lambdas[kk] = (levels[kk].lambda_min_subband, levels[kk].lambda_max_subband)
        res.iterations[kk] = int(its)
        op, sBk = prep[kk]
        solver.subband_finish(kk, op, sBk, zp, int(its), rel, bool(conv), int(brk), psi=psik)
        psin = _psi_next_cols(comm, levels[kk], psik, n, kk, sched, w12, f0, f1, s)
        if lean and not keep:
            levels[kk].psi = None
        psik = psin
        del sols[kk], prep[kk]
    levels[1].psi = psik
    solver.coarse(gs[1])
    for kk in sorted(solver.incs.keys(), reverse=True):
        inc = solver.incs.device(kk)
        nat.call("gb_vadd", (f1 - f0) * n, dv.ptr(uacc) + f0 * n * 8,
                 inc.data_ptr() + f0 * n * 8, dv.ptr(uacc) + f0 * n * 8, s)
    ctx.check()
    # hand the overhang of the distributed levels' increments to its owners,
    # then every rank collects the whole solution
    ov = torch.tensor(over, dtype=torch.int64, device=uacc.device)
    comm.allreduce(ov, "max")
    up, down = (int(x) for x in ov.tolist())
    comm.halo_add(uacc, n, n, up, down)
    comm.allgather_rows(uacc, n, n)
    res.u = uacc
    res.levels = levels
    res.peak_bytes = torch.cuda.max_memory_allocated()
    res.halo_bytes = getattr(comm, "bytes_sent", 0) - bytes0
    return res
