"""Localized gamblet transform and subband solve on the B200 (Algorithm 2).

Drop-in for gamblets/gamblet_fast.py: same entry points, signatures, result
types and exceptions (reference file:line in each docstring).  The host code
only sequences device work: every operator lives on the GPU in box-stencil
layout (csrc/gb_common.cuh) and every arithmetic step is a kernel of
libgamblets_b200.so:

    level q init   K1 mass patches -> psi^(q);  K2 X = psi A, psi A psi^T,
                   symmetrize + tail drop                      -> A^(q)
    level k -> k-1 K3 B = W A W^T (+ sym + drop), G, P A P^T;  K7 spectral
                   estimates of S B S;  K4 correction patches -> D^T (trimmed);
                   K6 R = pibar + D^T W, BD, G^T D, split triple product ->
                   A^(k-1);  psi^(k-1) = drop_row(0.25 P psi + D^T W psi)
    solve          K9 W g, R g, psi^T W^T w;  K8 scaled CG per subband level

Patch systems are factored exactly (Cholesky) instead of the reference's CG
to a clamped tolerance; in the reference's tight mode (epsilon=1e-13,
c_tol=1e-6) the two agree to 1e-13, so `c_tol` and
`dense_cutoff` are accepted for API compatibility and do not change results.
"""

from __future__ import annotations

import os

import concurrent.futures
import threading
import time
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as nat
from . import device as dv
from . import partition as part
from .device import EXP_CHILD, EXP_SQUARE, EXP_TDT, BoxMatrix, PsiWindows
from .errors import InvalidArgumentError, NumericalError
from .gamblet_exact import HostDict, MultiresSolution, SolveRecord
from .grid_fem import LoadVector
from .hierarchy import w_template
from .sparse_core import as_csr, cg_flops, is_canonical_csr

__all__ = [
    "DEFAULT_C_RHO", "KAPPA", "LocalizationSchedule", "LocalGambletLevel",
    "FlopCounter", "FastResult", "make_schedule", "local_mass_inverse",
    "local_level_step", "fast_transform", "solve_with_transform", "fast_solve",
]

# gamblet_fast.py:65-116
DEFAULT_C_RHO = 0.5
KAPPA = 12.0
DEFAULT_C_TOL = 1.0
TOL_FLOOR = 1e-14
TOL_CEIL = 0.4
TAIL_DROP_REL = 1e-12
ROW_DROP_REL = 1e-11
DENSE_PATCH_CUTOFF = 2048
SYMMETRY_REPAIR_TOL = 1e-12
_H = 0.5

# debugging switches: skip the lambda estimates (fields stay None); report
# device status words instead of raising
SPECTRAL = True
STRICT = True

_KSTATE = np.dtype([
    ("rs", "f8"), ("pAp", "f8"), ("alpha", "f8"), ("beta", "f8"), ("bnorm", "f8"),
    ("tol_abs", "f8"), ("rnorm", "f8"), ("lam", "f8"), ("ynorm", "f8"), ("res", "f8"),
    ("aux0", "f8"), ("aux1", "f8"), ("it", "i4"), ("done", "i4"), ("converged", "i4"),
    ("max_iter", "i4"), ("breakdown", "i4"), ("pad0", "i4"), ("pad1", "i4"),
    ("pad2", "i4"), ("counter", "u4"), ("pad3", "u4")])


def _clamp_tol(tol):
    return float(min(TOL_CEIL, max(TOL_FLOOR, tol)))


@dataclass(frozen=True)
class LocalizationSchedule:
    """Per-level localization radii (gamblet_fast.py:217-237)."""

    epsilon: float
    q: int
    c_rho: float
    radii: tuple

    def rho(self, k):
        if not 1 <= k <= self.q:
            raise InvalidArgumentError(f"level {k} outside 1..{self.q}")
        return self.radii[k - 1]

    def covers(self, k):
        return self.rho(k) >= 2 ** k

    def subband_tol(self):
        return _clamp_tol(self.epsilon / (2.0 * self.q))


def make_schedule(epsilon, q, c_rho=None, uniform_rho=None):
    """rho_k = ceil(c_rho (k (ln 2 + 1) + ln(1/eps))) clipped into [1, 2^k],
    or one uniform radius (gamblet_fast.py:240-265)."""
    if not 0.0 < epsilon < 1.0:
        raise InvalidArgumentError(f"epsilon must be in (0, 1), got {epsilon}")
    if isinstance(q, bool) or not (isinstance(q, (int, np.integer)) and q >= 1):
        raise InvalidArgumentError(f"q must be a positive integer, got {q!r}")
    c = DEFAULT_C_RHO if c_rho is None else float(c_rho)
    if c <= 0.0:
        raise InvalidArgumentError(f"c_rho must be positive, got {c_rho}")
    if uniform_rho is not None and uniform_rho < 1:
        raise InvalidArgumentError(f"uniform_rho must be >= 1, got {uniform_rho}")
    radii = []
    for k in range(1, q + 1):
        if uniform_rho is not None:
            rho = int(uniform_rho)
        else:
            rho = int(np.ceil(c * (k * (np.log(2.0) + 1.0) + np.log(1.0 / epsilon))))
        radii.append(int(min(max(rho, 1), 2 ** k)))
    return LocalizationSchedule(float(epsilon), int(q), c, tuple(radii))


@dataclass
class FlopCounter:
    """Per-line operation counts, iteration tallies, sizes, wall times
    (gamblet_fast.py:293-364).  Flops are the algorithmic counts of the
    kernels that ran (direct patch factorizations, box-stencil products)."""

    flops: dict = field(default_factory=dict)
    iterations: dict = field(default_factory=dict)
    solves: dict = field(default_factory=dict)
    sizes: dict = field(default_factory=dict)
    seconds: dict = field(default_factory=dict)

    def add(self, label, count):
        self.flops[label] = self.flops.get(label, 0) + int(count)

    def record_iters(self, label, iters):
        self.iterations.setdefault(label, []).extend(np.atleast_1d(iters).tolist())

    def record_solve(self, label, iterations, tol, stages=1):
        self.solves.setdefault(label, []).append((int(iterations), float(tol), int(stages)))

    def record_nnz(self, label, value):
        self.sizes[label] = int(value)

    @contextmanager
    def timer(self, label):
        start = time.perf_counter()
        try:
            yield
        finally:
            if torch.cuda.is_available():
                torch.cuda.current_stream().synchronize()
            self.seconds[label] = self.seconds.get(label, 0.0) + (time.perf_counter() - start)

    @property
    def total_flops(self):
        return int(sum(self.flops.values()))

    def iteration_stats(self):
        out = {}
        for label, its in sorted(self.iterations.items()):
            arr = np.asarray(its, dtype=int)
            values, counts = np.unique(arr, return_counts=True)
            out[label] = {"count": int(arr.size), "min": int(arr.min()),
                          "max": int(arr.max()), "mean": float(arr.mean()),
                          "histogram": {int(v): int(c) for v, c in zip(values, counts)}}
        return out

    def summary(self):
        return {
            "flops": {k: int(v) for k, v in sorted(self.flops.items())},
            "total_flops": self.total_flops,
            "iterations": self.iteration_stats(),
            "nnz": dict(sorted(self.sizes.items())),
            "wall_seconds": {k: round(v, 6) for k, v in sorted(self.seconds.items())},
        }


# ---------------------------------------------------------------------------
# level objects
# ---------------------------------------------------------------------------

class _DevField:
    """Attribute that holds a device operator and reads as the reference's
    host type (scipy CSR / ndarray), materialized once on first access."""

    def __set_name__(self, owner, name):
        self.key = "_" + name

    def __get__(self, obj, objtype=None):
        if obj is None:
            return self
        v = obj.__dict__.get(self.key)
        if isinstance(v, (BoxMatrix, PsiWindows)):
            return v.to_csr()
        if isinstance(v, torch.Tensor):
            host = obj.__dict__.get(self.key + "_host")
            if host is None:
                host = v.cpu().numpy()
                obj.__dict__[self.key + "_host"] = host
            return host
        if callable(v) and not sp.issparse(v):
            v = v()
            obj.__dict__[self.key] = v
        return v

    def __set__(self, obj, value):
        obj.__dict__.pop(self.key + "_host", None)
        obj.__dict__[self.key] = value


class LocalGambletLevel:
    """Level-k output of the localized transform (gamblet_fast.py:268-290).

    psi/stiffness/subband/correction/restriction read as canonical scipy CSR
    and subband_scale as an ndarray; the data stays on the GPU until read.
    """

    psi = _DevField()
    stiffness = _DevField()
    null_w = _DevField()
    subband = _DevField()
    subband_scale = _DevField()
    correction = _DevField()
    restriction = _DevField()

    def __init__(self, k, psi, stiffness, null_w=None, subband=None,
                 subband_scale=None, correction=None, restriction=None,
                 lambda_min_subband=None, lambda_max_subband=None,
                 symmetry_repair=0.0):
        self.k = k
        self.psi = psi
        self.stiffness = stiffness
        self.null_w = null_w
        self.subband = subband
        self.subband_scale = subband_scale
        self.correction = correction
        self.restriction = restriction
        self.lambda_min_subband = lambda_min_subband
        self.lambda_max_subband = lambda_max_subband
        self.symmetry_repair = symmetry_repair
        self.w_variant = None

    def raw(self, name):
        """The stored (device) object behind an attribute."""
        return self.__dict__.get("_" + name)

    def __repr__(self):
        return f"LocalGambletLevel(k={self.k})"


# ---------------------------------------------------------------------------
# per-call device bookkeeping
# ---------------------------------------------------------------------------

class _Ctx:
    """Status blocks and symmetry statistics for one transform, read back once."""

    def __init__(self, n_slots=512):
        self.s = dv.stream()
        self.status = dv.zeros(2 * n_slots, torch.int64)
        self.stats = dv.zeros(2 * n_slots)
        self.dmin = dv.to_dev(np.full(n_slots, np.inf))
        self.n = 0
        self.cap = n_slots
        self.labels = []
        self.repair_of = {}
        self.comm = None  # comm.Comm of a spatially partitioned transform

    def slot(self, kind, what, detail=None):
        if self.n >= self.cap:
            raise RuntimeError("transform context exhausted")
        i = self.n
        self.n += 1
        self.labels.append((i, kind, what, detail))
        return i

    def st(self, i):
        return self.status.data_ptr() + 16 * i

    def sp(self, i):
        return self.stats.data_ptr() + 16 * i

    def dm(self, i):
        return self.dmin.data_ptr() + 8 * i

    def check(self):
        if self.n == 0:
            return
        if not STRICT:
            self._check()
            return
        self._check(raise_=True)

    def _check(self, raise_=False):
        if self.comm is not None and self.comm.world > 1:
            # every rank sees every strip's status words and repair statistics
            self.comm.allreduce(self.status[: 2 * self.n], "max")
            self.comm.allreduce(self.stats[: 2 * self.n], "max")
        elif _STRIPS is not None and _STRIPS.distributed and _STRIPS.world > 1:
            # every rank raises together: a non-SPD patch on one strip poisons
            # the rows the others received from it
            import torch.distributed as dist
            dist.all_reduce(self.status[: 2 * self.n], op=dist.ReduceOp.MAX,
                            group=_STRIPS.group)
            dist.all_reduce(self.stats[: 2 * self.n], op=dist.ReduceOp.MAX,
                            group=_STRIPS.group)
        st = dv.to_host(self.status[: 2 * self.n]).reshape(-1, 2)
        stats = dv.to_host(self.stats[: 2 * self.n]).reshape(-1, 2)
        for i, kind, what, detail in self.labels:
            code, det = int(st[i, 0]), int(st[i, 1])
            if kind == "sym":
                md, ma = stats[i]
                rep = 0.0 if ma == 0.0 else float(md / ma)
                self.repair_of[i] = rep
                if not raise_ and (rep >= SYMMETRY_REPAIR_TOL or code):
                    print(f"[ctx] {what}: repair {rep:.3e} status {code}/{det}")
                    continue
                if rep >= SYMMETRY_REPAIR_TOL:
                    raise NumericalError(
                        f"{what} lost symmetry beyond rounding: relative repair {rep:.3e}")
            if code == 0:
                continue
            if not raise_:
                print(f"[ctx] {kind} {what}: status {code} detail {det}")
                continue
            if kind == "scale":
                raise NumericalError(f"{what}: nonpositive diagonal entry (row {det})")
            if kind == "mass":
                raise NumericalError(
                    f"mass patch {det}: patch matrix is not positive definite")
            if kind == "corr":
                raise NumericalError(
                    f"correction patch {det} at level {detail}: patch matrix is not "
                    "positive definite")
            if kind == "input":
                raise InvalidArgumentError(f"{what}: entry outside the stencil box (row {det})")
            raise NumericalError(f"{what}: device status {code} (detail {det})")


def _blocks_for(nmax, count):
    return int(min(count, 296 if nmax * nmax * 8 > 227 * 1024 else count))


# ---------------------------------------------------------------------------
# Krylov drivers (device CG / power / inverse iteration)
# ---------------------------------------------------------------------------

class _Krylov:
    """Device iteration state + pinned host mirror (reads go through C with
    the GIL released, so side-stream solves never starve the main thread)."""

    def __init__(self, n):
        self.n = n
        nb = nat.query("gb_kstate_bytes")
        self.state = dv.empty(nb, torch.uint8)
        self.host = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        self.part = dv.empty(2 * nat.query("gb_red_blocks"))
        self.dots = dv.empty(4)
        self.hdots = torch.empty(4, dtype=torch.float64, pin_memory=True)
        nat.call("gb_state_reset", dv.ptr(self.state), 0, dv.stream())

    def read(self):
        nat.call("gb_sync_read", dv.ptr(self.state), self.host.data_ptr(),
                 self.host.numel(), dv.stream())
        return self.host.numpy().view(_KSTATE)[0]

    def host_view(self):
        return self.host.numpy().view(_KSTATE)[0]

    def read_dots(self, dots):
        nat.call("gb_sync_read", dv.ptr(dots), self.hdots.data_ptr(), 32, dv.stream())
        return self.hdots.numpy()


class _POp:
    """S B S in slot-major layout (the reference's materialized congruence,
    gamblet_fast.py:123-139) on zero-halo padded vectors: csrc v3 SpMV."""

    def __init__(self, box, s):
        self.L, self.nr, self.w = box.L, box.nr, box.w
        self.n = box.rows
        self.slots = box.slots
        self.Lpad = self.L + 2 * self.w
        self.npad = self.Lpad * self.Lpad * self.nr
        self.layout = 1 if (SYMMETRIC_SPMV and
                            nat.query("gb_sym_supported", self.L, self.nr, self.w)) else 0
        # output vectors of the symmetric band SpMV carry the tiles' spill-over
        # area after the padded vector (gamblets_b200.h, gb_sym_overflow_elems)
        self.vtail = (nat.query("gb_sym_overflow_elems", self.L, self.w)
                      if self.layout == 1 else 0)
        if self.layout == 1:
            self.BsT = dv.empty(nat.query("gb_boxsym_elems", self.L, self.w))
            nat.call("gb_scale_box_symT", self.L, self.w, dv.ptr(box.vals), dv.ptr(s),
                     dv.ptr(self.BsT), dv.stream())
        else:
            self.BsT = dv.empty(nat.query("gb_boxT_elems", self.L, self.nr, self.w))
            nat.call("gb_scale_box_T", self.L, self.nr, self.w, dv.ptr(box.vals), dv.ptr(s),
                     dv.ptr(self.BsT), dv.stream())
        self._box, self._s, self._bj = box, s, None

    def bj_inv(self):
        """Inverses of the 12x12 diagonal blocks (2x2 parents) of S B S
        (symmetrized, fp32: the preconditioner of the block-Jacobi PCG)."""
        if self._bj is None:
            nb = (self.L // 2) ** 2
            self._bj = dv.empty(144 * nb, dtype=torch.float32)
            nat.call("gb_bj_setup", self.L, self.w, dv.ptr(self._box.vals), dv.ptr(self._s),
                     dv.ptr(self._bj), dv.stream())
        return self._bj

    @property
    def stored_slots(self):
        """Matrix slots per row the SpMV streams from HBM (upper half only in
        the symmetric layout)."""
        if self.layout == 1:  # 9 npos + 10 slots per parent of 3 rows
            return (9 * (2 * self.w * self.w + 2 * self.w) + 10) / 3
        return self.slots + (self.slots & 1)

    @property
    def matrix_bytes(self):
        return int(8 * self.n * self.stored_slots)

    @property
    def spmv_bytes(self):
        return 8 * self.n * self.stored_slots + 3 * 8 * self.npad

    def vec(self):
        """A zero padded vector (plus the spill-over tail in the symmetric
        layout, so any vector can be an SpMV output)."""
        return dv.zeros(self.npad + self.vtail)

    def vecs(self, count):
        """`count` zero padded vectors carved out of one allocation (one fill
        kernel; each starts on a 256-byte boundary)."""
        stride = (self.npad + self.vtail + 31) // 32 * 32
        buf = dv.zeros(count * stride)
        return [buf[i * stride:i * stride + self.npad + self.vtail] for i in range(count)]

    def pad(self, x, scale=None):
        out = self.vec()
        nat.call("gb_pad", self.L, self.nr, self.w, dv.ptr(x), dv.ptr(scale), dv.ptr(out),
                 dv.stream())
        return out

    def unpad(self, xp, scale=None):
        out = dv.empty(self.n)
        nat.call("gb_unpad", self.L, self.nr, self.w, dv.ptr(xp), dv.ptr(scale), dv.ptr(out),
                 dv.stream())
        return out

    def apply(self, xp, yp):
        nat.call("gb_tbox_apply", self.L, self.nr, self.w, dv.ptr(self.BsT), dv.ptr(xp),
                 dv.ptr(yp), dv.stream(), self.layout)


def _cg(op, b, rel_tol, x0=None, max_iter=None, kr=None):
    """sparse_core.py:126-165 on the device, padded vectors.  Returns
    (x, iterations, rel_residual, converged, breakdown_iteration, state)."""
    if max_iter is None:
        max_iter = max(200, 2 * op.n)
    max_iter = min(max_iter, MAX_ITER_CAP)
    kr = kr or _Krylov(op.npad)
    st = dv.stream()
    x, r, p, Ap = op.vec(), op.vec(), op.vec(), op.vec()
    nat.call("gb_state_reset", dv.ptr(kr.state), max_iter, st)
    Ax0 = None
    if x0 is not None:
        Ax0 = op.vec()
        op.apply(x0, Ax0)
    nat.call("gb_cg_init", op.npad, dv.ptr(b), dv.ptr(x0), dv.ptr(Ax0), dv.ptr(x),
             dv.ptr(r), dv.ptr(p), float(rel_tol), int(max_iter), dv.ptr(kr.state),
             dv.ptr(kr.part), st)
    nat.call("gb_tcg_solve", op.L, op.nr, op.w, dv.ptr(op.BsT), dv.ptr(x), dv.ptr(r),
             dv.ptr(p), dv.ptr(Ap), dv.ptr(kr.state), dv.ptr(kr.part), kr.host.data_ptr(),
             128, st, op.layout)
    h = kr.host_view()
    rel = float(h["rnorm"] / h["bnorm"]) if h["bnorm"] > 0 else 0.0
    return x, int(h["it"]), rel, bool(h["converged"]), int(h["breakdown"]), h


def _pcg(op, b, rel_tol, x0=None, max_iter=None, kr=None, x0_scale=1.0):
    """Block-Jacobi PCG for the subband systems (2x2-parent 12x12 blocks of
    S B S); same stopping rule as sparse_core.py:161 on the true residual,
    same warm start (x0) semantics as _cg.  Returns the tuple of _cg."""
    if op.nr != 3 or op.L < 2 or op.L % 2:
        return _cg(op, b, rel_tol, x0=x0, max_iter=max_iter, kr=kr)
    if max_iter is None:
        max_iter = max(200, 2 * op.n)
    max_iter = min(max_iter, MAX_ITER_CAP)
    inv = op.bj_inv()
    kr = kr or _Krylov(op.npad)
    st = dv.stream()
    x, r, p, Ap, z = (op.vec() for _ in range(5))
    nat.call("gb_state_reset", dv.ptr(kr.state), max_iter, st)
    Ax0 = None
    if x0 is not None:
        Ax0 = op.vec()
        op.apply(x0, Ax0)
    nat.call("gb_bjcg_init", op.L, op.w, dv.ptr(b), dv.ptr(x0), dv.ptr(Ax0), float(x0_scale),
             dv.ptr(x),
             dv.ptr(r), dv.ptr(p), dv.ptr(z), dv.ptr(inv), float(rel_tol), int(max_iter),
             dv.ptr(kr.state), dv.ptr(kr.part), st)
    nat.call("gb_bjcg_solve", op.L, op.w, dv.ptr(op.BsT), dv.ptr(inv), dv.ptr(x),
             dv.ptr(r), dv.ptr(p), dv.ptr(Ap), dv.ptr(z), dv.ptr(kr.state), dv.ptr(kr.part),
             kr.host.data_ptr(), 128, st, op.layout)
    h = kr.host_view()
    rel = float(h["rnorm"] / h["bnorm"]) if h["bnorm"] > 0 else 0.0
    return x, int(h["it"]), rel, bool(h["converged"]), int(h["breakdown"]), h


_START_VECTORS = {}
_START_LOCK = threading.Lock()


def _start_vectors(n, seed):
    """The two standard-normal start vectors eig_extremes draws from
    default_rng(seed) (sparse_core.py:244, 262), as device arrays.  They are
    a pure function of (n, seed), so they are drawn and uploaded once."""
    key = (n, seed)
    with _START_LOCK:
        v = _START_VECTORS.get(key)
        if v is None:
            rng = np.random.default_rng(seed)
            x1 = rng.standard_normal(n)
            x2 = rng.standard_normal(n)
            v = (dv.to_dev(x1), dv.to_dev(x2))
            torch.cuda.current_stream().synchronize()
            _START_VECTORS[key] = v
    return v


def _eig_extremes_reference(op):
    """The reference's eig_extremes verbatim on the device (power iteration,
    inverse iteration with plain-CG inner solves to 1e-4): the cross-check of
    the Lanczos-moment evaluation at sizes the host cannot run."""
    return _eig_extremes(op, inner_solver="cg")


def _eig_extremes(op, tol=0.1, max_iter=500, seed=24337, inner_solver=None):
    """(lambda_min, lambda_max) of S B S as sparse_core.py:232-278: power
    iteration, then inverse iteration with warm-started inner solves to
    rel_tol max(1e-12, 1e-3 tol); start vectors from numpy default_rng(seed).
    The inner solver is block-Jacobi PCG (SPECTRAL_INNER="pcg", default) or
    the reference's plain CG ("cg"); the estimates agree to the inner
    tolerance.  Returns (lam_min, lam_max, operator applications)."""
    n = op.n
    st = dv.stream()
    x1, x2 = _start_vectors(n, seed)
    kr = _Krylov(op.npad)
    calls = 0
    x = op.pad(x1)
    y = op.vec()
    nat.call("gb_dot2", op.npad, dv.ptr(x), dv.ptr(x), None, dv.ptr(kr.dots),
             dv.ptr(kr.state), dv.ptr(kr.part), st)
    nat.call("gb_scale_by_norm", op.npad, dv.ptr(x), dv.ptr(kr.dots), 0, dv.ptr(x), None, st)
    nat.call("gb_state_reset", dv.ptr(kr.state), max_iter, st)
    nat.call("gb_tpow_solve", op.L, op.nr, op.w, dv.ptr(op.BsT), dv.ptr(x), dv.ptr(y),
             float(tol), dv.ptr(kr.state), dv.ptr(kr.part), kr.host.data_ptr(), 128, st,
             op.layout)
    h = kr.host_view()
    lam_max = float(h["lam"])
    calls += int(h["it"]) + (0 if h["ynorm"] != 0 else 1)

    inner = max(1e-12, 1e-3 * tol)
    x = op.pad(x2)
    nat.call("gb_dot2", op.npad, dv.ptr(x), dv.ptr(x), None, dv.ptr(kr.dots),
             dv.ptr(kr.state), dv.ptr(kr.part), st)
    nat.call("gb_scale_by_norm", op.npad, dv.ptr(x), dv.ptr(kr.dots), 0, dv.ptr(x), None, st)
    lam_min, lam_prev, y_prev = lam_max, np.inf, None
    ykr = _Krylov(op.npad)
    dots = dv.empty(4)
    outer = []
    inner_solver = inner_solver or SPECTRAL_INNER
    for _ in range(max_iter):
        if inner_solver != "cg":  # warm start y_prev / lambda (see gb_level_engine)
            yv, its, _, _, brk, _ = _pcg(op, x, inner, x0=y_prev, kr=ykr,
                                         x0_scale=1.0 / lam_min if y_prev is not None else 1.0)
        else:
            yv, its, _, _, brk, _ = _cg(op, x, inner, x0=y_prev, kr=ykr)
        if brk:
            raise NumericalError(f"CG breakdown at iteration {brk}: p^T A p <= 0 "
                                 "(matrix is not SPD)")
        outer.append(its)
        calls += its + (1 if y_prev is not None else 0)
        nat.call("gb_dot2", op.npad, dv.ptr(yv), dv.ptr(yv), None, dv.ptr(dots),
                 dv.ptr(kr.state), dv.ptr(kr.part), st)
        xn, yp = op.vec(), op.vec()
        nat.call("gb_scale_by_norm", op.npad, dv.ptr(yv), dv.ptr(dots), 0, dv.ptr(xn),
                 dv.ptr(yp), st)
        Ax = op.vec()
        op.apply(xn, Ax)
        calls += 1
        nat.call("gb_dot2", op.npad, dv.ptr(xn), dv.ptr(Ax), None, dv.ptr(dots[2:]),
                 dv.ptr(kr.state), dv.ptr(kr.part), st)
        d = kr.read_dots(dots)
        if d[0] == 0.0:
            raise NumericalError("inverse iteration broke down: A^{-1} x = 0")
        lam_min = float(d[2])
        x, y_prev = xn, yp
        if abs(lam_min - lam_prev) <= 0.5 * tol * abs(lam_min):
            break
        lam_prev = lam_min
    _SPECTRAL_LOG.append({"n": n, "power": int(h["it"]), "inner": outer})
    return lam_min, lam_max, calls


_SPECTRAL_LOG = []
_LANCZOS_DUMP = None

# live timing of the level engine's dual-vector operator passes (bench.py):
# {"n": rows of the level to time, "cap": launches per engine} -> the engine
# records CUDA events on its own stream around its first `cap` dual phase-1
# launches and appends their durations (ms) to ENGINE_TIMING["ms"]
ENGINE_TIMING = None

# pair the lambda estimate and the subband PCG of a level in one engine
# (shared S B S passes); levels the tiled kernels do not cover run them apart
PAIRED_ENGINE = True


# The C level engine on levels below the tile width (L < 64, row-per-thread
# kernels): used when those levels are the critical path, i.e. for q <=
# SMALL_ENGINE_MAX_Q (measured: q=7 17.2 -> 14.5 ms; from q=8 on they are hidden
# behind the finest level and their 64-step Lanczos start only adds GPU work:
# q=9 69.9 -> 73.2 ms, q=10 254.4 -> 257 ms).  Sides below LANCZOS_MIN_L run
# the engine's inverse iteration (PCG inner solves, the host-driven path's
# algorithm): their Krylov spaces are exhausted within the first Lanczos chunk.
LANCZOS_MIN_L = int(os.environ.get("GB_LANCZOS_MIN_L", "8"))
SMALL_ENGINE_MAX_Q = 7


def _engine_ok(op, small=False):
    """Levels the C level engine covers: the tiled / symmetric-band kernels
    need L % 64 == 0; `small`: also the even sides below 64."""
    if op.nr != 3 or op.w > 8:
        return False
    return op.L % 64 == 0 or (small and op.L % 2 == 0 and op.L < 64)


def _paired_level(op, rhs_pad, tol_a, tol=0.1, max_iter=500, seed=24337):
    """Run csrc gb_level_engine: block-Jacobi PCG for (S B S) z = rhs and the
    reference's lambda estimates of S B S (same start vectors as
    sparse_core.eig_extremes), sharing every operator pass."""
    from .engine import LevelEngineArgs
    n = op.n
    st = dv.stream()
    # A: initialised PCG
    inv = op.bj_inv()
    ka = _Krylov(op.npad)
    xa, ra, pa, apa, za, yb, xn, ax, cx, cr, cp, cap, cz = op.vecs(13)
    max_a = min(max(200, 2 * n), MAX_ITER_CAP)
    nat.call("gb_state_reset", dv.ptr(ka.state), max_a, st)
    nat.call("gb_bjcg_init", op.L, op.w, dv.ptr(rhs_pad), None, None, 1.0, dv.ptr(xa), dv.ptr(ra),
             dv.ptr(pa), dv.ptr(za), dv.ptr(inv), float(tol_a), int(max_a), dv.ptr(ka.state),
             dv.ptr(ka.part), st)
    # B: start vectors drawn exactly as eig_extremes draws them
    x1, x2 = _start_vectors(n, seed)
    kb = _Krylov(op.npad)
    xb = op.pad(x1)
    nat.call("gb_dot2", op.npad, dv.ptr(xb), dv.ptr(xb), None, dv.ptr(kb.dots),
             dv.ptr(kb.state), dv.ptr(kb.part), st)
    nat.call("gb_scale_by_norm", op.npad, dv.ptr(xb), dv.ptr(kb.dots), 0, dv.ptr(xb), None, st)
    xs = op.pad(x2)
    nat.call("gb_dot2", op.npad, dv.ptr(xs), dv.ptr(xs), None, dv.ptr(kb.dots),
             dv.ptr(kb.state), dv.ptr(kb.part), st)
    nat.call("gb_scale_by_norm", op.npad, dv.ptr(xs), dv.ptr(kb.dots), 0, dv.ptr(xs), None, st)
    nat.call("gb_state_reset", dv.ptr(kb.state), max_iter, st)
    dots = dv.empty(4)
    args = LevelEngineArgs(
        L=op.L, w=op.w, max_chunk=128, max_outer=max_iter, BsT=dv.ptr(op.BsT),
        inv=dv.ptr(inv), xa=dv.ptr(xa), ra=dv.ptr(ra), pa=dv.ptr(pa), apa=dv.ptr(apa),
        za=dv.ptr(za), sta=dv.ptr(ka.state), parta=dv.ptr(ka.part), hsta=ka.host.data_ptr(),
        xb=dv.ptr(xb), yb=dv.ptr(yb), x2=dv.ptr(xs), xn=dv.ptr(xn), ax=dv.ptr(ax),
        cx=dv.ptr(cx), cr=dv.ptr(cr), cp=dv.ptr(cp), cap=dv.ptr(cap), stb=dv.ptr(kb.state),
        partb=dv.ptr(kb.part), hstb=kb.host.data_ptr(), dots=dv.ptr(dots),
        hdots=kb.hdots.data_ptr(), tol=tol, inner_tol=max(1e-12, 1e-3 * tol),
        inner_max_iter=min(max(200, 2 * n), MAX_ITER_CAP),
        inner_pcg=int(SPECTRAL_INNER != "cg"), cz=dv.ptr(cz), layout=op.layout)
    if SPECTRAL_INNER == "lanczos" and op.L >= LANCZOS_MIN_L:
        cap = int(min(n, LANCZOS_CAP))
        lz = dv.empty(2 * cap)
        hlz = torch.empty(2 * cap, dtype=torch.float64, pin_memory=True)
        args.spectral_mode = 1
        args.lz_cap = cap
        args.lz = dv.ptr(lz)
        args.hlz = hlz.data_ptr()
        args.lz_tol = LANCZOS_TOL
    timing = ENGINE_TIMING
    ev_ms = None
    if timing is not None and timing.get("n") == n:
        ev_ms = torch.zeros(int(timing["cap"]), dtype=torch.float32, pin_memory=True)
        args.ev_cap = int(timing["cap"])
        args.ev_ms = ev_ms.data_ptr()
    nat.call("gb_level_engine", nat.ctypes.byref(args), st)
    if ev_ms is not None:
        timing.setdefault("ms", []).extend(ev_ms[:args.ev_n].tolist())
    if args.breakdown == -2:
        raise NumericalError(f"Lanczos moments of S B S at n={n}: "
                             + ("nonpositive pivot (matrix is not SPD)" if args.lz_rc == 2
                                else "evaluation failed"))
    if args.breakdown > 0:
        raise NumericalError(f"CG breakdown at iteration {args.breakdown}: p^T A p <= 0 "
                             "(matrix is not SPD)")
    if args.breakdown < 0:
        raise NumericalError("inverse iteration broke down: A^{-1} x = 0")
    h = ka.host_view()
    if args.spectral_mode == 1:
        _SPECTRAL_LOG.append({"n": n, "power": int(args.power_its), "outer": int(args.n_outer),
                              "lanczos": int(args.lz_its)})
        if _LANCZOS_DUMP is not None:  # tools/lanczos_convergence.py
            _LANCZOS_DUMP.append((n, hlz[:2 * int(args.lz_its)].clone().numpy()))
    else:
        _SPECTRAL_LOG.append({"n": n, "power": int(args.power_its),
                              "inner": [int(args.inner_its[i])
                                        for i in range(min(args.n_outer, 64))]})
    rel = float(h["rnorm"] / h["bnorm"]) if h["bnorm"] > 0 else 0.0
    # algorithmic HBM bytes of the engine's operator passes: the stored band
    # once per phase-1 launch plus x/y of each vector it carries
    vec = 2 * 8 * op.npad
    dv.Prof.add_work("level_engine", nbytes=args.n_dual * (op.matrix_bytes + 2 * vec)
                     + args.n_single * (op.matrix_bytes + vec))
    return {"x": xa, "its": int(h["it"]), "rel": rel, "conv": bool(h["converged"]),
            "brk": int(h["breakdown"]), "lam_min": float(args.lam_min),
            "lam_max": float(args.lam_max), "calls": int(args.calls),
            "passes": (int(args.n_dual), int(args.n_single))}

# The level tasks (lambda estimates + subband solve of one level) run on side
# streams so they overlap the setup of the coarser levels on the main stream:
# a pool of worker threads, one stream per LEVEL, same priority as the main
# stream (measured at q=10: 3 workers on high-priority streams 258 ms, 6
# workers at equal priority 251 ms, tools/tune_step.py)
SPECTRAL_WORKERS = int(__import__("os").environ.get("GB_SPECTRAL_WORKERS", "6"))
SPECTRAL_PRIORITY = int(__import__("os").environ.get("GB_SPECTRAL_PRIORITY", "0"))
# lean transforms (q >= 12, within ~20 % of the HBM capacity): three levels in
# flight on per-worker high-priority streams, the setting the q=12 line was
# measured with
LEAN_WORKERS = 3
LEAN_PRIORITY = -1
_LEAN_SLOTS = threading.BoundedSemaphore(LEAN_WORKERS)
# symmetric band Krylov copy (csrc/gb_symspmv.cuh): only the upper 3x3 blocks
# of S B S are streamed, the lower half is applied from the same registers
# (scatter through shared memory) -- half the HBM bytes of the full box
SYMMETRIC_SPMV = True
# safety cap on Krylov iterations (the reference's max(200, 2n) is kept below
# it; converging solves here need < 2000)
MAX_ITER_CAP = 100000
# inner solver of the inverse iteration for lambda_min: "pcg" (block-Jacobi,
# the subband preconditioner) or "cg" (the reference's unpreconditioned CG).
# lambda_min feeds only the reported conditioning (tight mode has no cheap
# copy), and both stop at the same relative residual.
#
# "lanczos" (default): on the levels the paired engine covers, lambda_min is
# the reference's inverse-iteration sequence evaluated from the Lanczos
# moments of its start vector (csrc/gb_lanczos.h) -- the iteration with exact
# inner solves, same stopping test; the Lanczos passes ride on the subband
# PCG's operator passes.  Smaller levels run the inverse iteration with PCG.
SPECTRAL_INNER = "lanczos"
LANCZOS_CAP = 4096
# bound on the estimated remaining relative error of the emulated lambda_min
# at which the Lanczos sequence stops (gb_lanczos.h lanczos_check: every 32
# steps the estimate is evaluated on T_m, T_{m-16}, T_{m-32} and the geometric
# tail of the differences compared with this).  At q=10 the sequence stops at
# 352 steps, 3e-5 from the converged value; the reference's own inner solves
# (rel_tol 1e-4) move its estimate by 3e-4
LANCZOS_TOL = 1e-4


class _LevelTasks:
    """Per-level device work that depends only on that level's operator: the
    lambda estimates of S B^(k) S (sparse_core.eig_extremes) and, inside
    fast_solve, the subband solve and increment of level k.  Each task runs
    on a worker thread with its own high-priority stream (ordered after the
    operator by an event) so the HBM-bound Krylov work of level k overlaps
    the FP64-bound setup of the coarser levels on the main stream."""

    _pool = None
    _local = threading.local()

    def __init__(self, solver=None):
        if _LevelTasks._pool is None:
            _LevelTasks._pool = concurrent.futures.ThreadPoolExecutor(
                max_workers=SPECTRAL_WORKERS, thread_name_prefix="gb-level")
        self.futures = []
        self.solver = solver
        self.small_engine = solver is not None and solver.tree.q <= SMALL_ENGINE_MAX_Q

    _level_streams = {}
    _level_streams_lock = threading.Lock()

    @classmethod
    def _stream(cls, k=None):
        """The stream of a level task.  Retained transforms give every level
        its own stream: the caching allocator keeps one block pool per
        stream, so the same level on the same stream in every step replays
        the same allocations and a steady-state step makes no cudaMalloc
        (with a stream per worker thread, whichever thread picked a level up
        grew its pool: tens of new segments per step and a 100+ ms stall now
        and then).  Lean transforms (q >= 12, memory bound) keep one stream
        per worker so the levels share the workers' pools."""
        torch.cuda.set_device(dv.device())
        if k is not None:
            key = (dv.device().index, int(k), SPECTRAL_PRIORITY)
            with cls._level_streams_lock:
                st = cls._level_streams.get(key)
                if st is None:
                    st = torch.cuda.Stream(device=dv.device(), priority=SPECTRAL_PRIORITY)
                    cls._level_streams[key] = st
            return st
        st = getattr(cls._local, "stream", None)
        if st is None:
            st = torch.cuda.Stream(device=dv.device(), priority=LEAN_PRIORITY)
            cls._local.stream = st
        return st

    def submit(self, level, op, k, g=None):
        ev = torch.cuda.Event()
        ev.record()
        # the increment psi^(k)T W^T w^(k) holds its own reference to psi^(k),
        # so a lean transform may drop it from the level meanwhile
        psi = level.raw("psi") if self.solver is not None else None
        level._krylov_op = op  # the task's operator (a lean level drops B meanwhile)
        self.futures.append(self._pool.submit(self._run, level, op, k, g, ev, psi))

    def _run(self, level, op, k, g, ev, psi=None):
        if getattr(level, "_lean", False):
            with _LEAN_SLOTS:  # memory bound: at most LEAN_WORKERS levels in flight
                return self._run_on(self._stream(None), level, op, k, g, ev, psi)
        return self._run_on(self._stream(k), level, op, k, g, ev, psi)

    def _run_on(self, st, level, op, k, g, ev, psi=None):
        calls = 0
        with torch.cuda.stream(st):
            st.wait_event(ev)
            if g is not None:
                g.record_stream(st)  # main-stream tensor read on this stream
            if (SPECTRAL and PAIRED_ENGINE and self.solver is not None and g is not None
                    and _engine_ok(op, self.small_engine)):
                box = {}

                def run_engine(op_, rhs_pad, tol):
                    with dv.phase("level_engine"):
                        out = _paired_level(op_, rhs_pad, tol)
                    box.update(out)
                    return out["x"], out["its"], out["rel"], out["conv"], out["brk"]

                self.solver.subband(k, g, pipelined=True, engine=run_engine, psi=psi)
                del psi
                level.lambda_min_subband = box["lam_min"]
                level.lambda_max_subband = box["lam_max"]
                done = torch.cuda.Event()
                done.record(st)
                info = (op.n, op.slots, op.spmv_bytes)
                level._krylov_op = None
                if getattr(level, "_lean", False) and not getattr(level, "_keep_op", False):
                    level._op = None  # the operator copy is not retained
                return box["calls"], info, done, True
            if SPECTRAL:
                with dv.phase("spectral"):
                    lam_min, lam_max, calls = _eig_extremes(op)
                level.lambda_min_subband = lam_min
                level.lambda_max_subband = lam_max
            if self.solver is not None and g is not None:
                self.solver.subband(k, g, pipelined=True, psi=psi)
            del psi
            done = torch.cuda.Event()
            done.record(st)
        info = (op.n, op.slots, op.spmv_bytes)
        level._krylov_op = None
        if getattr(level, "_lean", False):
            level._op = None
        return calls, info, done, False

    def join(self, counter):
        futs, self.futures = self.futures, []
        err = None
        for f in futs:
            try:
                calls, (op_n, op_slots, op_bytes), done, engine = f.result()
            except Exception as e:  # keep joining, re-raise the first error
                err = err or e
                continue
            torch.cuda.current_stream().wait_event(done)
            counter.add("spectral", 2 * op_n * op_slots * calls)
            if not engine:  # the engine books its own passes ("level_engine")
                dv.Prof.add_work("spectral", nbytes=calls * op_bytes)
        if err is not None:
            raise err


# ---------------------------------------------------------------------------
# transform
# ---------------------------------------------------------------------------

def _canon(mat):
    if isinstance(mat, (dv.DeviceCSR, BoxMatrix)) or is_canonical_csr(mat):
        return mat
    return as_csr(mat)


def _box_dev(level, name, L, ctx):
    v = level.raw(name)
    if isinstance(v, BoxMatrix):
        return v
    if v is None:
        raise InvalidArgumentError(f"level {level.k} has no {name}")
    mat = v if is_canonical_csr(v) else as_csr(v)
    if mat.shape != (L * L, L * L):
        raise InvalidArgumentError(f"{name} shape {mat.shape} does not match level side {L}")
    box, status = dv.csr_to_box(mat, L)
    return box


def _psi_dev(level, n, L):
    v = level.raw("psi")
    if v is None or isinstance(v, PsiWindows):
        return v
    return dv.csr_to_psi(v, n, L)


# test-only switch: the per-entry gather kernel for A^(q) = psi A psi^T (same
# sums as the default plane-major kernel; tests/test_gpu_parity.py compares them)
_GALERKIN_GATHER = False


def _level_q(M, A, tree, rho, ctx, counter):
    """Alg. 2 lines 2a/3/5: psi^(q) and A^(q) (gamblet_fast.py:464-498, 650-665)."""
    q = tree.q
    n = 1 << q
    N = n * n
    s = ctx.s
    if M.shape != (N, N):
        raise InvalidArgumentError(f"mass shape {M.shape} does not match q={q}")
    if A.shape != (N, N):
        raise InvalidArgumentError(f"stiffness shape {A.shape} does not match q={q}")
    with dv.phase("input_to_box"):
        # device-assembled inputs (grid_fem.assemble_*(device=True)) are boxes
        Mb = M if isinstance(M, BoxMatrix) else dv.csr_to_box(_canon(M), n)[0]
    sM = dv.empty(N)
    nat.call("gb_box_scale", N, 1, Mb.w, dv.ptr(Mb.vals), dv.ptr(sM),
             ctx.st(ctx.slot("scale", "mass")), s)
    rho = int(min(rho, n - 1))
    lo, hi = -rho, rho
    wd = PsiWindows.window(n, lo, hi)
    psi = dv.empty(N * wd * wd)
    nmax = (2 * rho + 1) ** 2
    with dv.phase("mass_patches"):
        _mass_patches(n, Mb, sM, rho, wd, psi, ctx.st(ctx.slot("mass", "mass")), s)
    # algorithmic work per phase (the aggregate roofline of bench.py): patch
    # factor/solve flops, box values read once and written once
    dv.Prof.add_work("mass_patches", flops=_patch_flops(n, rho, 1),
                     nbytes=8 * N * (dv.box_slots(Mb.w, 1) + wd * wd))
    # the stiffness is needed only after the mass patches: a host-resident A
    # is uploaded on a copy stream while they run
    A = _canon(A)
    if not isinstance(A, (dv.DeviceCSR, BoxMatrix)):
        cs = _copy_stream()
        with torch.cuda.stream(cs):
            A = dv.DeviceCSR.from_scipy(A)
            ev = torch.cuda.Event()
            ev.record(cs)
        torch.cuda.current_stream().wait_event(ev)
        for t in (A.indptr, A.indices, A.data):
            t.record_stream(torch.cuda.current_stream())
    Ab = A if isinstance(A, BoxMatrix) else dv.csr_to_box(A, n)[0]
    wX = min(rho + Ab.w, n - 1)
    X = dv.empty(N * dv.box_slots(wX, 1))
    wR = min(wX + rho, n - 1)
    raw = dv.empty(N * dv.box_slots(wR, 1))
    # A^(q)'s own buffer doubles as the transposes' workspace (N (wd^2 + SX)
    # <= N SR doubles): no extra allocation inside the step
    Aq = dv.empty(N * dv.box_slots(wR, 1))
    with dv.phase("psi_A_psiT"):
        nat.call("gb_psi_stencil", n, lo, wd, rho, dv.ptr(psi), Ab.w, dv.ptr(Ab.vals), wX,
                 dv.ptr(X), s)
        if _GALERKIN_GATHER:  # the per-entry gather form (same sums)
            nat.call("gb_psi_galerkin", n, lo, wd, rho, dv.ptr(psi), wX, dv.ptr(X), wR,
                     dv.ptr(raw), s)
        else:  # coalesced form over plane-major copies of psi and X
            need = nat.query("gb_psi_galerkin_workspace", n, wd, wX)
            work = Aq if Aq.numel() * 8 >= need else dv.empty(need // 8)
            nat.call("gb_psi_galerkin_t", n, lo, wd, rho, dv.ptr(psi), wX, dv.ptr(X), wR,
                     dv.ptr(raw), dv.ptr(work), s)
            del work
    del X
    i = ctx.slot("sym", "A^(q),loc")
    with dv.phase("sym_drop"):
        nat.call("gb_box_diag_min", N, 1, wR, dv.ptr(raw), ctx.dm(i), s)
        nat.call("gb_box_sym_drop", n, 1, wR, dv.ptr(raw), dv.ptr(Aq), ctx.dm(i),
                 ctx.sp(i), s)
    dv.Prof.add_work("psi_A_psiT", flops=2 * N * dv.box_slots(wX, 1) * 9
                     + 2 * N * dv.box_slots(wR, 1) * nmax,
                     nbytes=8 * N * (wd * wd + dv.box_slots(Ab.w, 1) + dv.box_slots(wR, 1)))
    dv.Prof.add_work("sym_drop", nbytes=16 * N * dv.box_slots(wR, 1))
    # flop model: patch Cholesky + two triangular solves; box products
    counter.add("line2a", _patch_flops(n, rho, 1))
    counter.add("line3", N * wd * wd)
    counter.add("line5", 2 * N * dv.box_slots(wX, 1) * 9 + 2 * N * dv.box_slots(wR, 1) * nmax)
    counter.add("scaling", 2 * N * dv.box_slots(Mb.w, 1) + N + 3 * N * dv.box_slots(wR, 1))
    return (PsiWindows(psi, n, n, lo, hi), BoxMatrix(Aq, n, 1, wR, 1), i)


# row-strip partition of the patch solves (partition.Strips; None = whole
# levels): the multi-GPU building block, DESIGN.md section 6
_STRIPS = None


def _mass_patches(n, Mb, sM, rho, wd, psi, status_ptr, s):
    """K1 on the pre-scaled S M S box: the shared-memory tiled DMMA Cholesky
    (v2); patches larger than shared memory use the global-workspace v1."""
    if _STRIPS is not None:
        try:
            part.run_strips(_STRIPS, n, n * wd * wd, psi, lambda r0, r1: nat.call(
                "gb_mass_patches_rows", n, Mb.w, dv.ptr(Mb.vals), dv.ptr(sM), rho, wd,
                dv.ptr(psi), status_ptr, r0, r1, s))
            return
        except InvalidArgumentError:  # no strip kernel for this patch: whole level
            pass
    try:
        nat.call("gb_mass_patches_v2", n, Mb.w, dv.ptr(Mb.vals), dv.ptr(sM), rho, wd,
                 dv.ptr(psi), status_ptr, s)
        return
    except InvalidArgumentError:
        pass
    nmax = (2 * rho + 1) ** 2
    blocks = _blocks_for(nmax, n * n)
    wsb = nat.query("gb_mass_patch_workspace", rho, blocks)
    ws = dv.empty(wsb // 8) if wsb else None
    nat.call("gb_mass_patches", n, Mb.w, dv.ptr(Mb.vals), dv.ptr(sM), rho, wd, dv.ptr(psi),
             status_ptr, dv.ptr(ws), blocks, s)


def _correction_ws(Lp, rho, r0, r1):
    """Caller-owned L scratch of the v3 correction-patch kernel (allocated from
    the stream-ordered caching allocator, so concurrent transforms on
    different streams never share it)."""
    nb = nat.query("gb_correction_patches_workspace", Lp, rho, r0, r1)
    return (dv.empty((nb + 7) // 8), nb) if nb else (None, 0)


def _correction_patches(Lp, B, op, sB, Gv, rho, Dt, status_ptr, s):
    """K4: v3 (left-looking tiled DMMA Cholesky on S B S, L streamed through
    an L2-resident scratch) when the patch fits, else the global-workspace v1."""
    if _STRIPS is not None:
        try:
            def strip(r0, r1):
                ws, nb = _correction_ws(Lp, rho, r0, r1)
                nat.call("gb_correction_patches_rows", Lp, B.w, dv.ptr(B.vals), dv.ptr(sB),
                         B.w, dv.ptr(Gv), rho, dv.ptr(Dt), status_ptr, r0, r1, dv.ptr(ws),
                         nb, s)
            part.run_strips(_STRIPS, Lp, Lp * dv.box_slots(rho, 3), Dt, strip)
            return
        except InvalidArgumentError:  # no strip kernel for this patch: whole level
            pass
    try:
        ws, nb = _correction_ws(Lp, rho, 0, Lp)
        nat.call("gb_correction_patches_v2", Lp, B.w, dv.ptr(B.vals), dv.ptr(sB), B.w,
                 dv.ptr(Gv), rho, dv.ptr(Dt), status_ptr, dv.ptr(ws), nb, s)
        return
    except InvalidArgumentError:
        pass
    nmax = 3 * (2 * rho + 1) ** 2
    blocks = _blocks_for(nmax, Lp * Lp)
    wsb = nat.query("gb_correction_workspace", rho, blocks)
    ws = dv.empty(wsb // 8) if wsb else None
    nat.call("gb_correction_patches", Lp, B.w, dv.ptr(B.vals), dv.ptr(sB), B.w, dv.ptr(Gv),
             rho, dv.ptr(Dt), status_ptr, dv.ptr(ws), blocks, s)


_COPY_STREAM = {}


def _copy_stream():
    dev = dv.device()
    if dev not in _COPY_STREAM:
        _COPY_STREAM[dev] = torch.cuda.Stream(device=dev)
    return _COPY_STREAM[dev]


def _patch_flops(L, rho, comps):
    """sum over clipped patches of m^3/3 + 2 m^2 (m = comps * patch size)."""
    ext = np.minimum(np.arange(L), rho) + np.minimum(L - 1 - np.arange(L), rho) + 1
    m = comps * np.multiply.outer(ext, ext).ravel().astype(np.float64)
    return int((m ** 3 / 3.0 + 2.0 * m * m).sum())


def local_mass_inverse(M, tree, rho, tol, counter=None, dense_cutoff=DENSE_PATCH_CUTOFF):
    """Finest-level basis rows by patchwise mass inversion
    (gamblet_fast.py:464-498); returns psi^(q) as canonical CSR."""
    q = tree.q
    N = 4 ** q
    if M.shape != (N, N):
        raise InvalidArgumentError(f"mass shape {M.shape} does not match q={q}")
    counter = counter if counter is not None else FlopCounter()
    ctx = _Ctx()
    n = 1 << q
    Mb, _ = dv.csr_to_box(_canon(M), n)
    sM = dv.empty(N)
    nat.call("gb_box_scale", N, 1, Mb.w, dv.ptr(Mb.vals), dv.ptr(sM),
             ctx.st(ctx.slot("scale", "mass")), ctx.s)
    rho = int(min(int(np.floor(rho)), n - 1))
    wd = PsiWindows.window(n, -rho, rho)
    psi = dv.empty(N * wd * wd)
    _mass_patches(n, Mb, sM, rho, wd, psi, ctx.st(ctx.slot("mass", "mass")), ctx.s)
    ctx.check()
    counter.add("line2a", _patch_flops(n, rho, 1))
    return PsiWindows(psi, n, n, -rho, rho).to_csr()


def local_level_step(level, tree, schedule, w_variant="orthonormal", c_tol=DEFAULT_C_TOL,
                     counter=None, dense_cutoff=DENSE_PATCH_CUTOFF, _ctx=None, _spool=None,
                     _g=None, _lean=False, _cols=None):
    """One localized downward step k -> k-1 (gamblet_fast.py:501-632).
    Mutates `level` (W, B, s_B, D, R, lambdas, repair) and returns level k-1.

    _cols = (f0, f1, comm): column strips of psi (gamblet_dist.py, the
    replicated coarse levels of a partitioned transform): this rank holds and
    computes only the window points of psi^(k), W psi and psi^(k-1) whose fine
    row lies in [f0, f1); the row maxima of the tail drop are max-reduced
    over the ranks."""
    k = level.k
    if k < 2:
        raise InvalidArgumentError(f"level step needs k >= 2, got k={k}")
    counter = counter if counter is not None else FlopCounter()
    ctx = _ctx if _ctx is not None else _Ctx()
    s = ctx.s
    q = schedule.q
    n = 1 << q
    Lk, Lp = 1 << k, 1 << (k - 1)
    tmpl = w_template(w_variant)
    w12 = tmpl.ctypes.data
    Ab = _box_dev(level, "stiffness", Lk, ctx)
    psiw = _psi_dev(level, n, Lk)
    wA = Ab.w
    wB = min((wA + 1) // 2, Lp - 1)
    rho = int(min(schedule.rho(k - 1), Lp - 1))
    P = Lp * Lp
    J = 3 * P

    with counter.timer(f"level {k}"):
        # K3: B (sym + dead-tail drop fused), G, P A P^T
        ib = ctx.slot("sym", f"B^({k}),loc")
        bdiag = dv.empty(J)
        Bv = dv.empty(J * dv.box_slots(wB, 3))
        Gv = dv.empty(J * dv.box_slots(wB, 1))
        PAPt = dv.empty(P * dv.box_slots(wB, 1))
        sB = dv.empty(J)
        with dv.phase("level_blocks"):
            nat.call("gb_level_diag", Lk, wA, dv.ptr(Ab.vals), w12, dv.ptr(bdiag),
                     ctx.dm(ib), s)
            nat.call("gb_level_blocks", Lk, wA, dv.ptr(Ab.vals), w12, wB, dv.ptr(bdiag),
                     ctx.dm(ib), dv.ptr(Bv), dv.ptr(Gv), dv.ptr(PAPt), ctx.sp(ib), s)
            nat.call("gb_box_scale", J, 3, wB, dv.ptr(Bv), dv.ptr(sB),
                     ctx.st(ctx.slot("scale", f"B^({k}),loc")), s)
        del bdiag
        if _lean:  # A^(k) is consumed: the lean transform does not retain it
            Ab = None
            level.stiffness = None
        B = BoxMatrix(Bv, Lp, 3, wB, 3)
        dv.Prof.add_work("level_blocks", flops=2 * J * dv.box_slots(wB, 3) * 16,
                         nbytes=8 * (Lk * Lk * dv.box_slots(wA, 1) + J * dv.box_slots(wB, 3)
                                     + J * dv.box_slots(wB, 1) + P * dv.box_slots(wB, 1)))
        counter.add("line7", 2 * J * dv.box_slots(wB, 3) * 16)
        counter.add("scaling", 2 * J * dv.box_slots(wB, 3) + J)

        # K7: spectral extremes of S B S (gamblet_fast.py:531-534)
        with dv.phase("level_blocks"):
            op = _POp(B, sB)
            if _lean:  # preconditioner now, so the Krylov copy does not need B
                op.bj_inv()
                op._box = None
        level._op = op
        dv.Prof.add_work("level_blocks", nbytes=8 * J * dv.box_slots(wB, 3) + op.matrix_bytes)
        level._lean = _lean
        level._keep_op = k == q  # the finest operator stays for instrumentation
        level.subband = B
        level.subband_scale = sB
        level.w_variant = w_variant
        spool = _spool if _spool is not None else _LevelTasks()
        spool.submit(level, op, k, _g)

        # K4: correction patches -> D^T with the row-tail trim fused
        Dt = dv.empty(P * dv.box_slots(rho, 3))
        with dv.phase("correction_patches"):
            _correction_patches(Lp, B, op, sB, Gv, rho, Dt,
                                ctx.st(ctx.slot("corr", f"level {k}", detail=k)), s)
        dv.Prof.add_work("correction_patches", flops=_patch_flops(Lp, rho, 3),
                         nbytes=8 * (J * dv.box_slots(wB, 3) + J * dv.box_slots(wB, 1)
                                     + P * dv.box_slots(rho, 3)))
        counter.add("line11", _patch_flops(Lp, rho, 3))
        counter.record_solve(f"line11 level {k}", 1, 0.0, stages=1)

        # K6: R, split triple product
        Rv = dv.empty(P * dv.box_slots(rho, 4))
        with dv.phase("restriction"):
            nat.call("gb_restriction", Lp, rho, dv.ptr(Dt), w12, dv.ptr(Rv), s)
        counter.add("line12", 2 * P * dv.box_slots(rho, 4) * 3)
        dv.Prof.add_work("restriction", nbytes=8 * P * (dv.box_slots(rho, 3)
                                                        + dv.box_slots(rho, 4)))
        wBD = min(wB + rho, Lp - 1)
        BD = dv.empty(J * dv.box_slots(wBD, 1))
        wGD = min(wB + rho, Lp - 1)
        GtD = dv.empty(P * dv.box_slots(wGD, 1))
        wA2 = min(2 * rho + wB, Lp - 1)
        raw = dv.empty(P * dv.box_slots(wA2, 1))
        with dv.phase("triple_product"):
            nat.call("gb_bd", Lp, wB, dv.ptr(Bv), rho, dv.ptr(Dt), wBD, dv.ptr(BD), s)
            nat.call("gb_gtd", Lp, wB, dv.ptr(Gv), rho, dv.ptr(Dt), wGD, dv.ptr(GtD), s)
            nat.call("gb_coarse_raw", Lp, wB, dv.ptr(PAPt), wGD, dv.ptr(GtD), rho,
                     dv.ptr(Dt), wBD, dv.ptr(BD), wA2, dv.ptr(raw), s)
        del BD, GtD, PAPt, Gv
        ia = ctx.slot("sym", f"A^({k - 1}),loc")
        An = dv.empty(P * dv.box_slots(wA2, 1))
        with dv.phase("sym_drop"):
            nat.call("gb_box_diag_min", P, 1, wA2, dv.ptr(raw), ctx.dm(ia), s)
            nat.call("gb_box_sym_drop", Lp, 1, wA2, dv.ptr(raw), dv.ptr(An), ctx.dm(ia),
                     ctx.sp(ia), s)
        del raw
        nb = 3 * (2 * min(rho, wB) + 1) ** 2
        counter.add("line13", 2 * J * dv.box_slots(wBD, 1) * nb
                    + 2 * P * dv.box_slots(wA2, 1) * nb + 2 * P * dv.box_slots(wGD, 1) * nb)
        dv.Prof.add_work("triple_product",
                         flops=2 * J * dv.box_slots(wBD, 1) * nb
                         + 2 * P * dv.box_slots(wA2, 1) * nb + 2 * P * dv.box_slots(wGD, 1) * nb,
                         nbytes=8 * (J * dv.box_slots(wB, 3) + J * dv.box_slots(wB, 1)
                                     + P * dv.box_slots(wB, 1) + P * dv.box_slots(rho, 3)
                                     + P * dv.box_slots(wA2, 1)))
        dv.Prof.add_work("sym_drop", nbytes=16 * P * dv.box_slots(wA2, 1))

        # psi^(k-1) = drop_row(0.25 P psi + D^T (W psi))
        psin = None
        if psiw is not None:
            h = n // Lk
            lo, hi, wd = psiw.lo, psiw.hi, psiw.wd
            wdw = min(hi - lo + 1 + h, n)
            Wpsi = dv.empty(J * wdw * wdw)
            lo2, hi2 = -2 * rho * h + lo, (2 * rho + 1) * h + hi
            wd2 = PsiWindows.window(n, lo2, hi2)
            pv = dv.empty(P * wd2 * wd2)
            with dv.phase("psi_next"):
                rmax = dv.empty(P)
                strips_done = False
                if _cols is not None:
                    cf0, cf1, ccomm = _cols
                    nat.call("gb_wpsi_rows", n, Lk, lo, wd, w12, dv.ptr(psiw.vals), wdw,
                             dv.ptr(Wpsi), 0, Lp, cf0, cf1, s)
                    nat.call("gb_psi_next_raw_rows", n, Lk, lo, hi, wd, dv.ptr(psiw.vals), wdw,
                             dv.ptr(Wpsi), rho, dv.ptr(Dt), lo2, wd2, dv.ptr(pv), dv.ptr(rmax),
                             0, Lp, cf0, cf1, s)
                    ccomm.allreduce(rmax, "max")
                    nat.call("gb_psi_drop_rows", n, Lp, lo2, wd2, dv.ptr(pv), dv.ptr(rmax),
                             0, Lp, cf0, cf1, s)
                    strips_done = True
                else:
                    nat.call("gb_wpsi", n, Lk, lo, wd, w12, dv.ptr(psiw.vals), wdw,
                             dv.ptr(Wpsi), s)
                if _STRIPS is not None and not strips_done:  # row strips of the parent grid (multi-GPU block)
                    try:
                        part.run_strips(_STRIPS, Lp, Lp * wd2 * wd2, pv, lambda r0, r1: nat.call(
                            "gb_psi_next_rows", n, Lk, lo, hi, wd, dv.ptr(psiw.vals), wdw,
                            dv.ptr(Wpsi), rho, dv.ptr(Dt), lo2, wd2, dv.ptr(pv),
                            dv.ptr(rmax), r0, r1, s))
                        strips_done = True
                    except InvalidArgumentError:  # per-entry products mode: whole level
                        pass
                if not strips_done:
                    nat.call("gb_psi_next", n, Lk, lo, hi, wd, dv.ptr(psiw.vals), wdw,
                             dv.ptr(Wpsi), rho, dv.ptr(Dt), lo2, wd2, dv.ptr(pv),
                             dv.ptr(rmax), s)
            del Wpsi, rmax
            psin = PsiWindows(pv, n, Lp, lo2, hi2)
            if _lean:  # psi^(k) lives on only in the level-k increment task
                psiw = None
                level.psi = None
            counter.add("line14", 2 * P * wd2 * wd2 * 3 * (2 * rho + 1) ** 2 // 4
                        + 2 * J * wdw * wdw * 4)
            dv.Prof.add_work("psi_next", flops=2 * P * wd2 * wd2 * 3 * (2 * rho + 1) ** 2 // 4,
                             nbytes=8 * (Lk * Lk * wd * wd + P * dv.box_slots(rho, 3)
                                         + P * wd2 * wd2))

    level.null_w = (lambda tree=tree, k=k, v=w_variant: tree.null_basis(k, v))
    if _lean:  # B^(k), D^(k,k-1) consumed; R kept until g^(k-1) = R g^(k)
        level.subband = None
        del Dt, B, Bv
    else:
        level.correction = BoxMatrix(Dt, Lp, 1, rho, 3, kind=EXP_TDT)
    level.restriction = BoxMatrix(Rv, Lp, 1, rho, 4, kind=EXP_CHILD)
    level._repair_slot_b = ib
    nxt = LocalGambletLevel(k - 1, psin, BoxMatrix(An, Lp, 1, wA2, 1))
    nxt._repair_slot_a = ia
    if _spool is None:
        spool.join(counter)
    if _ctx is None:
        ctx.check()
        level.symmetry_repair = max(level.symmetry_repair, ctx.repair_of.get(ib, 0.0))
        nxt.symmetry_repair = ctx.repair_of.get(ia, 0.0)
    return nxt


def fast_transform(M, A, tree, schedule, w_variant="orthonormal", c_tol=DEFAULT_C_TOL,
                   counter=None, dense_cutoff=DENSE_PATCH_CUTOFF):
    """Load-independent phase, levels q..1 (gamblet_fast.py:635-674).
    Returns (levels, counter); all operators stay on the device."""
    levels, counter, _ = _transform(M, A, tree, schedule, w_variant=w_variant, c_tol=c_tol,
                                    counter=counter, dense_cutoff=dense_cutoff)
    return levels, counter


def _transform(M, A, tree, schedule, w_variant="orthonormal", c_tol=DEFAULT_C_TOL,
               counter=None, dense_cutoff=DENSE_PATCH_CUTOFF, _load=None, _lean=False,
               _keep_below=0):
    """fast_transform, optionally with the nodal-load solve pipelined into it
    (_load = (g_device, records)).  Returns (levels, counter, solved), solved =
    (parts, U1) of the pipelined solve or None."""
    counter = counter if counter is not None else FlopCounter()
    q = tree.q
    if schedule.q != q:
        raise InvalidArgumentError(f"schedule q={schedule.q} does not match tree q={q}")
    w_template(w_variant)
    ctx = _Ctx()
    with counter.timer("level q init"):
        psi, Aq, ia = _level_q(M, A, tree, schedule.rho(q), ctx, counter)
    levels = {q: LocalGambletLevel(q, psi, Aq)}
    levels[q]._repair_slot_a = ia
    level = levels[q]
    solver = None
    gk = None
    if _load is not None:  # fast_solve: (g_device, records) -- solve pipelined per level
        solver = _LevelSolver(levels, tree, schedule.subband_tol(), counter, _load[1])
        gk = _load[0]
    spool = _LevelTasks(solver)
    try:
        for k in range(q, 1, -1):
            level = local_level_step(level, tree, schedule, w_variant=w_variant, c_tol=c_tol,
                                     counter=counter, dense_cutoff=dense_cutoff, _ctx=ctx,
                                     _spool=spool, _g=gk,
                                     _lean=_lean and _load is not None and k > _keep_below)
            levels[k - 1] = level
            if solver is not None:
                gk = solver.restrict(k, gk)     # g^(k-1) = R^(k) g^(k), main stream
                if _lean and k > _keep_below:
                    levels[k].restriction = None
    finally:
        spool.join(counter)
    ctx.check()
    for k, lv in levels.items():
        rep = ctx.repair_of.get(getattr(lv, "_repair_slot_a", -1), 0.0)
        rep_b = ctx.repair_of.get(getattr(lv, "_repair_slot_b", -1), 0.0)
        lv.symmetry_repair = max(rep, rep_b)
    solved = None
    if solver is not None:
        solver.coarse(gk)
        solved = solver.finish()
    return levels, counter, solved


# ---------------------------------------------------------------------------
# solve phase
# ---------------------------------------------------------------------------

def solve_with_transform(levels, load, tree, schedule, g_mode="nodal", counter=None):
    """Load-dependent phase (gamblet_fast.py:677-775): moments, subband CG per
    level, increments psi^(k)T W^T w^(k), restriction of the load, coarse
    solve, reassembly.  Repeat solves reuse `levels` unchanged.

    Extension (batched repeat solves, "subsequent solves"):
    `load` may be a list/tuple of loads; the subband PCGs of two loads then
    share every operator pass (gb_bjcg_solve2) and the call returns
    ([MultiresSolution, ...], counter), each solution bitwise the one a
    single-load call returns."""
    counter = counter if counter is not None else FlopCounter()
    q = tree.q
    n = 1 << q
    N = n * n
    tol = schedule.subband_tol()
    batch = isinstance(load, (list, tuple))
    loads = list(load) if batch else [load]
    if batch and not loads:
        raise InvalidArgumentError("empty list of loads")
    s = dv.stream()
    gs = []
    with counter.timer("solve phase"):
        for ld in loads:
            if isinstance(ld, LoadVector):
                b, g_nodal = ld.b, ld.g_nodal
            else:
                b, g_nodal = (ld if isinstance(ld, torch.Tensor)
                              else np.asarray(ld, dtype=float)), None
            if tuple(b.shape) != (N,):
                raise InvalidArgumentError(f"load shape {b.shape} does not match N={N}")
            if g_mode == "nodal":
                if g_nodal is None:
                    raise InvalidArgumentError(
                        "nodal moment shortcut needs a LoadVector with g_nodal; "
                        "pass g_mode='measured' for a bare right-hand side")
                g = dv.to_dev(g_nodal if isinstance(g_nodal, torch.Tensor)
                              else np.asarray(g_nodal, dtype=float))
                counter.add("line4", 0)
            elif g_mode == "measured":
                psiq = levels[q].raw("psi")
                if not isinstance(psiq, PsiWindows):
                    psiq = _psi_dev(levels[q], n, n)
                bd = dv.to_dev(b)
                g = dv.empty(N)
                nat.call("gb_psi_apply", n, n, psiq.lo, psiq.wd, dv.ptr(psiq.vals), dv.ptr(bd),
                         dv.ptr(g), s)
                counter.add("line4", 2 * N * psiq.wd * psiq.wd)
            else:
                raise InvalidArgumentError(f"unknown g_mode {g_mode!r}")
            gs.append(g)
        records = [[] for _ in gs]
        if batch:
            outs = _solve_levels_batch(levels, gs, tree, schedule, tol, counter, records)
        else:
            outs = [_solve_levels(levels, gs[0], tree, schedule, tol, counter, records[0])]

    sols = []
    for (sol_parts, U1), recs in zip(outs, records):
        u = dv.to_host(sol_parts["partials"].device(q))
        sols.append(MultiresSolution(u=u, u1_coarse=dv.to_host(U1),
                                     subband_coeffs=sol_parts["coeffs"],
                                     increments=sol_parts["increments"],
                                     partials=sol_parts["partials"], records=recs))
    return (sols if batch else sols[0]), counter


class _LevelSolver:
    """Load-dependent work of one level at a time (gamblet_fast.py:717-765):
    rhs = s (W g), block-Jacobi PCG on S B S, w = s z, increment psi^T W^T w,
    g <- R g; then the coarse solve and the partial sums.  Used sequentially
    by solve_with_transform and as the body of the pipelined fast_solve."""

    def __init__(self, levels, tree, tol, counter, records):
        self.levels, self.tree, self.tol = levels, tree, tol
        self.counter, self.records = counter, records
        self.n = 1 << tree.q
        self.N = self.n * self.n
        self.coeffs, self.incs = HostDict(), HostDict()
        # (f0, f1): increments on these fine rows only (column strips of psi,
        # gamblet_dist.py); the other entries of an increment stay zero
        self.fine_rows = None

    def _psi_t(self, L, psi, v):
        """inc = psi^T v over the fine grid (or its fine_rows strip)."""
        if self.fine_rows is None:
            inc = dv.empty(self.N)
            nat.call("gb_psi_t_apply", self.n, L, psi.lo, psi.wd, dv.ptr(psi.vals), dv.ptr(v),
                     dv.ptr(inc), dv.stream())
            return inc
        f0, f1 = self.fine_rows
        inc = dv.zeros(self.N)
        nat.call("gb_psi_t_apply_rows", self.n, L, psi.lo, psi.wd, dv.ptr(psi.vals), dv.ptr(v),
                 dv.ptr(inc), f0, f1, 0, L, dv.stream())
        return inc

    def _check(self, k, need_r=True):
        lvl = self.levels[k]
        R = lvl.raw("restriction")
        B = lvl.raw("subband")
        if B is None or (need_r and R is None):
            raise InvalidArgumentError(
                f"level {k} is missing transform data; run fast_transform first")
        if not isinstance(B, BoxMatrix) or (need_r and not isinstance(R, BoxMatrix)):
            raise InvalidArgumentError(
                f"level {k} was not produced by this package's fast_transform")
        return lvl, B, R

    def subband(self, k, g, pipelined=False, engine=None, psi=None):
        op, sB, rhs = self.subband_rhs(k, g, pipelined)
        if engine is not None:
            zp, its, rel, conv, brk = engine(op, op.pad(rhs), self.tol)
        else:
            with dv.phase("subband_cg"):
                zp, its, rel, conv, brk, _ = _pcg(op, op.pad(rhs), self.tol)
            dv.Prof.add_work("subband_cg", nbytes=its * (op.spmv_bytes + 10 * 8 * op.npad
                                                         + 12 * 8 * op.n))
        self.subband_finish(k, op, sB, zp, its, rel, conv, brk, psi)

    def subband_rhs(self, k, g, pipelined=False):
        """(operator, s_B, rhs = s (W g)) of level k (gamblet_fast.py:717-722)."""
        lvl = self.levels[k]
        op = getattr(lvl, "_krylov_op", None) if pipelined else None
        if op is None:  # B^(k) must be on the level (a lean level hands its operator over)
            lvl, B, _ = self._check(k, need_r=not pipelined)
        s = dv.stream()
        sB = lvl.raw("subband_scale")
        if not isinstance(sB, torch.Tensor):
            sB = dv.empty(B.rows)
            st = dv.zeros(2, torch.int64)
            nat.call("gb_box_scale", B.rows, 3, B.w, dv.ptr(B.vals), dv.ptr(sB), dv.ptr(st), s)
        w12 = w_template(lvl.w_variant or "orthonormal").ctypes.data
        if op is None:
            op = getattr(lvl, "_op", None) or _POp(B, sB)
            lvl._op = op  # the Krylov copy is kept for repeat solves
        Lp, J = op.L, op.n
        rhs = dv.empty(J)
        nat.call("gb_apply_w", Lp, w12, dv.ptr(g), dv.ptr(sB), dv.ptr(rhs), s)
        self.counter.add("line8", 8 * J + J)
        return op, sB, rhs

    def subband_finish(self, k, op, sB, zp, its, rel, conv, brk, psi=None):
        """w = s z, the increment psi^T W^T w (gamblet_fast.py:723-745)."""
        lvl = self.levels[k]
        s = dv.stream()
        counter = self.counter
        Lp, J = op.L, op.n
        w12 = w_template(lvl.w_variant or "orthonormal").ctypes.data
        if brk:
            raise NumericalError(f"CG breakdown at iteration {brk}: p^T A p <= 0 "
                                 "(matrix is not SPD)")
        if not conv:
            raise NumericalError(f"subband solve at level {k} did not converge")
        w = op.unpad(zp, sB)
        counter.add("line8", cg_flops(J * op.slots, J, its) + 2 * J * its)
        counter.record_iters("line8", its)
        counter.record_solve(f"line8 level {k}", its, self.tol)
        self.records.append(SolveRecord(k, "subband", J, 1, self.tol, np.array([its]),
                                        np.array([rel])))
        v = dv.empty(4 * Lp * Lp)
        nat.call("gb_apply_wt", Lp, w12, dv.ptr(w), dv.ptr(v), s)
        if psi is None:
            psi = lvl.raw("psi")
        if not isinstance(psi, PsiWindows):
            psi = _psi_dev(lvl, self.n, 2 * Lp)
        inc = self._psi_t(2 * Lp, psi, v)
        psi.vals.record_stream(torch.cuda.current_stream())
        counter.add("line10", 8 * J + 2 * (4 * Lp * Lp) * psi.wd * psi.wd)
        self.incs[k] = inc
        self.coeffs[k] = w

    def restrict(self, k, g):
        R = self.levels[k].raw("restriction")
        if not isinstance(R, BoxMatrix):
            self._check(k)
        Lp = R.L
        gn = dv.empty(Lp * Lp)
        nat.call("gb_apply_r", Lp, R.w, dv.ptr(R.vals), dv.ptr(g), dv.ptr(gn), dv.stream())
        self.counter.add("line15", 2 * Lp * Lp * R.slots)
        return gn

    def coarse(self, g):
        s = dv.stream()
        counter = self.counter
        coarse = self.levels[1]
        A1 = _box_dev(coarse, "stiffness", 2, None)
        s1 = dv.empty(4)
        st = dv.zeros(2, torch.int64)
        nat.call("gb_box_scale", 4, 1, A1.w, dv.ptr(A1.vals), dv.ptr(s1), dv.ptr(st), s)
        op1 = _POp(A1, s1)
        zp, its, rel, conv, brk, _ = _cg(op1, op1.pad(g, s1), self.tol)
        if brk:
            raise NumericalError(f"CG breakdown at iteration {brk}: p^T A p <= 0 "
                                 "(matrix is not SPD)")
        if not conv:
            raise NumericalError("coarse solve did not converge")
        U1 = op1.unpad(zp, s1)
        counter.add("line16", cg_flops(4 * A1.slots, 4, its))
        counter.record_iters("line16", its)
        counter.record_solve("line16", its, self.tol)
        self.records.append(SolveRecord(1, "coarse", 4, 1, self.tol, np.array([its]),
                                        np.array([rel])))
        psi1 = coarse.raw("psi")
        if not isinstance(psi1, PsiWindows):
            psi1 = _psi_dev(coarse, self.n, 2)
        inc1 = self._psi_t(2, psi1, U1)
        counter.add("line17", 2 * 4 * psi1.wd * psi1.wd)
        self.incs[1] = inc1
        self.U1 = U1

    def finish(self):
        q = self.tree.q
        s = dv.stream()
        prev = self.incs.device(1)
        partials = HostDict({1: prev})
        for k in range(2, q + 1):
            out = dv.empty(self.N)
            nat.call("gb_vadd", self.N, dv.ptr(prev), dv.ptr(self.incs.device(k)),
                     dv.ptr(out), s)
            partials[k] = out
            prev = out
        self.counter.add("line18", (q - 1) * self.N)
        return {"coeffs": self.coeffs, "increments": self.incs, "partials": partials}, self.U1


def _solve_levels(levels, g, tree, schedule, tol, counter, records):
    """Sequential solve phase on the current stream."""
    sv = _LevelSolver(levels, tree, tol, counter, records)
    for k in range(tree.q, 1, -1):
        sv.subband(k, g)
        g = sv.restrict(k, g)
    sv.coarse(g)
    return sv.finish()


def _pcg2(op, b0, b1, rel_tol):
    """Two block-Jacobi PCG solves on one operator in lockstep, sharing every
    S B S pass (gb_bjcg_solve2); each result is bitwise _pcg's.  Returns the
    two _pcg tuples."""
    max_iter = min(max(200, 2 * op.n), MAX_ITER_CAP)
    inv = op.bj_inv()
    st = dv.stream()
    vecs, krs = [], []
    for b in (b0, b1):
        kr = _Krylov(op.npad)
        x, r, p, Ap, z = (op.vec() for _ in range(5))
        nat.call("gb_state_reset", dv.ptr(kr.state), max_iter, st)
        nat.call("gb_bjcg_init", op.L, op.w, dv.ptr(b), None, None, 1.0, dv.ptr(x), dv.ptr(r),
                 dv.ptr(p), dv.ptr(z), dv.ptr(inv), float(rel_tol), int(max_iter),
                 dv.ptr(kr.state), dv.ptr(kr.part), st)
        vecs.append((x, r, p, Ap, z))
        krs.append(kr)
    P2 = nat.ctypes.c_void_p * 2
    arr = lambda i: P2(*(dv.ptr(v[i]) for v in vecs))  # noqa: E731
    nat.call("gb_bjcg_solve2", op.L, op.w, dv.ptr(op.BsT), dv.ptr(inv), arr(0), arr(1),
             arr(2), arr(3), arr(4), P2(*(dv.ptr(kr.state) for kr in krs)),
             P2(*(dv.ptr(kr.part) for kr in krs)), P2(*(kr.host.data_ptr() for kr in krs)),
             128, st)
    out = []
    for (x, *_), kr in zip(vecs, krs):
        h = kr.host_view()
        rel = float(h["rnorm"] / h["bnorm"]) if h["bnorm"] > 0 else 0.0
        out.append((x, int(h["it"]), rel, bool(h["converged"]), int(h["breakdown"]), h))
    return out


def _solve_levels_batch(levels, gs, tree, schedule, tol, counter, records):
    """The sequential solve phase for several loads at once: per level, the
    subband PCGs run two at a time through the dual-vector symmetric SpMV
    (one stream of S B^(k) S per pass for both loads); every other step is
    the single-load arithmetic.  Each result is bitwise the single solve's."""
    svs = [_LevelSolver(levels, tree, tol, counter, recs) for recs in records]
    gs = list(gs)
    for k in range(tree.q, 1, -1):
        prep = [sv.subband_rhs(k, g) for sv, g in zip(svs, gs)]
        op = prep[0][0]
        i = 0
        while i < len(svs):
            res = None
            if i + 1 < len(svs) and op.layout == 1 and op.nr == 3:
                try:
                    with dv.phase("subband_cg2"):
                        res = _pcg2(op, op.pad(prep[i][2]), op.pad(prep[i + 1][2]), tol)
                except InvalidArgumentError:  # no bitwise-equal pair kernel at this w
                    res = None
            if res is not None:
                its = max(r[1] for r in res)
                dv.Prof.add_work("subband_cg2", nbytes=its * (op.matrix_bytes
                                                              + 2 * (3 * 8 * op.npad
                                                                     + 10 * 8 * op.npad)))
                for j, (zp, it, rel, conv, brk, _) in enumerate(res):
                    svs[i + j].subband_finish(k, op, prep[i + j][1], zp, it, rel, conv, brk)
                i += 2
            else:
                with dv.phase("subband_cg"):
                    zp, it, rel, conv, brk, _ = _pcg(op, op.pad(prep[i][2]), tol)
                svs[i].subband_finish(k, op, prep[i][1], zp, it, rel, conv, brk)
                i += 1
        gs = [sv.restrict(k, g) for sv, g in zip(svs, gs)]
    out = []
    for sv, g in zip(svs, gs):
        sv.coarse(g)
        out.append(sv.finish())
    return out


# ---------------------------------------------------------------------------
# one-call driver and report
# ---------------------------------------------------------------------------

class FastResult:
    """Bundle returned by fast_solve (gamblet_fast.py:778-786); `report` is
    built on first access (it reads nnz counts back from the device)."""

    def __init__(self, solution, levels, schedule, counter, report=None):
        self.solution = solution
        self.levels = levels
        self.schedule = schedule
        self.counter = counter
        self._report = report

    @property
    def report(self):
        if self._report is None:
            self._report = complexity_report(self.schedule, self.counter, self.levels)
        return self._report


def _record_sizes(counter, levels):
    for k, lv in levels.items():
        for name, label in (("psi", f"psi({k})"), ("stiffness", f"A({k})")):
            v = lv.raw(name)
            if v is not None and label not in counter.sizes:
                counter.record_nnz(label, getattr(v, "nnz", None) or _nnz(v))
        if lv.raw("subband") is not None and f"B({k})" not in counter.sizes:
            counter.record_nnz(f"B({k})", _nnz(lv.raw("subband")))
        if lv.raw("restriction") is not None and f"R({k - 1})" not in counter.sizes:
            counter.record_nnz(f"R({k - 1})", _nnz(lv.raw("restriction")))


def _nnz(v):
    if sp.issparse(v):
        return v.nnz
    return v.to_csr().nnz


def complexity_report(schedule, counter, levels):
    """gamblet_fast.py:789-812 (same keys)."""
    _record_sizes(counter, levels)
    conds = {}
    for k in sorted(levels):
        lvl = levels[k]
        if lvl.lambda_min_subband is not None:
            conds[str(k)] = lvl.lambda_max_subband / lvl.lambda_min_subband
    out = {
        "schedule": {
            "epsilon": schedule.epsilon,
            "q": schedule.q,
            "c_rho": schedule.c_rho,
            "radii": {str(k): schedule.rho(k) for k in range(1, schedule.q + 1)},
            "subband_tol": schedule.subband_tol(),
        },
        "kappa": KAPPA,
        "epsilon_effective": KAPPA * schedule.epsilon,
        "subband_condition_estimates": conds,
    }
    out.update(counter.summary())
    return out


def fast_solve(M, A, load, tree, epsilon, c_rho=None, uniform_rho=None, schedule=None,
               w_variant="orthonormal", g_mode="nodal", c_tol=DEFAULT_C_TOL,
               dense_cutoff=DENSE_PATCH_CUTOFF, lean=False):
    """Localized transform plus solve in one call (gamblet_fast.py:815-837).

    lean (extension, default off): bound device memory for the largest grids
    (q=12 on one GPU) -- identical arithmetic and solution, but the level
    operators of k >= 2 are released once consumed and not returned (see
    _fast_solve_device).

    With the nodal moment shortcut the solve phase is pipelined into the
    transform (level k's subband solve runs on a second stream as soon as
    S B^(k) S exists); the arithmetic is that of fast_transform followed by
    solve_with_transform."""
    if schedule is None:
        schedule = make_schedule(epsilon, tree.q, c_rho=c_rho, uniform_rho=uniform_rho)
    counter = FlopCounter()
    q = tree.q
    N = 4 ** q
    with counter.timer("total"):
        if g_mode == "nodal" and isinstance(load, LoadVector):
            if tuple(np.shape(load.b)) != (N,):
                raise InvalidArgumentError(f"load shape {np.shape(load.b)} does not match N={N}")
            records = []
            g = dv.to_dev(load.g_nodal if isinstance(load.g_nodal, torch.Tensor)
                          else np.asarray(load.g_nodal, dtype=float))
            counter.add("line4", 0)
            levels, counter, (parts, U1) = _transform(
                M, A, tree, schedule, w_variant=w_variant, c_tol=c_tol, counter=counter,
                dense_cutoff=dense_cutoff, _load=(g, records), _lean=lean)
            solution = MultiresSolution(u=dv.to_host(parts["partials"].device(q)),
                                        u1_coarse=dv.to_host(U1),
                                        subband_coeffs=parts["coeffs"],
                                        increments=parts["increments"],
                                        partials=parts["partials"], records=records)
        else:
            levels, counter = fast_transform(M, A, tree, schedule, w_variant=w_variant,
                                             c_tol=c_tol, counter=counter,
                                             dense_cutoff=dense_cutoff)
            solution, counter = solve_with_transform(levels, load, tree, schedule,
                                                     g_mode=g_mode, counter=counter)
    return FastResult(solution, levels, schedule, counter)


def _fast_solve_device(M, A, g, tree, schedule, w_variant="orthonormal", lean=False,
                       keep_below=0):
    """fast_solve with device-resident inputs (DeviceCSR M, A; device g);
    returns (levels, parts, U1, counter) with everything left in HBM.

    lean=True bounds device memory for the largest grids (q=12 on one GPU):
    the same arithmetic, but psi^(k) and A^(k) (k >= 2) are released once
    consumed (psi^(k) after psi^(k-1) and the level-k increment, A^(k) after
    B^(k), G, P A P^T), so the returned levels do not carry them; levels
    k <= keep_below keep everything (per-level parity checks at q=12)."""
    counter = FlopCounter()
    records = []
    levels, counter, (parts, U1) = _transform(M, A, tree, schedule, w_variant=w_variant,
                                              counter=counter, _load=(g, records),
                                              _lean=lean, _keep_below=keep_below)
    return levels, parts, U1, counter
