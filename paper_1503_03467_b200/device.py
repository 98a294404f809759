"""Device-resident operators in box-stencil layout and their lazy CSR export.

torch owns the memory (caching allocator, streams); every computation is a
call into libgamblets_b200.so.  A level operator lives on the GPU as a
`BoxMatrix` or `PsiWindows`; the scipy CSR the reference API exposes is
produced on first access by the export kernels (count -> scan -> emit) and
cached on the host.
"""

from __future__ import annotations

import threading
from contextlib import contextmanager

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as nat
from .errors import InvalidArgumentError

EXP_SQUARE, EXP_CHILD, EXP_PSI, EXP_TDT = 0, 1, 2, 3

_DEV = None


def device():
    """The CUDA device the package runs on; raises when there is none."""
    global _DEV
    if _DEV is None:
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_1503_03467_b200 needs a CUDA device (B200, sm_100a); "
                "there is no CPU fallback")
        nat.load()
        _DEV = torch.device("cuda", torch.cuda.current_device())
    return _DEV


def stream():
    return torch.cuda.current_stream(device()).cuda_stream


def ptr(t):
    return None if t is None else t.data_ptr()


def reserve(nbytes):
    """Grow the caching allocator by one segment of `nbytes` (released back to
    the cache immediately).  Later work tensors are carved out of it, so a
    steady-state solve makes no cudaMalloc calls -- those stall every stream."""
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    blk = torch.empty(int(nbytes), dtype=torch.uint8, device=device())
    del blk


def empty(n, dtype=torch.float64):
    return torch.empty(int(n), dtype=dtype, device=device())


def zeros(n, dtype=torch.float64):
    return torch.zeros(int(n), dtype=dtype, device=device())


class Traffic:
    """Host<->device byte counters (the bench's e2e h2d/d2h accounting)."""

    h2d = 0
    d2h = 0

    @classmethod
    def reset(cls):
        cls.h2d = cls.d2h = 0


# host->device: arrays above this size go through the library's pinned
# staging ring (gb_h2d_staged: multi-threaded host copy overlapped with the
# DMA) -- a pageable copy is bounded by one driver memcpy thread
_STAGE_MIN_BYTES = 4 << 20
_STAGE_THREADS = 4
# the staging ring is one per process: in-process ranks (comm.ThreadComm) take turns
_STAGE_LOCK = threading.Lock()


def _staged_copy(t):
    out = torch.empty(t.shape, dtype=t.dtype, device=device())
    with _STAGE_LOCK:
        nat.call("gb_h2d_staged", out.data_ptr(), t.data_ptr(), t.numel() * t.element_size(),
                 _STAGE_THREADS, stream())
    return out


def _index_to_dev(idx):
    """Host CSR index array (int32 or int64) -> device int32; int64 input is
    narrowed by the staging threads instead of a host astype pass."""
    idx = np.ascontiguousarray(idx)
    if idx.dtype == np.int64 and idx.nbytes >= _STAGE_MIN_BYTES and torch.cuda.is_available():
        out = torch.empty(idx.shape, dtype=torch.int32, device=device())
        Traffic.h2d += idx.size * 4
        with _STAGE_LOCK:
            nat.call("gb_h2d_staged_i64_i32", out.data_ptr(), idx.ctypes.data, idx.size,
                     _STAGE_THREADS, stream())
        return out
    return to_dev(idx.astype(np.int32, copy=False))


def to_dev(arr, dtype=None):
    """Host array -> new device tensor (counted in Traffic.h2d).  A torch
    tensor already on the device is returned as is."""
    if isinstance(arr, torch.Tensor):
        if arr.is_cuda:
            return arr if dtype is None else arr.to(dtype)
        arr = arr.numpy()
    a = np.ascontiguousarray(arr)
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    Traffic.h2d += t.numel() * t.element_size()
    if t.numel() * t.element_size() >= _STAGE_MIN_BYTES and torch.cuda.is_available():
        return _staged_copy(t)
    return t.to(device(), non_blocking=False)


def to_host(t):
    """Device tensor -> numpy (counted in Traffic.d2h)."""
    Traffic.d2h += t.numel() * t.element_size()
    return t.cpu().numpy()


class DeviceCSR:
    """A canonical CSR matrix already resident in HBM (int32 indptr/indices,
    float64 data) -- the device-side form of the API's M and A."""

    def __init__(self, indptr, indices, data, shape):
        self.indptr, self.indices, self.data, self.shape = indptr, indices, data, shape

    @classmethod
    def from_scipy(cls, mat):
        return cls(_index_to_dev(mat.indptr), _index_to_dev(mat.indices),
                   to_dev(mat.data.astype(np.float64, copy=False)), mat.shape)


class Prof:
    """Optional per-phase CUDA-event timing on the launching stream."""

    enabled = False
    events = []
    flops = {}
    bytes = {}

    @classmethod
    def reset(cls, enabled=True):
        cls.enabled = enabled
        cls.events = []
        cls.flops = {}
        cls.bytes = {}

    @classmethod
    def add_work(cls, label, flops=0, nbytes=0):
        if cls.enabled:
            cls.flops[label] = cls.flops.get(label, 0) + flops
            cls.bytes[label] = cls.bytes.get(label, 0) + nbytes

    @classmethod
    def times_ms(cls):
        torch.cuda.synchronize()
        out = {}
        for label, a, b in cls.events:
            out[label] = out.get(label, 0.0) + a.elapsed_time(b)
        return out

    @classmethod
    def counts(cls):
        out = {}
        for label, _, _ in cls.events:
            out[label] = out.get(label, 0) + 1
        return out


@contextmanager
def phase(label):
    if not Prof.enabled:
        yield
        return
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    try:
        yield
    finally:
        b.record()
        Prof.events.append((label, a, b))


def box_slots(w, nc):
    return (2 * w + 1) ** 2 * nc


class _Exportable:
    """Mixin: CSR export through the device kernels, cached."""

    _csr = None

    def _export_args(self):
        raise NotImplementedError

    def to_csr(self):
        if self._csr is not None:
            return self._csr
        kind, L, nr, w, nc, n, lo, wd, rows, S, shape = self._export_args()
        s = stream()
        counts = zeros(rows + 1, torch.int64)
        nat.call("gb_export_count", kind, L, nr, w, nc, n, lo, wd, ptr(self.vals),
                 rows, S, ptr(counts), s)
        indptr = empty(rows + 1, torch.int64)
        tmp_bytes = nat.ctypes.c_size_t(0)
        nat.call("gb_exclusive_scan", ptr(counts), ptr(indptr), rows, None,
                 nat.ctypes.byref(tmp_bytes), s)
        tmp = empty(max(1, tmp_bytes.value), torch.uint8)
        nat.call("gb_exclusive_scan", ptr(counts), ptr(indptr), rows, ptr(tmp),
                 nat.ctypes.byref(tmp_bytes), s)
        nnz = int(to_host(indptr[rows:rows + 1])[0])
        indices = empty(max(nnz, 1), torch.int32)
        data = empty(max(nnz, 1), torch.float64)
        nat.call("gb_export_emit", kind, L, nr, w, nc, n, lo, wd, ptr(self.vals), rows,
                 S, ptr(indptr), ptr(indices), ptr(data), s)
        ip = to_host(indptr)
        if nnz < 2 ** 31 - 1:
            ip = ip.astype(np.int32)
        out = sp.csr_array((to_host(data[:nnz]), to_host(indices[:nnz]), ip),
                           shape=shape)
        out.has_sorted_indices = True
        self._csr = out
        return out


class BoxMatrix(_Exportable):
    """Box-stencil operator.

    kind EXP_SQUARE: rows (p, c) on an L x L grid with nr components, columns
    (p + d, c') with nc components, |d| <= w.  kind EXP_CHILD: rows on L x L,
    columns are the 4 children of (p + d) on the 2L x 2L grid (R).  kind
    EXP_TDT: the stored rows are D^T (nr=1, nc=3) and the exported matrix is
    D = (D^T)^T with shape (3 L^2, L^2).
    """

    def __init__(self, vals, L, nr, w, nc, kind=EXP_SQUARE):
        self.vals, self.L, self.nr, self.w, self.nc, self.kind = vals, L, nr, w, nc, kind
        self._csr = None

    @property
    def rows(self):
        return self.L * self.L * self.nr

    @property
    def shape(self):
        return self._export_args()[-1]

    @property
    def slots(self):
        return box_slots(self.w, self.nc)

    def _export_args(self):
        L, w = self.L, self.w
        if self.kind == EXP_SQUARE:
            shape = (L * L * self.nr, L * L * self.nc)
            return (EXP_SQUARE, L, self.nr, w, self.nc, 0, 0, 0, self.rows,
                    self.slots, shape)
        if self.kind == EXP_CHILD:
            shape = (L * L, 4 * L * L)
            return (EXP_CHILD, L, 1, w, 4, 0, 0, 0, self.rows, self.slots, shape)
        if self.kind == EXP_TDT:
            shape = (3 * L * L, L * L)
            return (EXP_TDT, L, 3, w, 3, 0, 0, 0, 3 * L * L, (2 * w + 1) ** 2, shape)
        raise InvalidArgumentError(f"unknown box kind {self.kind}")


class PsiWindows(_Exportable):
    """Rows of psi^(k) over the fine grid in origin-clamped square windows.

    Row i of level side L (h = n / L) has support in [c + lo, c + hi] per
    dimension (c = (s h, t h)); the stored window has width wd = min(hi - lo
    + 1, n) and origin clamp(c + lo, 0, n - wd).
    """

    def __init__(self, vals, n, L, lo, hi):
        self.vals, self.n, self.L, self.lo, self.hi = vals, n, L, lo, hi
        self.wd = min(hi - lo + 1, n)
        self._csr = None

    @staticmethod
    def window(n, lo, hi):
        return min(hi - lo + 1, n)

    def _export_args(self):
        rows = self.L * self.L
        return (EXP_PSI, self.L, 1, 0, 1, self.n, self.lo, self.wd, rows,
                self.wd * self.wd, (rows, self.n * self.n))


def csr_to_box(mat, L):
    """Canonical CSR on an L x L grid -> BoxMatrix (half-width from the data).
    Host CSR (scipy) is uploaded; a DeviceCSR is used in place."""
    s = stream()
    if not isinstance(mat, DeviceCSR):
        mat = DeviceCSR.from_scipy(mat)
    indptr, indices, data = mat.indptr, mat.indices, mat.data
    wbuf = zeros(1, torch.int32)
    nat.call("gb_csr_halfwidth", L, ptr(indptr), ptr(indices), ptr(wbuf), s)
    w = int(to_host(wbuf)[0])
    box = zeros(L * L * box_slots(w, 1))
    status = zeros(2, torch.int64)
    nat.call("gb_csr_to_box", L, w, ptr(indptr), ptr(indices), ptr(data), ptr(box),
             ptr(status), s)
    return BoxMatrix(box, L, 1, w, 1), status


def csr_to_psi(mat, n, L):
    """Host CSR rows of psi^(k) (level side L over the fine n x n grid) into
    the window layout (used only when a caller hands in its own psi)."""
    mat = sp.csr_array(mat)
    h = n // L
    rows = np.repeat(np.arange(mat.shape[0]), np.diff(mat.indptr))
    rs, rt = rows // L * h, rows % L * h
    fs, ft = mat.indices // n, mat.indices % n
    lo = int(min((fs - rs).min(initial=0), (ft - rt).min(initial=0)))
    hi = int(max((fs - rs).max(initial=0), (ft - rt).max(initial=0)))
    wd = PsiWindows.window(n, lo, hi)
    os_ = np.clip(rs + lo, 0, n - wd)
    ot_ = np.clip(rt + lo, 0, n - wd)
    buf = np.zeros((L * L, wd, wd))
    buf[rows, fs - os_, ft - ot_] = mat.data
    return PsiWindows(to_dev(buf.ravel()), n, L, lo, hi)


def assemble_q1(n, cell_scale, const_scale, element):
    """On-device Q1 assembly (grid_fem.py:205-214) into the half-width-1 box:
    bitwise the reference's canonical CSR values (csrc gb_assemble_q1).
    cell_scale: (n+1)^2 per-cell factors (host array or device tensor) or
    None for const_scale everywhere."""
    s = stream()
    e16 = np.ascontiguousarray(np.asarray(element, dtype=np.float64).reshape(16))
    cs = None
    if cell_scale is not None:
        cs = cell_scale if isinstance(cell_scale, torch.Tensor) else to_dev(
            np.ascontiguousarray(cell_scale, dtype=np.float64))
        if cs.numel() != (n + 1) * (n + 1):
            raise InvalidArgumentError(f"expected {(n + 1) ** 2} cell values, got {cs.numel()}")
    box = empty(n * n * 9)
    nat.call("gb_assemble_q1", n, None if cs is None else ptr(cs), float(const_scale),
             e16.ctypes.data, ptr(box), s)
    if cs is not None:
        cs.record_stream(torch.cuda.current_stream())
    return BoxMatrix(box, n, 1, 1, 1)


def box1_matvec(M, g):
    """b = M g for a half-width-1 BoxMatrix, scipy csr_matvec order (bitwise)."""
    s = stream()
    gd = g if isinstance(g, torch.Tensor) else to_dev(np.ascontiguousarray(g, dtype=np.float64))
    b = empty(M.L * M.L)
    nat.call("gb_box1_matvec", M.L, ptr(M.vals), ptr(gd), ptr(b), s)
    return b, gd
