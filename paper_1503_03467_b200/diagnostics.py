"""Diagnostics tables on the device.

Mirrors gamblets/diagnostics.py (names, arguments, return types, errors) for
the localized path's results: the per-cell energies and energy-decay profile
of a basis vector (diagnostics.py:40-85), the conditioning table
(88-94), the coefficient spectrum (97-107), compression (110-142) and the
convergence table (145-155).  The arithmetic runs in csrc/gb_diag.cu and the
solve-phase transfer kernels (W^T, psi^T); host code only orders launches
and formats rows.  The reference's own Report writer (CSV/PGM files) is out
of scope.

Inputs: `levels` / `solution` from this package's fast_transform /
fast_solve / solve_with_transform (operators resident in HBM), fine vectors
as numpy arrays or device tensors, `A_fine` as scipy CSR or a device box
(grid_fem.assemble_stiffness(..., device=True)).
"""

from __future__ import annotations

import hashlib

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as nat
from . import device as dv
from .device import BoxMatrix, PsiWindows
from .errors import InvalidArgumentError, NumericalError
from .grid_fem import STIFFNESS_ELEMENT
from .hierarchy import w_template

__all__ = [
    "config_hash", "cell_energies", "cell_centers", "decay_profile", "fit_log_slope",
    "conditioning_table", "coefficient_spectrum", "compress", "convergence_table",
]

_E16 = np.ascontiguousarray(STIFFNESS_ELEMENT.reshape(16))


def config_hash(config):
    """12-hex digest of a flat config mapping (diagnostics.py:34-37)."""
    lines = [f"{k}={config[k]}" for k in sorted(config)]
    return hashlib.sha256("\n".join(lines).encode()).hexdigest()[:12]


def _vec(x, n, what):
    shape = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
    if shape != (n,):
        raise InvalidArgumentError(f"expected {n} {what}, got shape {shape}")
    return x if isinstance(x, torch.Tensor) and x.is_cuda else dv.to_dev(
        np.ascontiguousarray(x, dtype=np.float64))


def _cell_energies_dev(grid, coefficient, v):
    vd = _vec(v, grid.num_nodes, "nodal values")
    coef = dv.to_dev(np.ascontiguousarray(coefficient.values, dtype=np.float64))
    out = dv.empty(grid.num_cells)
    nat.call("gb_cell_energies", grid.n, dv.ptr(vd), dv.ptr(coef), _E16.ctypes.data,
             dv.ptr(out), dv.stream())
    return out


def cell_energies(grid, coefficient, v):
    """Per-cell energy contributions of a fine vector v, summing to v^T A v
    (diagnostics.py:40-49)."""
    return dv.to_host(_cell_energies_dev(grid, coefficient, v))


def cell_centers(grid):
    """(num_cells, 2) cell centres (diagnostics.py:52-55)."""
    m = grid.n + 1
    ci, cj = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    return np.column_stack([(ci.ravel() + 0.5) * grid.h, (cj.ravel() + 0.5) * grid.h])


def decay_profile(grid, coefficient, psi_row, center, radii):
    """Energy fraction of psi_row outside B(center, r) for each r; a cell is
    outside when its centre is at distance >= r (diagnostics.py:58-74)."""
    en = _cell_energies_dev(grid, coefficient, psi_row)
    radii = np.ascontiguousarray(np.asarray(radii, dtype=float).ravel())
    nr = radii.size
    rd = dv.to_dev(radii) if nr else dv.empty(1)
    part = dv.empty(int(nat.query("gb_decay_part_elems", nr)))
    out = dv.empty(nr + 1)
    nat.call("gb_decay_sums", grid.n, float(grid.h), dv.ptr(en), float(center[0]),
             float(center[1]), dv.ptr(rd), nr, dv.ptr(part), dv.ptr(out), dv.stream())
    sums = dv.to_host(out)
    total = sums[nr]
    if total <= 0.0:
        raise InvalidArgumentError("basis vector has zero energy")
    return np.clip(sums[:nr] / total, 0.0, None)


def fit_log_slope(radii, fractions, floor=1e-13):
    """Least-squares slope of log(fraction) against r over the decaying range
    (diagnostics.py:77-85; a handful of host numbers)."""
    radii = np.asarray(radii, dtype=float)
    fractions = np.asarray(fractions, dtype=float)
    mask = (fractions > floor) & (fractions < 1.0)
    if mask.sum() < 2:
        raise InvalidArgumentError("not enough positive samples to fit a slope")
    return float(np.polyfit(radii[mask], np.log(fractions[mask]), 1)[0])


def conditioning_table(named_matrices, tol=1e-2):
    """Rows (label, size, lambda_min, lambda_max, cond) by the reference's
    power / inverse iteration on the device (diagnostics.py:88-94)."""
    from .krylov import eig_extremes
    rows = []
    for label, mat in named_matrices:
        lmin, lmax = eig_extremes(mat, tol=tol)
        rows.append((label, int(mat.shape[0]), lmin, lmax, lmax / lmin))
    return rows


def _level_box(level, name):
    v = level.raw(name) if hasattr(level, "raw") else None
    if not isinstance(v, BoxMatrix):
        raise InvalidArgumentError(
            f"level {getattr(level, 'k', '?')}: {name} is not resident on the device "
            "(device diagnostics take levels from fast_transform / fast_solve)")
    return v


def _coeff_dev(solution, k):
    d = solution.subband_coeffs
    v = d.device(k) if hasattr(d, "device") else d[k]
    return v if isinstance(v, torch.Tensor) and v.is_cuda else dv.to_dev(
        np.ascontiguousarray(v, dtype=np.float64))


def _spectrum_dev(solution, levels):
    """Concatenated device spectrum (levels 1, 2, ..., q in sorted order) and
    the per-level (k, offset, size)."""
    parts = [(1, _level_box(levels[1], "stiffness"),
              dv.to_dev(np.ascontiguousarray(solution.u1_coarse, dtype=np.float64)))]
    for k in sorted(solution.subband_coeffs):
        parts.append((k, _level_box(levels[k], "subband"), _coeff_dev(solution, k)))
    sizes = [B.rows for _, B, _ in parts]
    for (k, B, c), size in zip(parts, sizes):
        if c.numel() != size:
            raise InvalidArgumentError(f"level {k}: {c.numel()} coefficients for {size} rows")
    total = int(sum(sizes))
    out = dv.empty(total)
    s = dv.stream()
    layout, off = [], 0
    for (k, B, c), size in zip(parts, sizes):
        nat.call("gb_box_diag_spectrum", size, B.nr, B.w, dv.ptr(B.vals), dv.ptr(c),
                 dv.ptr(out) + 8 * off, s)
        layout.append((k, off, size))
        off += size
    return out, layout, parts


def coefficient_spectrum(solution, levels):
    """{k: |coefficient| x energy norm of its basis vector}: |U_i| sqrt(A^(1)_ii)
    on level 1, |w_i^(k)| sqrt(B^(k)_ii) in the subbands (diagnostics.py:97-107)."""
    out, layout, _ = _spectrum_dev(solution, levels)
    host = dv.to_host(out)
    return {k: host[off:off + size].copy() for k, off, size in layout}


def _box_fine(A_fine, n):
    if isinstance(A_fine, BoxMatrix):
        if A_fine.nr != 1 or A_fine.L != n:
            raise InvalidArgumentError("A_fine box does not match the fine grid")
        return A_fine
    if not sp.issparse(A_fine):
        raise InvalidArgumentError("A_fine must be a sparse matrix or a device box")
    if A_fine.shape != (n * n, n * n):
        raise InvalidArgumentError(f"A_fine shape {A_fine.shape} does not match N={n * n}")
    box, _ = dv.csr_to_box(A_fine, n)
    return box


def _energy_norm_dev(Ab, x, tol=1e-12):
    """sqrt(x^T A x) with the reference's indefinite guard (grid_fem.py:248-257)."""
    part = dv.empty(int(nat.query("gb_quad_part_elems")))
    out = dv.empty(1)
    nat.call("gb_box_quadform", Ab.L, Ab.w, dv.ptr(Ab.vals), dv.ptr(x), dv.ptr(part),
             dv.ptr(out), dv.stream())
    val = float(dv.to_host(out)[0])
    if val < 0.0:
        s = dv.stream()
        st = dv.empty(int(nat.query("gb_kstate_bytes")), torch.uint8)
        nat.call("gb_state_reset", dv.ptr(st), 0, s)
        dots = dv.empty(2)
        npart = dv.empty(2 * int(nat.query("gb_red_blocks")))
        nat.call("gb_dot2", x.numel(), dv.ptr(x), dv.ptr(x), None, dv.ptr(dots), dv.ptr(st),
                 dv.ptr(npart), s)
        nat.call("gb_max_abs", Ab.vals.numel(), dv.ptr(Ab.vals), dv.ptr(part), dv.ptr(out), s)
        xx = float(dv.to_host(dots)[0])
        scale = float(dv.to_host(out)[0])
        if val < -tol * scale * xx:
            raise NumericalError(f"quadratic form is negative: x^T A x = {val:.3e}")
        val = 0.0
    return float(np.sqrt(val))


def _fine_n(levels):
    q = max(levels)
    return 1 << q


def compress(solution, levels, A_fine, keep_fraction):
    """Zero all but the largest keep_fraction of the normalized coefficients
    (stable selection); returns (u_compressed, relative A-norm error against
    the full reconstruction) (diagnostics.py:110-142)."""
    if not 0.0 < keep_fraction <= 1.0:
        raise InvalidArgumentError(f"keep_fraction must be in (0, 1], got {keep_fraction}")
    mags, layout, parts = _spectrum_dev(solution, levels)
    total = mags.numel()
    n_keep = int(np.ceil(keep_fraction * total))
    s = dv.stream()
    mask = dv.empty(total)
    wb = nat.ctypes.c_size_t(0)
    nat.call("gb_topk_mask", total, dv.ptr(mags), n_keep, dv.ptr(mask), None,
             nat.ctypes.byref(wb), s)
    work = dv.empty(max(1, (wb.value + 7) // 8))
    nat.call("gb_topk_mask", total, dv.ptr(mags), n_keep, dv.ptr(mask), dv.ptr(work),
             nat.ctypes.byref(wb), s)
    n = _fine_n(levels)
    N = n * n
    from .gamblet_fast import _psi_dev
    u_comp = None
    for (k, off, size), (_, B, c) in zip(layout, parts):
        cm = dv.empty(size)
        nat.call("gb_vmul", size, dv.ptr(mask) + 8 * off, dv.ptr(c), dv.ptr(cm), s)
        lvl = levels[k]
        psi = lvl.raw("psi")
        if not isinstance(psi, PsiWindows):
            if psi is None:
                raise InvalidArgumentError(f"level {k} has no psi (lean transform)")
            psi = _psi_dev(lvl, n, 1 << k)
        if k == 1:
            v = cm
        else:
            Lp = 1 << (k - 1)
            v = dv.empty(4 * Lp * Lp)
            w12 = w_template(getattr(lvl, "w_variant", None) or "orthonormal").ctypes.data
            nat.call("gb_apply_wt", Lp, w12, dv.ptr(cm), dv.ptr(v), s)
        inc = dv.empty(N)
        nat.call("gb_psi_t_apply", n, 1 << k, psi.lo, psi.wd, dv.ptr(psi.vals), dv.ptr(v),
                 dv.ptr(inc), s)
        if u_comp is None:
            u_comp = inc
        else:
            nxt = dv.empty(N)
            nat.call("gb_vadd", N, dv.ptr(u_comp), dv.ptr(inc), dv.ptr(nxt), s)
            u_comp = nxt
    u = _vec(solution.u, N, "solution values")
    diff = dv.empty(N)
    nat.call("gb_axpby", N, 1.0, dv.ptr(u_comp), -1.0, dv.ptr(u), dv.ptr(diff), s)
    Ab = _box_fine(A_fine, n)
    rel = _energy_norm_dev(Ab, diff) / _energy_norm_dev(Ab, u)
    return dv.to_host(u_comp), float(rel)


def convergence_table(solution, u_ref, A_fine, lambda_min_a, g_l2, H=0.5):
    """Rows (k, error, bound, ratio, relative error) with the a-priori bound
    (2 / (pi sqrt(lambda_min(a)))) H^k ||g||_L2 (diagnostics.py:145-155)."""
    parts = solution.partials
    q = max(parts)
    n = 1 << q
    N = n * n
    Ab = _box_fine(A_fine, n)
    ur = _vec(u_ref, N, "reference values")
    u_norm = _energy_norm_dev(Ab, ur)
    s = dv.stream()
    rows = []
    for k in sorted(parts):
        pk = parts.device(k) if hasattr(parts, "device") else parts[k]
        pk = _vec(pk, N, "partial sum values")
        d = dv.empty(N)
        nat.call("gb_axpby", N, 1.0, dv.ptr(ur), -1.0, dv.ptr(pk), dv.ptr(d), s)
        err = _energy_norm_dev(Ab, d)
        bound = 2.0 / (np.pi * np.sqrt(lambda_min_a)) * H ** k * g_l2
        rows.append((k, float(err), float(bound), float(err / bound), float(err / u_norm)))
    return rows
