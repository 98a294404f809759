"""Canonical CSR helpers and the reference's flop models (host side).

Mirrors the non-kernel parts of gamblets/sparse_core.py: the canonical CSR
form every API matrix is exchanged in (sparse_core.py:47-67), the CgReport
record (116-123) and the flop accounting helpers (293-307).  The Krylov
solvers themselves run on the device (csrc/gb_krylov.cu); see
`paper_1503_03467_b200.krylov` for the GPU cg_solve / cg_solve_block /
eig_extremes entry points.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import InvalidArgumentError

__all__ = ["CgReport", "as_csr", "spmv_flops", "matmul_flops", "cg_flops", "cg_solve",
           "cg_solve_block", "eig_extremes"]


def _require(cond, msg):
    if not cond:
        raise InvalidArgumentError(msg)


def as_csr(matrix, drop_tol=0.0):
    """Canonical CSR: duplicates summed, explicit zeros removed, indices sorted
    (sparse_core.py:47-67, same scipy calls so results are bitwise equal)."""
    if sp.issparse(matrix):
        out = sp.csr_array(matrix)
    else:
        arr = np.asarray(matrix, dtype=float)
        _require(arr.ndim == 2, f"expected a 2-d matrix, got shape {arr.shape}")
        out = sp.csr_array(arr)
    out = out.astype(float)
    out.sum_duplicates()
    if drop_tol > 0.0:
        out.data[np.abs(out.data) <= drop_tol] = 0.0
    out.eliminate_zeros()
    out.sort_indices()
    return out


def is_canonical_csr(mat):
    """True when `mat` is a float64 CSR in canonical form (no copy needed)."""
    return (sp.issparse(mat) and mat.format == "csr" and mat.dtype == np.float64
            and mat.has_canonical_format)


@dataclass
class CgReport:
    """Outcome of one conjugate-gradient solve (sparse_core.py:116-123)."""

    iterations: int
    rel_residual: float
    converged: bool
    breakdown: bool = False


def spmv_flops(A, ncols=1):
    return 2 * A.nnz * ncols


def matmul_flops(A, B):
    _require(A.shape[1] == B.shape[0], f"shape mismatch: {A.shape} @ {B.shape}")
    row_nnz = np.diff(B.indptr)
    return int(2 * row_nnz[A.indices].sum())


def cg_flops(nnz, n, iterations, ncols=1):
    return int(iterations) * (2 * int(nnz) + 12 * int(n)) * ncols


# GPU Krylov solvers with the reference's signatures (sparse_core.py:126-278);
# imported lazily so the host-side helpers above stay importable without CUDA.
def cg_solve(A, b, rel_tol=1e-10, max_iter=None, x0=None):
    from .krylov import cg_solve as _f
    return _f(A, b, rel_tol=rel_tol, max_iter=max_iter, x0=x0)


def cg_solve_block(A, B, rel_tol=1e-10, max_iter=None):
    from .krylov import cg_solve_block as _f
    return _f(A, B, rel_tol=rel_tol, max_iter=max_iter)


def eig_extremes(A, tol=1e-2, max_iter=500, seed=24337):
    from .krylov import eig_extremes as _f
    return _f(A, tol=tol, max_iter=max_iter, seed=seed)
