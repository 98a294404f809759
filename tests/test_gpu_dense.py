"""The exact path's dense kernels (config 0, gamblet_exact.py:115-263): the
hand-written DMMA DGEMM, Cholesky and triangular solves against a plain
PyTorch fp64 reference of the same op (the library links no BLAS)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _gemm(m, n, k, A, ta, B, tb, alpha=1.0, beta=0.0, C=None):
    from paper_1503_03467_b200 import _native as nat, device as dv
    lda = A.shape[1]
    ldb = B.shape[1]
    out = torch.zeros(m, n, dtype=torch.float64, device="cuda") if C is None else C.clone()
    nat.call("gb_dense_gemm", m, n, k, alpha, dv.ptr(A), lda, ta, dv.ptr(B), ldb, tb, beta,
             dv.ptr(out), n, dv.stream())
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (65, 63, 17),
                                   (256, 1024, 768), (1024, 1024, 1024), (1000, 3, 513)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_dmma_gemm_matches_torch(m, n, k, ta, tb):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    A = torch.randn(*((k, m) if ta else (m, k)), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(*((n, k) if tb else (k, n)), dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    opA = A.T if ta else A
    opB = B.T if tb else B
    got = _gemm(m, n, k, A.contiguous(), ta, B.contiguous(), tb, alpha=-0.25, beta=1.5, C=C)
    want = 1.5 * C - 0.25 * (opA @ opB)
    err = (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item()
    assert err <= 1e-14, err


def test_dense_cholesky_and_solve_match_torch():
    from paper_1503_03467_b200 import _native as nat, device as dv
    n, nrhs = 768, 256
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    A = X @ X.T + n * torch.eye(n, dtype=torch.float64, device="cuda")
    B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda", generator=g)
    L = A.clone()
    st = torch.zeros(2, dtype=torch.int64, device="cuda")
    nat.call("gb_dense_potrf", n, dv.ptr(L), n, dv.ptr(st), dv.stream())
    Y = B.clone()
    nat.call("gb_dense_potrs", n, nrhs, dv.ptr(L), n, dv.ptr(Y), nrhs, dv.stream())
    torch.cuda.synchronize()
    assert int(st[0]) == 0
    want = torch.linalg.solve(A, B)
    err = (torch.linalg.norm(Y - want) / torch.linalg.norm(want)).item()
    assert err <= 1e-12, err
    Lt = torch.tril(L)
    err = (torch.linalg.norm(Lt @ Lt.T - A) / torch.linalg.norm(A)).item()
    assert err <= 1e-14, err
