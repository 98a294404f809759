"""Symmetric band SpMV (csrc/gb_symspmv.cuh) against the full-box SpMV and a
scipy CSR product of the same S B S, on multi-tile grids (L >= 128: several
tile columns and rows, so every spill-over path between tiles is used), and
the CG / power reductions it feeds."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from paper_1503_03467_b200 import _native as nat, device as dv

pytestmark = pytest.mark.gpu


def _sym_box(L, w, seed):
    """A symmetric, diagonally dominant 3-component box matrix on an L x L
    parent grid (the B^(k) format) and its CSR, plus a positive scale s."""
    rng = np.random.default_rng(seed)
    W2 = 2 * w + 1
    S = W2 * W2 * 3
    R = L * L * 3
    vals = np.zeros((R, S))
    data = []
    ps, pt = np.divmod(np.arange(L * L), L)
    for ds in range(0, w + 1):
        for dt in range(-w, w + 1):
            if ds == 0 and dt < 0:
                continue
            qs, qt = ps + ds, pt + dt
            ok = (qs < L) & (qt >= 0) & (qt < L)
            p, q = np.nonzero(ok)[0], (qs * L + qt)[ok]
            for c in range(3):
                for cp in range(3):
                    if ds == 0 and dt == 0 and cp < c:
                        continue
                    v = rng.standard_normal(p.size)
                    if ds == 0 and dt == 0 and cp == c:
                        v = 4.0 * S + np.abs(v)
                    r1, r2 = 3 * p + c, 3 * q + cp
                    vals[r1, ((ds + w) * W2 + dt + w) * 3 + cp] = v
                    vals[r2, ((-ds + w) * W2 - dt + w) * 3 + c] = v
                    data.append((r1, r2, v))
    r1 = np.concatenate([d[0] for d in data])
    r2 = np.concatenate([d[1] for d in data])
    v = np.concatenate([d[2] for d in data])
    off = r1 != r2
    A = sp.coo_array((np.concatenate([v, v[off]]), (np.concatenate([r1, r2[off]]),
                                                    np.concatenate([r2, r1[off]]))),
                     shape=(R, R)).tocsr()
    s = 0.5 + rng.random(R)
    return vals, A, s


def _pad(L, w, x):
    Lp = L + 2 * w
    out = np.zeros((Lp, Lp, 3))
    out[w:w + L, w:w + L] = x.reshape(L, L, 3)
    return out.reshape(-1)


def _unpad(L, w, xp):
    Lp = L + 2 * w
    return xp[:Lp * Lp * 3].reshape(Lp, Lp, 3)[w:w + L, w:w + L].reshape(-1)


@pytest.mark.parametrize("L,w", [(128, 4), (128, 6), (256, 4), (64, 5)])
def test_sym_band_apply_matches_full_box_and_csr(L, w):
    vals, A, s = _sym_box(L, w, seed=L + w)
    assert nat.query("gb_sym_supported", L, 3, w) == 1
    R = L * L * 3
    B, sd = dv.to_dev(vals.reshape(-1)), dv.to_dev(s)
    st = dv.stream()
    full = dv.empty(nat.query("gb_boxT_elems", L, 3, w))
    nat.call("gb_scale_box_T", L, 3, w, dv.ptr(B), dv.ptr(sd), dv.ptr(full), st)
    U = dv.empty(nat.query("gb_boxsym_elems", L, w))
    nat.call("gb_scale_box_symT", L, w, dv.ptr(B), dv.ptr(sd), dv.ptr(U), st)
    npad = (L + 2 * w) ** 2 * 3
    tail = nat.query("gb_sym_overflow_elems", L, w)
    x = np.random.default_rng(7).standard_normal(R)
    xd = dv.to_dev(_pad(L, w, x))
    y0 = dv.zeros(npad)
    y1 = dv.zeros(npad + tail)
    y2 = dv.zeros(npad + tail)
    nat.call("gb_tbox_apply", L, 3, w, dv.ptr(full), dv.ptr(xd), dv.ptr(y0), st, 0)
    nat.call("gb_tbox_apply", L, 3, w, dv.ptr(U), dv.ptr(xd), dv.ptr(y1), st, 1)
    nat.call("gb_tbox_apply", L, 3, w, dv.ptr(U), dv.ptr(xd), dv.ptr(y2), st, 1)
    torch.cuda.synchronize()
    Sm = sp.diags_array(s)
    ref = (Sm @ A @ Sm) @ x
    got_full = _unpad(L, w, dv.to_host(y0))
    got_sym = _unpad(L, w, dv.to_host(y1))
    scale = np.abs(ref).max()
    assert np.abs(got_full - ref).max() <= 1e-13 * scale
    assert np.abs(got_sym - ref).max() <= 1e-13 * scale
    # deterministic: a second application is bitwise identical
    assert np.array_equal(dv.to_host(y1)[:npad], dv.to_host(y2)[:npad])
    # halo of y untouched
    yp = dv.to_host(y1)[:npad].reshape(L + 2 * w, L + 2 * w, 3)
    assert not yp[:w].any() and not yp[L + w:].any()


@pytest.mark.parametrize("L,w", [(128, 4)])
def test_sym_band_cg_and_power_match_full_box(L, w):
    """A few CG and power iterations in both layouts: same reductions (alpha,
    lambda) to rounding, iterates within 1e-12."""
    vals, A, s = _sym_box(L, w, seed=3)
    R = L * L * 3
    B, sd = dv.to_dev(vals.reshape(-1)), dv.to_dev(s)
    st = dv.stream()
    ops = {}
    ops[0] = dv.empty(nat.query("gb_boxT_elems", L, 3, w))
    nat.call("gb_scale_box_T", L, 3, w, dv.ptr(B), dv.ptr(sd), dv.ptr(ops[0]), st)
    ops[1] = dv.empty(nat.query("gb_boxsym_elems", L, w))
    nat.call("gb_scale_box_symT", L, w, dv.ptr(B), dv.ptr(sd), dv.ptr(ops[1]), st)
    npad = (L + 2 * w) ** 2 * 3
    tail = nat.query("gb_sym_overflow_elems", L, w)
    b = dv.to_dev(_pad(L, w, np.random.default_rng(1).standard_normal(R)))
    red = nat.query("gb_red_blocks")
    out = {}
    for layout in (0, 1):
        x, r, p, Ap = (dv.zeros(npad + tail) for _ in range(4))
        state = dv.zeros(32)
        part = dv.empty(2 * red)
        nat.call("gb_state_reset", dv.ptr(state), 1000, st)
        nat.call("gb_cg_init", npad, dv.ptr(b), None, None, dv.ptr(x), dv.ptr(r), dv.ptr(p),
                 1e-30, 1000, dv.ptr(state), dv.ptr(part), st)
        nat.call("gb_tcg_iterations", L, 3, w, dv.ptr(ops[layout]), dv.ptr(x), dv.ptr(r),
                 dv.ptr(p), dv.ptr(Ap), 12, dv.ptr(state), dv.ptr(part), st, layout)
        xp = dv.to_dev(_pad(L, w, np.random.default_rng(2).standard_normal(R)))
        yp = dv.zeros(npad + tail)
        pst = dv.zeros(32)
        nat.call("gb_state_reset", dv.ptr(pst), 1000, st)
        nat.call("gb_tpow_iterations", L, 3, w, dv.ptr(ops[layout]), dv.ptr(xp), dv.ptr(yp),
                 1e-30, 6, dv.ptr(pst), dv.ptr(part), st, layout)
        torch.cuda.synchronize()
        out[layout] = (_unpad(L, w, dv.to_host(x)), _unpad(L, w, dv.to_host(xp)))
    for a, b_ in zip(out[0], out[1]):
        assert np.abs(a - b_).max() <= 1e-12 * np.abs(a).max()


@pytest.mark.parametrize("L,w", [(128, 4), (128, 6)])
def test_sym_band_block_jacobi_pcg_matches_full_box(L, w):
    """Block-Jacobi PCG steps: the symmetric layout's fused update (alpha from
    phase 1 by linearity, spill-over added in the update) follows the full-box
    iteration to rounding."""
    vals, A, s = _sym_box(L, w, seed=5)
    R = L * L * 3
    B, sd = dv.to_dev(vals.reshape(-1)), dv.to_dev(s)
    st = dv.stream()
    ops = {0: dv.empty(nat.query("gb_boxT_elems", L, 3, w)),
           1: dv.empty(nat.query("gb_boxsym_elems", L, w))}
    nat.call("gb_scale_box_T", L, 3, w, dv.ptr(B), dv.ptr(sd), dv.ptr(ops[0]), st)
    nat.call("gb_scale_box_symT", L, w, dv.ptr(B), dv.ptr(sd), dv.ptr(ops[1]), st)
    inv = dv.empty(144 * (L // 2) ** 2, dtype=torch.float32)
    nat.call("gb_bj_setup", L, w, dv.ptr(B), dv.ptr(sd), dv.ptr(inv), st)
    npad = (L + 2 * w) ** 2 * 3
    tail = nat.query("gb_sym_overflow_elems", L, w)
    b = dv.to_dev(_pad(L, w, np.random.default_rng(4).standard_normal(R)))
    red = nat.query("gb_red_blocks")
    out = {}
    for layout in (0, 1):
        x, r, p, Ap, z = (dv.zeros(npad + tail) for _ in range(5))
        state = dv.zeros(32)
        part = dv.empty(2 * red)
        nat.call("gb_state_reset", dv.ptr(state), 1000, st)
        nat.call("gb_bjcg_init", L, w, dv.ptr(b), None, None, 1.0, dv.ptr(x), dv.ptr(r),
                 dv.ptr(p), dv.ptr(z), dv.ptr(inv), 1e-30, 1000, dv.ptr(state), dv.ptr(part), st)
        nat.call("gb_bjcg_iterations", L, w, dv.ptr(ops[layout]), dv.ptr(inv), dv.ptr(x),
                 dv.ptr(r), dv.ptr(p), dv.ptr(Ap), dv.ptr(z), 10, dv.ptr(state), dv.ptr(part),
                 st, layout)
        torch.cuda.synchronize()
        out[layout] = _unpad(L, w, dv.to_host(x))
    assert np.abs(out[0] - out[1]).max() <= 1e-12 * np.abs(out[0]).max()
