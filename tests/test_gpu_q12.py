"""Config 3 (q = 12, 16.8 M fine DOFs, contrast 1e4) on one GPU through the
lean transform, checked level by level against the oracle (SURVEY.md 8(c):
the reference cannot run q=12 end to end; its level step applied to the
GPU's own A^(k) must reproduce B^(k), D, R and A^(k-1)).  ~1-2 min, most of
it host assembly of the 16.8 M-node inputs."""

import numpy as np
import pytest

from oracle import gamblets_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_q12_lean_levels_match_oracle_level_step():
    import torch
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
    from bench import build_inputs
    q, keep = 12, 6
    grid, M, A, load, tree = build_inputs(q, "checker")
    sched = gb.make_schedule(1e-13, q, uniform_rho=3)
    Md, Ad = dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A)
    gd = dv.to_dev(load.g_nodal)
    del M, A
    levels, parts, U1, _ = gf._fast_solve_device(Md, Ad, gd, tree, sched, lean=True,
                                                 keep_below=keep)
    torch.cuda.synchronize()
    u = dv.to_host(parts["partials"].device(q))
    assert u.shape == (4 ** q,) and np.all(np.isfinite(u))
    for k in (keep, keep - 1):
        lv = levels[k]
        ref = {"k": k, "stiffness": lv.stiffness}
        nxt = O.level_step(ref, k, sched.rho(k - 1), with_psi=False, spectral=False)
        for name, got, want in (("B", lv.subband, ref["subband"]),
                                ("R", lv.restriction, ref["restriction"]),
                                ("D", lv.correction, ref["correction"]),
                                ("A", levels[k - 1].stiffness, nxt["stiffness"])):
            assert O.rel_fro(got, want) <= 1e-10, (k, name, O.rel_fro(got, want))
            assert O.same_pattern(got, want), (k, name)
        assert 0 < lv.lambda_min_subband <= lv.lambda_max_subband
