"""Transform persistence: a transform saved in
its HBM layout and restored serves repeat solves bitwise
(gamblet_fast.py:677-775, the reference's reuse contract
test_gamblet_fast.py:230-244); Matrix Market dumps of the level operators
(sparse_core.py:281-288, cli.py:409-457) round-trip exactly."""

import numpy as np
import pytest

import paper_1503_03467_b200 as gb
from paper_1503_03467_b200.persistence import load_transform, mm_read, mm_write, save_transform

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("q,coeff", [(5, "example1"), (7, "checker")])
def test_saved_transform_solves_bitwise(problem, tmp_path, q, coeff):
    p = problem(q, coeff)
    schedule = gb.make_schedule(1e-13, q, uniform_rho=3)
    levels, _ = gb.fast_transform(p.M, p.A, p.tree, schedule)
    s1, _ = gb.solve_with_transform(levels, p.load, p.tree, schedule)
    path = save_transform(levels, tmp_path / "t.npz")
    back = load_transform(path, p.tree)
    assert sorted(back) == sorted(levels)
    s2, _ = gb.solve_with_transform(back, p.load, p.tree, schedule)
    assert np.array_equal(s1.u, s2.u)
    for k in (q, 2):
        for f in ("stiffness", "subband", "restriction", "correction", "psi"):
            a, b = getattr(levels[k], f), getattr(back[k], f)
            assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.data, b.data), f
        assert back[k].lambda_min_subband == levels[k].lambda_min_subband
        assert (back[k].null_w != levels[k].null_w).nnz == 0
    # Matrix Market dumps of the level operators (gamblets transform)
    for name, mat in (("B", levels[q].subband), ("R", levels[q].restriction),
                      ("A", levels[q - 1].stiffness)):
        f = tmp_path / f"{name}.mtx"
        mm_write(f, mat, comment="config test")
        m2 = mm_read(f)
        assert np.array_equal(m2.indptr, mat.indptr) and np.array_equal(m2.data, mat.data)
