"""On-device assembly (grid_fem.py:189-245): the
Q1 mass / stiffness boxes and b = M g built in HBM must be the reference's
canonical CSR and load bitwise -- checked against the digests the reference
itself produced (tests/golden/pins.npz) -- and fast_solve on device-assembled
inputs must return the identical solution."""

import numpy as np
import pytest

import paper_1503_03467_b200 as gb
from oracle.make_goldens import digest

pytestmark = pytest.mark.gpu


def _coeff(grid, kind):
    if kind == "example1":
        return gb.coefficient_example1(grid)
    return gb.coefficient_checkerboard(grid, 1e4, 0)


@pytest.mark.parametrize("q", [3, 5, 7, 10])
def test_device_assembly_matches_reference_digests(golden, q):
    P = golden("pins")
    grid = gb.build_grid(q)
    Md = gb.assemble_mass(grid, device=True)
    assert Md.shape == (grid.num_nodes, grid.num_nodes)
    assert digest(Md.to_csr()) == str(P[f"digest_M_q{q}"])
    A1 = gb.assemble_stiffness(grid, gb.coefficient_example1(grid), device=True)
    assert digest(A1.to_csr()) == str(P[f"digest_Aex1_q{q}"])
    A2 = gb.assemble_stiffness(grid, gb.coefficient_checkerboard(grid, 1e4, 0), device=True)
    assert digest(A2.to_csr()) == str(P[f"digest_Achk_q{q}"])


@pytest.mark.parametrize("q", [1, 2, 4, 7])
def test_device_assembly_csr_arrays_bitwise(q):
    grid = gb.build_grid(q)
    for kind in ("example1", "checker"):
        c = _coeff(grid, kind)
        for host, dev in ((gb.assemble_mass(grid), gb.assemble_mass(grid, device=True)),
                          (gb.assemble_stiffness(grid, c),
                           gb.assemble_stiffness(grid, c, device=True))):
            got = dev.to_csr()
            np.testing.assert_array_equal(got.indptr, host.indptr)
            np.testing.assert_array_equal(got.indices, host.indices)
            assert np.array_equal(got.data.view(np.int64), host.data.view(np.int64))


@pytest.mark.parametrize("q", [3, 6, 10])
def test_device_load_is_bitwise(q):
    grid = gb.build_grid(q)
    g = np.random.default_rng(1).standard_normal(grid.num_nodes)
    host = gb.assemble_load(grid, g)
    dev = gb.assemble_load(grid, g, device=True)
    b = dev.b.cpu().numpy()
    assert np.array_equal(b.view(np.int64), host.b.view(np.int64))
    assert np.array_equal(dev.g_nodal.cpu().numpy(), g)
    # the same through an explicit device mass
    dev2 = gb.assemble_load(grid, g, mass=gb.assemble_mass(grid, device=True))
    assert np.array_equal(dev2.b.cpu().numpy().view(np.int64), host.b.view(np.int64))


@pytest.mark.parametrize("q,kind", [(5, "example1"), (6, "checker")])
def test_fast_solve_on_device_inputs_is_identical(problem, q, kind):
    p = problem(q, kind)
    grid = gb.build_grid(q)
    c = _coeff(grid, kind)
    Md = gb.assemble_mass(grid, device=True)
    Ad = gb.assemble_stiffness(grid, c, device=True)
    load = gb.assemble_load(grid, p.load.g_nodal, mass=Md)
    ref = gb.fast_solve(p.M, p.A, p.load, p.tree, 1e-13, uniform_rho=3, c_tol=1e-6)
    res = gb.fast_solve(Md, Ad, load, p.tree, 1e-13, uniform_rho=3, c_tol=1e-6)
    assert np.array_equal(res.solution.u, ref.solution.u)
    for k in (q, q - 1):
        a, b = res.levels[k].stiffness, ref.levels[k].stiffness
        assert np.array_equal(a.data, b.data) and np.array_equal(a.indices, b.indices)


def test_device_assembly_rejects_bad_input():
    grid = gb.build_grid(3)
    other = gb.build_grid(4)
    with pytest.raises(gb.InvalidArgumentError):
        gb.assemble_stiffness(grid, gb.coefficient_example1(other), device=True)
    with pytest.raises(gb.InvalidArgumentError):
        gb.assemble_load(grid, np.zeros(5), device=True)
