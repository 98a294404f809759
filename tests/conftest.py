"""Shared fixtures: golden fixtures (generated from the reference by
oracle/make_goldens.py), cached problems built with the package's host-side
input builders, and the CPU oracle."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]

# the q=12 test (tests/test_gpu_q12.py) needs the settings bench.py uses for
# q >= 12; both must be in place before CUDA and the package initialize
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
os.environ.setdefault("GB_SPECTRAL_WORKERS", "3")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: larger GPU parity case")


class Golden:
    """Read-only view of one tests/golden/*.npz fixture."""

    def __init__(self, name):
        self.name = name
        self.z = np.load(GOLDEN / f"{name}.npz")

    def __contains__(self, key):
        return key in self.z.files or f"{key}/data" in self.z.files

    def __getitem__(self, key):
        if f"{key}/data" in self.z.files:
            shape = tuple(self.z[f"{key}/shape"])
            return sp.csr_array((self.z[f"{key}/data"], self.z[f"{key}/indices"],
                                 self.z[f"{key}/indptr"]), shape=shape)
        v = self.z[key]
        return v.item() if v.shape == () and v.dtype.kind in "fiU" else v


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]

    return get


def build_problem(q, coeff):
    import paper_1503_03467_b200 as gb
    grid = gb.build_grid(q)
    if coeff == "example1":
        c = gb.coefficient_example1(grid)
        g = gb.example_load(grid)
    elif coeff == "checker":
        c = gb.coefficient_checkerboard(grid, 1e4, 0)
        g = np.random.default_rng(1).standard_normal(grid.num_nodes)
    elif coeff == "constant":
        c = gb.coefficient_constant(grid)
        g = gb.example_load(grid)
    else:
        raise ValueError(coeff)
    M = gb.assemble_mass(grid)
    A = gb.assemble_stiffness(grid, c)
    load = gb.assemble_load(grid, g, mass=M)
    tree = gb.build_hierarchy(grid)
    from types import SimpleNamespace
    return SimpleNamespace(q=q, grid=grid, coef=c, M=M, A=A, load=load, tree=tree)


@pytest.fixture(scope="session")
def problem():
    cache = {}

    def get(q, coeff="example1"):
        if (q, coeff) not in cache:
            cache[(q, coeff)] = build_problem(q, coeff)
        return cache[(q, coeff)]

    return get


@pytest.fixture(scope="session")
def oracle_fast(problem):
    """Factory: tight-mode oracle fast_solve (uniform rho=3), cached."""
    from oracle import gamblets_oracle as O
    cache = {}

    def run(q, coeff="example1", epsilon=1e-13, uniform_rho=3):
        key = (q, coeff, epsilon, uniform_rho)
        if key not in cache:
            p = problem(q, coeff)
            cache[key] = O.fast_solve(p.M, p.A, p.load.g_nodal, q, epsilon,
                                      uniform_rho=uniform_rho)
        return cache[key]

    return run
