"""Spatially partitioned transform + solve (gamblet_dist.py) against the
single-GPU path: `world` in-process ranks (threads, one CUDA stream each,
comm.ThreadComm) run the multi-GPU program on one device.  The transform must
be bitwise the single-GPU transform on every rank's rows; the solution agrees
to the solver tolerance (the distributed reductions sum in another order)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

EPS, RHO = 1e-13, 3


def _inputs(q, coeff="checker"):
    import paper_1503_03467_b200 as gb
    grid = gb.build_grid(q)
    if coeff == "example1":
        c = gb.coefficient_example1(grid)
        g = gb.example_load(grid)
    else:
        c = gb.coefficient_checkerboard(grid, 1e4, 0)
        g = np.random.default_rng(1).standard_normal(grid.num_nodes)
    M = gb.assemble_mass(grid)
    A = gb.assemble_stiffness(grid, c)
    return grid, M, A, g, gb.build_hierarchy(grid)


def _single(M, A, g, tree):
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import device as dv, gamblet_fast as gf
    sched = gb.make_schedule(EPS, tree.q, uniform_rho=RHO)
    levels, parts, U1, counter = gf._fast_solve_device(
        dv.DeviceCSR.from_scipy(M), dv.DeviceCSR.from_scipy(A), dv.to_dev(g), tree, sched)
    torch.cuda.synchronize()
    return levels, parts["partials"].device(tree.q), counter


def _rank_body(comm, M, A, g, tree):
    from paper_1503_03467_b200 import gamblet_dist as gd
    return gd.fast_solve_dist(comm, M, A, g, tree, EPS, uniform_rho=RHO, keep=True)


def _check_rows(name, k, ref, rows_list, L, row_elems):
    """The ranks' own rows, concatenated, are bitwise the whole level."""
    for r, rows in enumerate(rows_list):
        p0, p1 = L * r // len(rows_list), L * (r + 1) // len(rows_list)
        got = rows.rows(p0, p1)
        want = ref[p0 * row_elems:p1 * row_elems]
        assert torch.equal(got, want), f"{name}^({k}) rows [{p0},{p1}) of rank {r} differ"


@pytest.mark.parametrize("q,world,coeff", [(7, 2, "checker"), (7, 4, "example1"),
                                           (8, 8, "checker"), (9, 2, "checker"),
                                           (9, 4, "checker"), (10, 2, "checker"),
                                           (10, 8, "checker")])
def test_partitioned_transform_bitwise_and_solution(q, world, coeff):
    from paper_1503_03467_b200 import comm as cm, device as dv
    grid, M, A, g, tree = _inputs(q, coeff)
    levels, u_ref, counter = _single(M, A, g, tree)
    out = cm.run_threads(world, _rank_body, M, A, g, tree, device=dv.device())
    torch.cuda.synchronize()
    kr = out[0].first_replicated
    assert kr < q, "nothing was distributed"
    n = 1 << q
    for k in range(q, kr - 1, -1):
        L = 1 << k
        ref = levels[k]
        A_ref = ref.raw("stiffness")
        _check_rows("A", k, A_ref.vals, [o.strips[k]["A"] for o in out], L, L * A_ref.slots)
        assert out[0].strips[k]["wA"] == A_ref.w
        psi_ref = ref.raw("psi")
        _check_rows("psi", k, psi_ref.vals, [o.strips[k]["psi"] for o in out], L,
                    L * psi_ref.wd ** 2)
        if k > kr:
            Lp = L // 2
            B = ref.raw("subband")
            _check_rows("B", k, B.vals, [o.strips[k]["B"] for o in out], Lp, Lp * 3 * B.slots)
            D = ref.raw("correction")
            _check_rows("Dt", k, D.vals, [o.strips[k]["Dt"] for o in out], Lp, Lp * D.slots)
            R = ref.raw("restriction")
            _check_rows("R", k, R.vals, [o.strips[k]["R"] for o in out], Lp, Lp * R.slots)
            sB = ref.raw("subband_scale")
            _check_rows("sB", k, sB, [o.strips[k]["sB"] for o in out], Lp, Lp * 3)
    # replicated levels: identical on every rank and bitwise the single-GPU levels
    for k in range(kr, 0, -1):
        for o in out:
            lv = o.levels[k]
            assert torch.equal(lv.raw("stiffness").vals, levels[k].raw("stiffness").vals), k
            if k >= 2:
                assert torch.equal(lv.raw("subband").vals, levels[k].raw("subband").vals), k
                assert torch.equal(lv.raw("restriction").vals,
                                   levels[k].raw("restriction").vals), k
    # column strips of the coarse psi: every rank's fine rows of every window
    for k in range(kr - 1, 0, -1):
        ref = levels[k].raw("psi")
        L, wd = 1 << k, ref.wd
        h = n // L
        org = np.clip(np.arange(L) * h + ref.lo, 0, n - wd)
        want = ref.vals.view(L, L, wd, wd)
        for r, o in enumerate(out):
            f0, f1 = n * r // world, n * (r + 1) // world
            got = o.levels[k].raw("psi").vals.view(L, L, wd, wd)
            for i in range(L):
                a, b = max(f0 - org[i], 0), min(f1 - org[i], wd)
                if b > a:
                    assert torch.equal(got[i, :, a:b, :], want[i, :, a:b, :]), (k, r, i)
    # solution: same on every rank, equal to the single-GPU one to the solver tolerance
    for o in out:
        assert torch.equal(o.u, out[0].u)
    err = float((out[0].u - u_ref).norm() / u_ref.norm())
    assert err <= 1e-9, err
    # lambda estimates and iteration counts of the distributed levels
    its = {k: counter.solves[f"line8 level {k}"][0][0] for k in range(2, q + 1)}
    for k in range(q, 1, -1):
        lmin, lmax = out[0].lambdas[k]
        assert lmax == pytest.approx(levels[k].lambda_max_subband, rel=1e-6), k
        assert lmin == pytest.approx(levels[k].lambda_min_subband, rel=2e-4), k
    for k in range(q, kr, -1):
        assert abs(out[0].iterations[k] - its[k]) <= 3, (k, out[0].iterations[k], its)


def test_world_one_is_the_single_gpu_program():
    from paper_1503_03467_b200 import comm as cm, gamblet_dist as gd
    grid, M, A, g, tree = _inputs(6)
    levels, u_ref, _ = _single(M, A, g, tree)
    res = gd.fast_solve_dist(cm.SelfComm(), M, A, g, tree, EPS, uniform_rho=RHO)
    assert torch.equal(res.u, u_ref)


def test_per_rank_memory_shrinks_with_world():
    """Peak device memory of a rank's distributed-level operators ~ 1 / world."""
    from paper_1503_03467_b200 import comm as cm, device as dv, gamblet_dist as gd
    grid, M, A, g, tree = _inputs(9)

    def body(comm):
        res = gd.fast_solve_dist(comm, M, A, g, tree, EPS, uniform_rho=RHO, keep=True)
        held = 0
        for k, d in res.strips.items():
            for v in d.values():
                if isinstance(v, gd.Rows):
                    held += v.nbytes
        return held

    one = None
    for world in (2, 4):
        held = cm.run_threads(world, body, device=dv.device())
        if one is None:
            one = held[0] * world
        # strips + halos: within 35% of an even split of the same operators
        assert max(held) <= 1.35 * one / world, (world, held, one)


def _proc_worker(rank, world, port, q, out_dir):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1503_03467_b200 as gb
    grid, M, A, g, tree = _inputs(q)
    res = gb.fast_solve_dist(gb.TorchComm(), M, A, g, tree, EPS, uniform_rho=RHO, keep=True)
    L = 1 << q
    p0, p1 = L * rank // world, L * (rank + 1) // world
    np.save(f"{out_dir}/u_{rank}.npy", res.u.cpu().numpy())
    np.save(f"{out_dir}/A_{rank}.npy", res.strips[q]["A"].rows(p0, p1).cpu().numpy())
    np.save(f"{out_dir}/meta_{rank}.npy", np.array([res.first_replicated, res.halo_bytes]))
    dist.destroy_process_group()


def test_two_processes_gloo_share_the_gpu(tmp_path):
    """The real multi-process path (torch.distributed, one process per rank):
    two gloo ranks on the one GPU run the partitioned solve on q = 8 level
    data (rows staged through the host) and reproduce the single-GPU result."""
    import socket
    import torch.multiprocessing as mp
    q, world = 8, 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    # the children allocate on the same device: hand the cached blocks back first
    import gc
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    mp.spawn(_proc_worker, args=(world, port, q, str(tmp_path)), nprocs=world, join=True)
    grid, M, A, g, tree = _inputs(q)
    levels, u_ref, _ = _single(M, A, g, tree)
    us = [np.load(tmp_path / f"u_{r}.npy") for r in range(world)]
    assert np.array_equal(us[0], us[1])
    ur = u_ref.cpu().numpy()
    assert np.linalg.norm(us[0] - ur) <= 1e-9 * np.linalg.norm(ur)
    Aq = levels[q].raw("stiffness")
    got = np.concatenate([np.load(tmp_path / f"A_{r}.npy") for r in range(world)])
    assert np.array_equal(got, Aq.vals.cpu().numpy())
    meta = np.load(tmp_path / "meta_0.npy")
    assert meta[0] < q and meta[1] > 0


def test_strip_program_on_one_rank_matches_the_pipeline():
    """force_strips: the partitioned code path with a single strip (no
    exchange) -- same transform bits, same solution to the solver tolerance."""
    from paper_1503_03467_b200 import comm as cm, gamblet_dist as gd
    q = 7
    grid, M, A, g, tree = _inputs(q)
    levels, u_ref, _ = _single(M, A, g, tree)
    res = gd.fast_solve_dist(cm.SelfComm(), M, A, g, tree, EPS, uniform_rho=RHO, keep=True,
                             force_strips=True)
    assert res.first_replicated < q
    for k in range(q, res.first_replicated - 1, -1):
        L = 1 << k
        assert torch.equal(res.strips[k]["A"].rows(0, L), levels[k].raw("stiffness").vals), k
        assert torch.equal(res.strips[k]["psi"].rows(0, L), levels[k].raw("psi").vals), k
    err = float((res.u - u_ref).norm() / u_ref.norm())
    assert err <= 1e-9, err


def test_partition_rejects_a_world_that_is_not_a_power_of_two():
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import comm as cm
    grid, M, A, g, tree = _inputs(6)

    class Three(cm.SelfComm):
        world = 3

    with pytest.raises(gb.InvalidArgumentError):
        gb.fast_solve_dist(Three(), M, A, g, tree, EPS, uniform_rho=RHO)


def test_non_spd_operator_raises_on_every_rank():
    """An indefinite stiffness surfaces as NumericalError on all ranks (the
    status words and repair statistics are all-reduced before the check, the
    Krylov breakdown flags come from all-reduced sums)."""
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import comm as cm, device as dv
    q = 8
    grid, M, A, g, tree = _inputs(q)
    Aneg = (-A).tocsr()
    seen = []

    def body(comm):
        try:
            gb.fast_solve_dist(comm, M, Aneg, g, tree, EPS, uniform_rho=RHO)
        except gb.NumericalError as e:
            seen.append((comm.rank, str(e)))
            return "raised"
        return "returned"

    out = cm.run_threads(2, body, device=dv.device())
    assert out == ["raised", "raised"], (out, seen)
