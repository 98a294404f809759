"""The exchange layer of the spatial partition (comm.py) on CPU tensors:
in-process thread ranks and a world-size-2 gloo process group move rows of a
real level operator (the oracle's A^(5) in box layout) and reduce scalars."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_03467_b200 import comm as cm
from paper_1503_03467_b200.partition import row_strips


def _level_box(q=5, w=3):
    """A^(q) of the oracle at q (contrast 1e4) as box rows: L x L grid rows of
    L * (2w+1)^2 values (the layout the kernels exchange)."""
    import paper_1503_03467_b200 as gb
    from oracle import gamblets_oracle as O
    grid = gb.build_grid(q)
    M = gb.assemble_mass(grid)
    A = gb.assemble_stiffness(grid, gb.coefficient_checkerboard(grid, 1e4, 0))
    psi = O.mass_inverse(M, q, 1)
    Aq, _ = O.level_q_stiffness(psi, A)
    L = 1 << q
    S = (2 * w + 1) ** 2
    box = np.zeros((L * L, S))
    Aq = Aq.tocoo()
    rs, rt = Aq.row // L, Aq.row % L
    ds, dt = Aq.col // L - rs, Aq.col % L - rt
    keep = (np.abs(ds) <= w) & (np.abs(dt) <= w)
    box[Aq.row[keep], (ds[keep] + w) * (2 * w + 1) + dt[keep] + w] = Aq.data[keep]
    return torch.from_numpy(box.ravel().copy()), L, L * S


def _exercise(comm, full, L, row_elems):
    """Every collective on this rank's strip of `full`; returns what it saw."""
    r0, r1 = comm.strip(L)
    up, down = 3, 5
    buf = torch.full_like(full, float("nan"))
    buf[r0 * row_elems:r1 * row_elems] = full[r0 * row_elems:r1 * row_elems]
    comm.halo(buf, L, row_elems, up, down)
    a, b = max(r0 - up, 0), min(r1 + down, L)
    ok_halo = torch.equal(buf[a * row_elems:b * row_elems], full[a * row_elems:b * row_elems])
    untouched = bool(torch.isnan(buf[:a * row_elems]).all() and
                     torch.isnan(buf[b * row_elems:]).all())
    # halo_add: every rank contributes (rank + 1) to the rows it holds around its strip
    acc = torch.zeros(L * 4, dtype=torch.float64)
    acc[a * 4:b * 4] = comm.rank + 1.0
    comm.halo_add(acc, L, 4, up, down)
    own = acc[r0 * 4:r1 * 4].clone()
    # all-reduce and all-gather
    t = torch.tensor([comm.rank + 1.0, -float(comm.rank)], dtype=torch.float64)
    tsum = comm.allreduce(t.clone(), "sum")
    tmax = comm.allreduce(t.clone(), "max")
    tmin = comm.allreduce(t.clone(), "min")
    g = torch.zeros_like(full)
    g[r0 * row_elems:r1 * row_elems] = full[r0 * row_elems:r1 * row_elems]
    comm.allgather_rows(g, L, row_elems)
    bc = torch.full((5,), float(comm.rank), dtype=torch.float64)
    comm.broadcast(bc, comm.world - 1)
    assert torch.equal(bc, torch.full((5,), comm.world - 1.0, dtype=torch.float64))
    return dict(ok_halo=ok_halo, untouched=untouched, own=own.numpy(), tsum=tsum.numpy(),
                tmax=tmax.numpy(), tmin=tmin.numpy(), gathered=torch.equal(g, full),
                strip=(r0, r1))


def _expect_halo_add(L, world, up, down):
    """Sum over ranks of (rank + 1) on [r0 - up, r1 + down) -- per grid row."""
    tot = np.zeros(L)
    for r, (r0, r1) in enumerate(row_strips(L, world)):
        tot[max(r0 - up, 0):min(r1 + down, L)] += r + 1.0
    return tot


@pytest.mark.parametrize("world", [2, 4, 8])
def test_thread_ranks_exchange_level_rows(world):
    full, L, row_elems = _level_box()
    out = cm.run_threads(world, _exercise, full, L, row_elems)
    want = _expect_halo_add(L, world, 3, 5)
    for r, o in enumerate(out):
        assert o["ok_halo"] and o["untouched"] and o["gathered"], (r, o)
        r0, r1 = o["strip"]
        assert np.array_equal(o["own"].reshape(-1, 4)[:, 0], want[r0:r1])
        assert np.array_equal(o["tsum"], [world * (world + 1) / 2, -world * (world - 1) / 2])
        assert np.array_equal(o["tmax"], [world, 0.0])
        assert np.array_equal(o["tmin"], [1.0, -(world - 1.0)])


def test_halo_wider_than_a_strip_reaches_the_second_neighbour():
    L, row = 16, 3
    full = torch.arange(L * row, dtype=torch.float64)

    def body(comm):
        r0, r1 = comm.strip(L)
        buf = torch.full_like(full, -1.0)
        buf[r0 * row:r1 * row] = full[r0 * row:r1 * row]
        comm.halo(buf, L, row, 5, 5)  # strips have 4 rows
        a, b = max(r0 - 5, 0), min(r1 + 5, L)
        return torch.equal(buf[a * row:b * row], full[a * row:b * row])

    assert all(cm.run_threads(4, body))


def _gloo_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full, L, row_elems = _level_box()
    res = _exercise(cm.TorchComm(), full, L, row_elems)
    out[rank] = res
    dist.destroy_process_group()


def test_two_rank_gloo_exchange_level_rows():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gloo_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    L = 32
    want = _expect_halo_add(L, 2, 3, 5)
    for r in (0, 1):
        o = res[r]
        assert o["ok_halo"] and o["untouched"] and o["gathered"]
        r0, r1 = o["strip"]
        assert np.array_equal(o["own"].reshape(-1, 4)[:, 0], want[r0:r1])
        assert np.array_equal(o["tsum"], [3.0, -1.0])
        assert np.array_equal(o["tmax"], [2.0, 0.0]) and np.array_equal(o["tmin"], [1.0, -1.0])


def test_window_reach_matches_brute_force():
    from paper_1503_03467_b200.gamblet_dist import _window_reach, min_distributed_rows
    n, L, lo, wd = 256, 64, -45, 98
    up, dn = _window_reach(n, L, lo, wd, 4)
    h = n // L
    org = np.clip(np.arange(L) * h + lo, 0, n - wd)
    for r in range(4):
        p0, p1 = L * r // 4, L * (r + 1) // 4
        for i in range(L):
            hits = org[i] < p1 * h and org[i] + wd > p0 * h
            if hits:
                assert p0 - up <= i < p1 + dn
    assert min_distributed_rows(2) == 64 and min_distributed_rows(8) == 128
