"""World-size-2 gloo tests of the N>1 host logic (CPU): per-rank instances,
max-over-ranks timing, whole-job rate aggregation, barrier."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_1503_03467_b200 as gb
    # every rank builds a distinct seeded instance of the same family
    grid, M, A, load, tree = bench.build_inputs(3, "checker", rank)
    digest = float(np.abs(A.data).sum() + np.abs(load.g_nodal).sum())
    gathered = [None] * world
    dist.all_gather_object(gathered, digest)
    # timing reduction: max over ranks
    ms = 10.0 + 5.0 * rank
    mx = bench.reduce_max(ms, world)
    rate = bench.whole_job_rate(4 ** 3, world, mx)
    dist.barrier()
    out[rank] = (gathered, mx, rate, bench.instance_seeds(rank))
    dist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    g0, mx0, rate0, seeds0 = res[0]
    g1, mx1, rate1, seeds1 = res[1]
    assert g0 == g1 and g0[0] != g0[1]          # distinct instances per rank
    assert mx0 == mx1 == 15.0                   # max over ranks
    assert rate0 == rate1 == pytest.approx(2 * 64 / 15e-3)
    assert seeds0 == (0, 1) and seeds1 == (2, 3)  # rank 0 = BASELINE seeds


def test_single_process_reduce_is_identity():
    import bench
    assert bench.reduce_max(3.5, 1) == 3.5
    assert bench.whole_job_rate(100, 1, 1000.0) == pytest.approx(100.0)


def test_row_strips_partition():
    from paper_1503_03467_b200.partition import row_strips
    for L in (0, 1, 7, 64, 513):
        for world in (1, 2, 3, 8):
            s = row_strips(L, world)
            assert len(s) == world and s[0][0] == 0 and s[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
            sizes = [b - a for a, b in s]
            assert max(sizes) - min(sizes) <= 1


def _strips_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1503_03467_b200 import partition as part
    L, row = 13, 5  # 13 grid rows of 5 elements: strips of 7 and 6 rows
    strips = part.Strips(world, rank, distributed=True)
    buf = torch.full((L * row,), -1.0, dtype=torch.float64)
    solved = []

    def solve(r0, r1):  # this rank's "patch solves": row index + 100 * rank
        solved.append((r0, r1))
        for r in range(r0, r1):
            buf[r * row:(r + 1) * row] = r + 100.0 * rank

    part.run_strips(strips, L, row, buf, solve)
    out[rank] = (solved, buf.numpy().copy())
    dist.destroy_process_group()


def test_two_rank_gloo_strip_exchange():
    """Each rank solves only its strip; after the exchange both hold the
    whole level, every row written by its owner."""
    from paper_1503_03467_b200.partition import row_strips
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_strips_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    strips = row_strips(13, 2)
    expect = np.concatenate([np.full(5, r + 100.0 * owner)
                             for owner, (a, b) in enumerate(strips) for r in range(a, b)])
    for rank in (0, 1):
        solved, buf = res[rank]
        assert solved == [strips[rank]]
        assert np.array_equal(buf, expect)
