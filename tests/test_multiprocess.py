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
