"""N > 1 host logic of bench.py on CPU (gloo, world size 2): every rank gets the max of the
per-rank times, the whole-job value counts the cells of all ranks, and ranks run independent
problems of the same shape."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = [1.0 + rank, 10.0 - rank]  # per-rank step / e2e times (ms)
        got = bench.reduce_max_over_ranks(mine, dist, "cpu")
        out[rank] = got
    finally:
        dist.destroy_process_group()


def test_reduce_max_two_ranks_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0] == res[1] == [2.0, 10.0]


def test_single_rank_passthrough_and_value():
    assert bench.reduce_max_over_ranks([3.5, 4.0], None) == [3.5, 4.0]
    # 2 ranks x 1000 cells in 2 ms (slowest rank) -> 1e6 cell-updates/s
    assert bench.whole_job_value(1000, 2, 2.0) == pytest.approx(1.0e6)


def test_ranks_run_independent_problems_of_one_shape():
    from paper_2301_01718_b200 import inputs
    a = inputs.config(4, nx=64, ny=64, seed=bench.rank_seed(4, 0))
    b = inputs.config(4, nx=64, ny=64, seed=bench.rank_seed(4, 1))
    qa, qb = inputs.initial_condition(a), inputs.initial_condition(b)
    assert qa.shape == qb.shape and not (qa == qb).all()
