"""N>1 plumbing of bench.py on CPU: gloo, world size 2.

The path shards as replicas over RB shards: every rank detects
its own seeded workload, the only collectives are the barrier and the
max-over-ranks timing reduction.  Here each rank runs the oracle on its shard
(the checker; the GPU path is not needed to test the plumbing)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from oracle import mpnl_oracle as orc
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = CONFIGS["C1"]
        d = generate(cfg, seed=bench.rank_seed(2409, rank), n_rb=1)
        c = constellation_for(cfg.order)
        hard, metric = orc.detect_rb(d["h"], d["y"], d["nv"][0], cfg.n_paths, cfg.order,
                                     c.points)[:2]
        fake_ms = 10.0 * (rank + 1)                       # rank 1 is the slow one
        tmax = bench.max_over_ranks(fake_ms, world)
        dist.barrier()
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, np.asarray(hard).tobytes(), tmax))
        if rank == 0:
            out.put(gathered)
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank sees the max over ranks
    assert [g[2] for g in gathered] == [20.0, 20.0]
    # ranks detect different (independently seeded) shards
    assert gathered[0][1] != gathered[1][1]
    # each rank's shard equals what a single process computes for that seed
    cfg = CONFIGS["C1"]
    c = constellation_for(cfg.order)
    for r in range(world):
        d = generate(cfg, seed=bench.rank_seed(2409, r), n_rb=1)
        hard = orc.detect_rb(d["h"], d["y"], d["nv"][0], cfg.n_paths, cfg.order, c.points)[0]
        assert np.asarray(hard).tobytes() == gathered[r][1]


def test_job_rate_is_whole_job_over_slowest_rank():
    # 2 ranks x 1000 vectors, slowest rank 10 ms per step over 5 steps
    assert bench.job_rate(1000, 2, 50.0, 5) == pytest.approx(2000 / 0.010)
    assert bench.max_over_ranks(3.5, 1) == 3.5
