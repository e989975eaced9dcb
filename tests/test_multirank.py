"""N>1 plumbing of bench.py on CPU: gloo, world size 2.

The path shards over RB ranges with no data-path collective:
each rank detects its own contiguous RB range; the only collectives are the
barrier and the max-over-ranks timing reduction.  Here each rank runs the
checker (oracle) on its shard — the plumbing does not need the GPU path — and
the concatenated shards must equal one process over the whole range
(the reference's own bit-identity-across-workers contract,
test_acceptance.py:237-247)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from oracle import mpnl_oracle as orc
from paper_2409_14355_b200.core import constellation_for
from paper_2409_14355_b200.workloads import CONFIGS, generate

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _detect(cfg, n_rb, rb0):
    d = generate(cfg, n_rb=n_rb, rb_offset=rb0)
    c = constellation_for(cfg.order)
    return orc.detect_rb(d["h"], d["y"], d["nv"][0], cfg.n_paths, cfg.order, c.points)[0]


def _worker(rank, world, port, scaling, total_rb, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = CONFIGS["C1"]
        n_rb, rb0 = bench.shard(total_rb, rank, world, scaling)
        hard = _detect(cfg, n_rb, rb0)
        fake_ms = 10.0 * (rank + 1)                       # rank 1 is the slow one
        tmax = bench.max_over_ranks(fake_ms, world)
        dist.barrier()
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, rb0, np.asarray(hard), tmax))
        if rank == 0:
            out.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scaling,total_rb", [("strong", 5), ("weak", 2)])
def test_two_rank_rb_shards_gloo(scaling, total_rb):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scaling, total_rb, q))
             for r in range(world)]
    for p in procs:
        p.start()
    gathered = sorted(q.get(timeout=240), key=lambda g: g[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [g[3] for g in gathered] == [20.0, 20.0]          # max over ranks everywhere
    cat = np.concatenate([g[2] for g in gathered])
    whole = total_rb if scaling == "strong" else world * total_rb
    assert cat.shape[0] == whole
    # the shards concatenate to one process's detection of the whole RB range
    assert np.array_equal(cat, _detect(CONFIGS["C1"], whole, 0))


def test_shard_ranges_partition():
    for n, w in ((2048, 8), (273, 4), (5, 2), (1, 1)):
        rs = [bench.shard(n, r, w, "strong") for r in range(w)]
        assert sum(k for k, _ in rs) == n
        assert [o for _, o in rs] == sorted(o for _, o in rs)
        assert all(rs[i][1] + rs[i][0] == rs[i + 1][1] for i in range(w - 1))
        assert [bench.shard(n, r, w, "weak") for r in range(w)] == [(n, r * n) for r in range(w)]


def test_job_rate_is_whole_job_over_slowest_rank():
    # 2000 vectors in all, slowest rank 10 ms per step over 5 steps
    assert bench.job_rate(2000, 50.0, 5) == pytest.approx(2000 / 0.010)
    assert bench.max_over_ranks(3.5, 1) == 3.5


def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` with no launcher re-runs itself under
    torch.distributed.run; with the reference arm rank 0 prints one line and
    rank 1 exits 0 (no GPU needed)."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--config", "C1", "--steps", "1", "--warmup", "0",
                        "--ref-step-s", "0.2"], capture_output=True, text=True, env=env,
                       timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["value"] > 0
