"""World-size-2 gloo checks (CPU) of the multi-GPU host logic of bench.py: sentence sharding gives
disjoint per-rank inputs (weak scaling, no data-path collective) and the job time is the max over
ranks while the word-score count is the sum (bench.py reduce_max / reduce_sum)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import synth
    t = bench.reduce_max(1.0 + rank, dist)
    n = bench.reduce_sum(100.0 * (rank + 1), dist)
    src = synth.make_source(50000, 49, seed=bench.shard_seed(rank, 0))
    q.put((rank, t, n, src.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_reductions_and_sharding_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == 2.0 for r in res)          # max over ranks
    assert all(r[2] == 300.0 for r in res)        # total work over ranks
    assert res[0][3] != res[1][3]                 # each rank scores its own sentences


def test_shard_seeds_disjoint():
    import bench
    seeds = {bench.shard_seed(r, s) for r in range(8) for s in range(1000)}
    assert len(seeds) == 8000


def test_c5_lpt_sharding_partitions_and_balances():
    """tools/workloads.py lpt_shard (C5 sentence sharding over ranks): a partition of
    the sentences, deterministic, and within the greedy-LPT bound max load <= 4/3 OPT + 1 job."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import numpy as np
    import workloads
    rng = np.random.default_rng(0)
    costs = [int(x) * 64 for x in rng.integers(11, 52, size=3000)]
    for world in (1, 2, 4, 8):
        sh = workloads.lpt_shard(costs, world)
        assert sorted(i for s in sh for i in s) == list(range(len(costs)))
        assert sh == workloads.lpt_shard(costs, world)
        loads = [sum(costs[i] for i in s) for s in sh]
        lower = max(sum(costs) / world, max(costs))
        assert max(loads) <= 4 / 3 * lower + max(costs)
        assert max(loads) - min(loads) <= max(costs)


def test_bench_launcher_spawns_ranks():
    """`python bench.py --gpus 2` without torchrun in the environment starts torchrun itself (2 ranks,
    127.0.0.1 rendezvous) and exactly one JSON line comes back, with n_gpus = 2 (the reference arm runs
    on the host, so this works without a GPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["impl"] == "reference" and j["value"] > 0


def test_bench_rejects_mismatched_world():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
