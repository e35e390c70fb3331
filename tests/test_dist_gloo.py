"""Multi-process host logic of the sweep-sharded path on CPU (gloo, world_size 2).

The sharded sweep itself needs NCCL on GPUs (covered by tests/test_gpu_sharded.py on one
GPU with in-process virtual ranks and a world-1 NCCL communicator).  Here: the NCCL
unique-id bootstrap over a torch process group, the edge-balanced shard ranges every rank
computes independently, and the max-over-ranks timing reduction bench.py uses.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    from paper_1805_10904_b200 import dist as lvd

    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    # 1) NCCL unique id from rank 0, broadcast over the gloo group
    uid = lvd.nccl_unique_id() if rank == 0 else None
    uid = lvd.broadcast_bytes(uid, 0)
    objs = [None] * world
    dist.all_gather_object(objs, uid)
    out["uid_equal"] = all(o == objs[0] for o in objs) and len(uid) == 128
    # 2) shard ranges: same seeded CSR on every rank, each keeps its own range
    rng = np.random.default_rng(123)
    deg = rng.zipf(1.8, 5000).clip(0, 3000)
    deg[rng.random(5000) < 0.3] = 0
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    b = lvd.shard_bounds(rp, world)
    mine = (int(b[rank]), int(b[rank + 1]))
    ranges = [None] * world
    dist.all_gather_object(ranges, mine)
    out["ranges"] = ranges
    out["rp_last"] = int(rp[-1])
    out["maxdeg"] = int(deg.max())
    out["n"] = len(deg)
    out["edges"] = [int(rp[hi] - rp[lo]) for lo, hi in ranges]
    # 3) max over ranks (bench.py timing rule)
    out["allmax"] = lvd.allmax(1.5 + rank)
    lvd.barrier()
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.parametrize("world", [2])
def test_gloo_sharding_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["uid_equal"]
        assert res[r]["allmax"] == 1.5 + world - 1
    ranges = res[0]["ranges"]
    assert ranges == res[1]["ranges"]
    # contiguous tiling of [0, n)
    assert ranges[0][0] == 0 and ranges[-1][1] == res[0]["n"]
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    # edge balance: every shard within one row of nnz/world
    nnz, maxdeg = res[0]["rp_last"], res[0]["maxdeg"]
    assert sum(res[0]["edges"]) == nnz
    for e in res[0]["edges"]:
        assert abs(e - nnz / world) <= maxdeg


def _bench(*args, timeout=600):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=root)
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return p.returncode, lines, p.stderr


def test_bench_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` with no launcher spawns 2 local ranks (torchrun environment,
    127.0.0.1 rendezvous); they meet in a gloo group, and only rank 0 prints a line."""
    import json

    rc, lines, err = _bench("--gpus", "2", "--dist-check")
    assert rc == 0, err[-2000:]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["allmax_rank"] == 1.0


def test_bench_reference_arm_world2_rank0_only():
    """--impl reference under N ranks: rank 0 alone runs the oracle and prints one line."""
    import json

    rc, lines, err = _bench("--gpus", "2", "--impl", "reference", "--workload", "karate", "--steps", "2",
                            "--warmup", "1")
    assert rc == 0, err[-2000:]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["same_config"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0
