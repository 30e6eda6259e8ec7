"""World-size-2 gloo test of bench.py's multi-rank logic (CPU): frame sharding is a disjoint cover
of the batch, each rank's workload is exactly its frames, and the max-over-ranks timing reduction
returns the slowest rank's time on every rank."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from workloads import make
    frames = bench.shard_frames(rank, 2)
    w = make("c5", frames=2, first_frame=frames[0], W=48, H=32, n_cells=6)
    solo = make("c5", frames=1, first_frame=frames[1], W=48, H=32, n_cells=6)
    same = bool(np.array_equal(w.rgb[1], solo.rgb[0]) and np.array_equal(w.t[1], solo.t[0]))
    gathered = [None] * world
    dist.all_gather_object(gathered, frames)
    mx = bench.reduce_max(10.0 + rank, world)
    out[rank] = (gathered, mx, same)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_max():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        gathered, mx, same = res[rank]
        allf = sorted(f for fr in gathered for f in fr)
        assert allf == list(range(4))  # disjoint cover of frames 0..3
        assert mx == 11.0  # the slowest rank's time on every rank
        assert same  # rank-local workload frame == the same frame generated alone (seed 5000+f)


def test_bench_gpus_n_launches_n_ranks():
    """`python bench.py --gpus 2` outside torchrun re-execs itself as 2 ranks (torch.distributed.run
    on 127.0.0.1, gloo in --dry-run); rank 0's line reports n_gpus == 2 and the ranks own a
    disjoint cover of the 2 × frames_per_gpu frames; the max-over-ranks time is the slowest
    rank's (1 + r ms)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--frames-per-gpu", "3",
                          "--dry-run"], capture_output=True, text=True, timeout=300, cwd=root)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["gpus_requested"] == 2
    assert line["frames"] == [[0, 1, 2], [3, 4, 5]]
    assert line["max_ms"] == 2.0
    assert "2 rank(s)" in line["config"]["parallelism"]


def test_bench_rejects_world_mismatch():
    """Under a launcher whose WORLD_SIZE differs from --gpus, bench.py refuses to run rather than
    label a 1-rank time as N GPUs."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--dry-run"],
                         capture_output=True, text=True, timeout=120, cwd=root, env=env)
    assert res.returncode != 0 and "WORLD_SIZE=1" in res.stderr
