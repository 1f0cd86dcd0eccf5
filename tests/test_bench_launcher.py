"""bench.py's multi-GPU plumbing on CPU: `--gpus 2` outside torchrun must
re-execute the script as two ranks (torch.distributed.run on 127.0.0.1),
shard the config-4 pairs by rank without overlap (weak scaling) and reduce
the work and the timings over ranks -- the real launcher, sharding and
reduction code, with the solve stubbed (--dry-run, gloo)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_relaunches_two_ranks_and_shards_pairs():
    import bench

    out = _run(["--gpus", "2", "--dry-run", "--pairs", "3", "--steps", "2", "--warmup", "3"])
    assert out["n_gpus"] == 2
    assert out["shards"] == [[0, 1, 2], [3, 4, 5]]
    per_pair = sum((n + 1) ** 2 for n in bench.level_sizes())
    assert out["cell_updates"] == 2 * 2 * 3 * per_pair
    assert out["config"]["pairs_per_step"] == 6


def test_bench_single_rank_dry_run():
    out = _run(["--dry-run", "--pairs", "2", "--steps", "1"])
    assert out["n_gpus"] == 1 and out["shards"] == [[0, 1]]


def test_relaunch_command_shape():
    import bench

    class A:
        gpus = 4

    old = os.environ.pop("WORLD_SIZE", None)
    try:
        cmd = bench.relaunch_cmd(A, ["--gpus", "4"])
    finally:
        if old is not None:
            os.environ["WORLD_SIZE"] = old
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-2:] == ["--gpus", "4"]
    A.gpus = 1
    assert bench.relaunch_cmd(A, []) is None
    assert bench.shard(3, 1024) == (3072, 1024)
    assert np.isfinite(bench.cell_updates(np.ones((1, 5))))
