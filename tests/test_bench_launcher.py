"""bench.py's multi-rank launcher on CPU: `python bench.py
--gpus 2 --stub` re-launches itself under torch.distributed.run (gloo), every rank computes its
shard and times its stubbed work between barriers, and rank 0 alone prints one JSON line with
the max-over-ranks time and the shard bounds of the weak and strong legs."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [1, 2, 3])
def test_bench_self_launch_stub(n):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK",
                                                              "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--stub",
                        "--steps", "4", "--warmup", "3"], capture_output=True, text=True, timeout=300,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    j = json.loads(lines[0])
    assert j["n_gpus"] == n and j["stub"] is True
    # the slowest rank (rank n-1 sleeps n ms per step) sets the time: max over ranks
    assert j["ms_per_step"] >= n * 1.0 * 0.9
    shards = j["config"]["strong_shards"]
    assert len(shards) == n and shards[0][0] == 0
    assert sum(c for _, c in shards) == 256 and all(b0 + c == b1 for (b0, c), (b1, _) in zip(shards, shards[1:]))
    assert j["config"]["weak_shard_rank0"] == [0, 16]
    assert j["value"] == pytest.approx(n * 2048 * 4 / (j["ms_per_step"] * 4 / 1e3), rel=1e-6)


def test_bench_rejects_mismatched_world():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode == 2
