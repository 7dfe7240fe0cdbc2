"""bench.py --gpus N without torchrun spawns N ranks itself (one process per
GPU, 127.0.0.1 rendezvous): the plumbing (spawn, shard tiling of the 2^27
headline points, sum / max all-reduce) checked on CPU with gloo."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("world", [2, 3])
def test_spawn_shards_and_reduces(world):
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(world),
                        "--plumbing-test"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    n = 1 << 27
    assert d["n_gpus"] == world
    shards = d["shards"]
    assert shards[0][0] == 0 and shards[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    assert all(lo % 32 == 0 for lo, _ in shards)
    assert d["points_sum"] == n
    assert d["rank_sum"] == world * (world + 1) / 2
    assert d["max_rank"] == world - 1


def test_world_mismatch_is_an_error():
    import os
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2",
                        "--plumbing-test"], capture_output=True, text=True, timeout=120, env=env)
    assert p.returncode != 0
