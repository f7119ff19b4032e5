"""bench.py's multi-GPU launch on CPU (ADVICE bench.py:64):
`--gpus N` outside torchrun re-launches itself with N ranks, each rank sees
world == N, and the BASELINE minibatch is split into contiguous shards
(strong scaling by default; --scaling weak keeps the per-GPU size)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(*args):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", *args], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    return sorted(lines, key=lambda r: r["rank"])


def test_shards_cover_the_minibatch_contiguously():
    for total in (64, 4096, 1048576, 1001):
        for world in (1, 2, 3, 4, 8):
            parts = [bench.shard(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


@pytest.mark.parametrize("gpus,workload,total,each", [(2, "cfg3", 4096, 2048), (2, "cfg5", 1048576, 524288),
                                                     (1, "cfg3", 4096, 4096)])
def test_spawned_world_and_strong_shards(gpus, workload, total, each):
    rows = _run("--gpus", str(gpus), "--workload", workload)
    assert [r["rank"] for r in rows] == list(range(gpus))
    for r in rows:
        assert r["world"] == gpus == r["gpus"] and r["scaling"] == "strong" and r["total"] == total
        assert r["shard"] == [r["rank"] * each, (r["rank"] + 1) * each]
        assert r["shard_sizes"] == [each] * gpus


def test_weak_scaling_keeps_the_per_gpu_size():
    rows = _run("--gpus", "2", "--scaling", "weak")
    assert [r["shard"] for r in rows] == [[0, 4096], [4096, 8192]] and rows[0]["total"] == 8192


def test_world_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", "--gpus", "2"], env=env,
                         capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "ranks for --gpus 2" in out.stderr
