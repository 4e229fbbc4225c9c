"""bench.py's multi-GPU launch path, runnable on a one-GPU box: --gpus 2
outside torchrun must spawn two ranks itself (torch.distributed.run), shard
the edge slots and all-reduce the histogram; with the gloo backend both
ranks share cuda:0 (a functional check, not a measurement).  The sharded
estimate must equal the one-rank estimate (the histogram is exact)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(gpus, extra_env=None):
    env = dict(os.environ, **(extra_env or {}))
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(gpus), "--config", "c2",
           "--steps", "2", "--warmup", "3", "--no-secondary", "--no-cpu-baseline",
           "--e2e-steps", "0", "--no-busy"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def test_bench_spawns_ranks_and_matches_single_rank():
    one = _bench(1)
    two = _bench(2, {"PG_BENCH_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["estimate"] == one["estimate"]
    assert two["layout"]["edges_per_rank"] < one["layout"]["edges_per_rank"]


def test_bench_rejects_mismatched_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2"],
                         env=env, capture_output=True, text=True, timeout=120, cwd=REPO)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
