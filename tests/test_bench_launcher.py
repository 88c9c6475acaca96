"""bench.py's multi-rank launcher on CPU ranks (gloo, world size 2).

``bench.py --gpus 2`` without a torchrun environment re-execs itself under
``torch.distributed.run`` with two ranks; ``--dry-run`` swaps the slice
executor for a kernel-free stand-in, so the deal of slice ids (round-robin
per step, ``distributed.partition``), the device-side fold and the single
all-reduce are checked end to end without a GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=240):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    return res


@pytest.mark.parametrize("per_rank", [1, 3])
def test_two_rank_launch_deals_round_robin_and_reduces(per_rank):
    res = _run("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "1", "--slices-per-step", str(per_rank))
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["backend"] == "gloo"
    steps = out["steps"] + out["warmup"]
    for rank, seen in enumerate(out["per_rank_ids"]):
        want = [s * 2 * per_rank + j for s in range(steps) for j in range(2 * per_rank) if j % 2 == rank]
        assert seen == want
    assert out["max_abs_err"] < 1e-9


def test_world_size_mismatch_fails_loudly():
    import os

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert res.returncode != 0
    assert "WORLD_SIZE" in res.stderr
