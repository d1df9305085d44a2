"""bench.py's multi-rank plumbing on a one-GPU box: ``--gpus 2`` re-launches
itself under torch.distributed.run, the ranks rendezvous, split or offset
their replicas, time with barriers and reduce max / sum over ranks, and rank
0 alone prints one JSON line.  MSB_BENCH_SHARE_DEVICE puts both ranks on
cuda:0 with gloo collectives (replica ranks never wait on each other); the
line is marked as a test and its numbers are not measurements."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _bench(*args):
    env = dict(os.environ, MSB_BENCH_SHARE_DEVICE="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_two_ranks_cfg2_weak():
    d = _bench("--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-alt")
    assert d["n_gpus"] == 2 and d["steps"] == 3 and "test_mode" in d
    assert d["config"]["global_replicas"] == 128 and d["config"]["replicas_rank0"] == 64
    S = d["config"]["sweeps_per_step"]
    assert d["config"]["attempts_per_step"] == 2 * 64 * 1024 * 1024 * S  # summed over ranks
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and "cpu_baseline" not in d


def test_two_ranks_cfg3_split():
    d = _bench("--gpus", "2", "--config", "cfg3", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-alt")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_replicas"] == 754 and d["config"]["replicas_rank0"] == 377
    assert d["config"]["attempts_per_step"] == 754 * 512 * 512 * d["config"]["sweeps_per_step"]
