"""bench.py keeps the driver's JSON-line contract (GPU).

One small C2-shaped run at N = 1, and the N > 1 replica path under
torch.distributed.run with both ranks sharing cuda:0 over gloo
(SRJ_BENCH_SHARE_DEVICE / SRJ_BENCH_BACKEND: a check of the barriers, the max
over ranks and rank 0's single line, never a bench number).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
        "roofline", "clocks", "gpu_launches"}


def _lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _check(d, n_gpus):
    assert KEYS <= set(d)
    assert d["n_gpus"] == n_gpus and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 16 * d["config"]["n"]


def test_bench_line_one_gpu():
    r = subprocess.run([sys.executable, "bench.py", "--size", "512", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    _check(d, 1)
    assert d["config"]["parallelism"] == "single GPU"


def test_bench_replicas_two_ranks_shared_device():
    env = dict(os.environ, SRJ_BENCH_SHARE_DEVICE="1", SRJ_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29531", "bench.py", "--gpus", "2", "--size", "512"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)  # rank 0 alone prints
    _check(d, 2)
    assert d["config"]["parallelism"] == "replicas x2"
    assert "cpu_baseline" not in d  # N = 1 only
