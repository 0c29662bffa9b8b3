"""bench.py --impl reference (CPU): the driver's reference-arm line.

The arm times the oracle port on the host cores (the reference is pure Python;
DESIGN.md section 6).  At N = 1 it prints one line with impl, cpu_baseline and
an e2e block with zero copy bytes; under torch.distributed.run only rank 0
prints and every rank exits 0.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--steps", "1", "--warmup", "1", "--size", "128",
        "--cpu-seconds", "0.5"]


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["unit"] == "GLUP/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GLUP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    host = d["cpu_baseline"]["host"]
    assert host["nproc"] >= 1 and "numpy" in host and "OMP_NUM_THREADS" in host
    stock = d["cpu_baseline"]["reference_stock"]
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "srj")):
        assert stock["kind"] == "reference" and stock["value"] > 0   # the unmodified reference
    else:
        assert "unavailable" in stock
    assert "not a whole solve" in d["config"]["step"]


def test_reference_arm_rank0_only():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", "bench.py", "--gpus", "2", *ARGS],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (d,) = _lines(r.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
