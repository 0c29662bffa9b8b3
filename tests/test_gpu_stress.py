"""Race and bounds evidence for the barrier-free kernels (the stress build).

compute-sanitizer is closed on the GPU pool, so the check is done with our own
instrumentation (csrc/srj_stress.cuh, libsrj_stress.so): every mbarrier
arrive / wait, TMA issue and grid barrier of every kernel sleeps a
pseudo-random subset of warps for up to ~4 us, so warps and CTAs drift apart
in orders a normal run never produces; mbarrier waits are bounded (a lost
arrival traps instead of hanging); shared-memory and global index bounds are
asserted in the staged kernels.  The parity tests below -- multi-tile grids
with masked tiles, every rollback stop position, the speculative next-pass
copy and its drain, the SOLVE and SLAB instantiations, the skewed-tile 2D kernel
(hand-off rounds, carry rows between tiles), the 1D register and
shared-memory kernels, the batched collection kernel -- must stay bit-identical
to the oracle under that build, several rounds each.  The negative control
removes one wait (SRJ_STRESS_BREAK=1: the TB2D halo hand-off) and must fail.

Logs: $SRJ_STRESS_LOG_DIR (default: a temporary directory).
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
STRESS_LIB = os.path.join(ROOT, "paper_2011_06636_b200", "libsrj_stress.so")

SELECTION = [
    "tests/test_gpu_tb2d.py::test_tb2d_cycle_bitwise_vs_oracle",
    "tests/test_gpu_tbvar.py::test_tbvar_cycle_bitwise_vs_oracle",
    "tests/test_gpu_tb3d.py::test_tb3d_cycle_bitwise_vs_oracle",
    "tests/test_gpu_device_solve.py::test_device_loop_matches_host_loop",
    "tests/test_gpu_device_solve.py::test_device_loop_pauses_and_resumes",
    "tests/test_gpu_tbslabs.py::test_tb_row_slabs_match_reference[c2_64-2-True]",
    "tests/test_gpu_tbslabs.py::test_tb_row_slabs_match_reference[c4_64-3-False]",
    "tests/test_gpu_tbslabs.py::test_tb_z_slabs_match_reference[c3_16-2-True]",
    "tests/test_gpu_tbslabs.py::test_tb_z_slabs_match_reference[c3_32-3-False]",
    "tests/test_gpu_tbslabs.py::test_tb_pass_owned_rows_vs_oracle",
    "tests/test_gpu_small1d.py::test_1d_cycle_bitwise_vs_oracle",
    "tests/test_datacollect.py::test_batched_collect_matches_reference",
    "tests/test_gpu_random_shapes.py::test_random_shape_cycle_bitwise[3d7varbig-0]",
    "tests/test_gpu_random_shapes.py::test_random_shape_cycle_bitwise[3d7varbig-3]",
    "tests/test_gpu_random_shapes.py::test_random_shape_cycle_bitwise[1d3var-1]",
    "tests/test_gpu_random_shapes.py::test_random_shape_cycle_bitwise[1d3var-4]",
    "tests/test_gpu_tbslabs.py::test_tb_slabs_graph_replay_matches_reference",
    "tests/test_gpu_var3d.py",
    "tests/test_gpu_tbs.py",
]


def _log_dir():
    d = os.environ.get("SRJ_STRESS_LOG_DIR")
    if not d:
        d = tempfile.mkdtemp(prefix="srj_stress_")
    os.makedirs(d, exist_ok=True)
    return d


def _run(selection, env_extra, log_name, timeout=1200):
    env = dict(os.environ)
    env.update(env_extra)
    env["SRJ_LIBRARY"] = STRESS_LIB
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
           *selection]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    path = os.path.join(_log_dir(), log_name)
    with open(path, "w") as f:
        extra = " ".join(f"{k}={v}" for k, v in env_extra.items())
        f.write(f"$ SRJ_LIBRARY={STRESS_LIB} {extra} {' '.join(cmd)}\n")
        f.write(res.stdout)
        f.write(res.stderr)
        f.write(f"\nrc={res.returncode}\n")
    return res


@pytest.mark.parametrize("round_", [0, 1, 2])
def test_parity_under_jitter_and_bounds_checks(round_):
    if not os.path.exists(STRESS_LIB):
        pytest.fail("libsrj_stress.so missing: run __graft_entry__.build()")
    res = _run(SELECTION, {}, f"stress_round{round_}.log")
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]


def test_stress_build_catches_an_injected_race():
    """Negative control: without the halo hand-off wait the jittered TB2D
    kernel must produce a wrong iterate (or trap) in the parity test."""
    sel = ["tests/test_gpu_tb2d.py::test_tb2d_cycle_bitwise_vs_oracle[dims0-1-6]"]
    res = _run(sel, {"SRJ_STRESS_BREAK": "1"}, "stress_negative_control.log", timeout=600)
    assert res.returncode != 0, "the injected race went undetected"
