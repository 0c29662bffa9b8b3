"""Device-resident solve (srj_solve) against the host controller loop (GPU).

`solve` runs the Heuristic / Increasing / FixedM controller loop on the device
where the operator's kernel supports it (the temporally blocked kernels and the
1D register kernel).  The host loop (one srj_run_cycle per cycle) is the
reference here: both must produce identical reports -- levels, M, executed
counts, residuals (same kernels, same reductions: bit-identical), histories and
iterates -- including budget cuts, pauses (cycle cap, history capacity) and the
golden traces of the reference.
"""

from __future__ import annotations

import numpy as np
import pytest

import _parity as P

pytestmark = pytest.mark.gpu

CASES = ["c1_seed0", "poisson1d_100_heuristic", "poisson1d_100_increasing", "fixed5_tol_tiny",
         "increasing_clamp", "tiny_1d_n1", "c2_32", "c2_64", "c3_16", "c4_32",
         "budget_midcycle_2d", "fixed2362_3d", "poisson3d_24_ones", "c1v_1024", "c1v_100_s2",
         "c3v_12", "c3v_24_budget"]


def _solve(c, device_loop, record_history=True, spp=None):
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.solver import solve_fields
    dev = torch.device("cuda", 0)
    fam, n, b, _, _ = P.case_inputs(c)
    A = P.case_operator(c, device=dev)
    if spp:
        A.set_sweeps_per_pass(spp)
    ctrl = c["controller"]
    if ctrl == "heuristic":
        controller = srj.Heuristic()
    elif ctrl == "increasing":
        controller = srj.Increasing()
    else:
        controller = srj.FixedM(int(ctrl.split(":")[1]))
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    bf = A.field(b)
    x = A.new_field()
    rep = solve_fields(A, bf, x, A.new_field(), controller, rule, record_history=record_history,
                       device_loop=device_loop)
    return A, rep


def _same(r1, r2):
    assert r1.converged == r2.converged
    assert r1.total_iterations == r2.total_iterations
    assert r1.cycles == r2.cycles  # dataclass equality: every field, exact floats
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(r1.x.cpu().numpy(), r2.x.cpu().numpy())


@pytest.mark.parametrize("name", CASES)
def test_device_loop_matches_host_loop(name):
    c = P.case(name)
    A, dev = _solve(c, True)
    assert A.solve_supported() or c["n"] < 4, A.describe()
    _, host = _solve(c, False)
    _same(dev, host)
    # and the reference's own trace
    rows = [(s.cycle, s.level, s.M, s.executed, s.residual_before, s.residual_after,
             s.average_rate) for s in dev.cycles]
    P.assert_trace_matches(c, rows, dev.total_iterations, dev.converged, x=dev.x.cpu().numpy())


@pytest.mark.parametrize("name", ["c2_64", "c1_seed0", "c3_16", "c4_32"])
def test_device_loop_pauses_and_resumes(name, monkeypatch):
    """A cycle cap of 3 per launch and the smallest history buffer: the host
    resumes from the paused state; the report is unchanged."""
    from paper_2011_06636_b200 import solver
    c = P.case(name)
    _, ref = _solve(c, True)
    monkeypatch.setattr(solver, "_SOLVE_MAX_CYCLES", 3)
    monkeypatch.setattr(solver, "_SOLVE_HIST_CAP", 10000)
    _, got = _solve(c, True)
    _same(got, ref)


def test_device_loop_without_history():
    c = P.case("c2_64")
    _, a = _solve(c, True, record_history=False)
    _, b = _solve(c, False, record_history=False)
    _same(a, b)
    assert a.residual_history == []


def test_device_loop_only_where_supported():
    """One sweep per pass on a 2D operator runs the host loop (no device solve
    for the tile-streaming kernel); the report is the same."""
    c = P.case("c2_64")
    A, r1 = _solve(c, True, spp=1)
    assert not A.solve_supported()
    _, r2 = _solve(c, True)
    assert r1.total_iterations == r2.total_iterations
    assert [s.level for s in r1.cycles] == [s.level for s in r2.cycles]


@pytest.mark.parametrize("fam,dims", [("2d5", (64, 64)), ("1d3", (300,)), ("3d7", (24, 24, 24))])
def test_device_loop_divergence_matches_host_loop(fam, dims):
    """Overflowing iterates: both loops raise SolveDivergedError with the same
    diagnostics (cycle, sweep, omega, level, M)."""
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.solver import SolveDivergedError, solve_fields
    dev = torch.device("cuda", 0)
    diag = []
    for device_loop in (True, False):
        A = srj.StencilOperator(fam, dims, device=dev)
        b = A.field(np.full(A.n, 1e306))
        rule = srj.StoppingRule("absolute_l2", 1e-8, 10**9)
        with pytest.raises(SolveDivergedError) as e:
            solve_fields(A, b, A.new_field(), A.new_field(), srj.Heuristic(), rule,
                         record_history=False, device_loop=device_loop)
        diag.append(e.value.diagnostics)
    assert diag[0] == diag[1]
