"""Host side of the device-resident solve (CPU).

`solver._solve_on_device` turns srj_solve's per-cycle records and history into
the reference's SolveReport, resuming paused launches.  Here the "device" is a
stand-in that follows the srj_solve contract (include/srj.h) on the CPU oracle;
the report must equal the oracle's own solve (reference solver.py:289-331):
levels, M, executed counts, totals, residuals, history and the iterate, also
when every launch is cut short by the cycle cap or the history capacity.
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np
import pytest

from oracle import srj_oracle as O
from paper_2011_06636_b200 import _lib, solver
from paper_2011_06636_b200.solver import FixedM, Heuristic, Increasing, StoppingRule


class _Field:
    def __init__(self, a):
        self.interior = np.array(a, dtype=np.float64)


class FakeDeviceOp:
    """srj_solve on the oracle: cycles from x (the result stays in x)."""

    device = "cpu"

    def __init__(self, op):
        self.op = op
        self.launches = 0

    def residual_sq(self, x, b):
        return self.op.residual(x.interior, b.interior)[1]

    def solve_device(self, x, x_alt, b, omegas_all, level_off, mode, level, t_hi, t_lo, res0,
                     prev, budget, tol, baseline, max_cycles, hist_cap, history):
        self.launches += 1
        om, off = omegas_all.numpy(), level_off.numpy()
        top = len(off) - 2
        X = x.interior
        B = b.interior
        r, _ = self.op.residual(X, B)
        recs, total, res_before, stop = [], 0, res0, _lib.SOLVE_PAUSED
        while len(recs) < max_cycles:
            M = int(off[level + 1] - off[level])
            if res_before <= tol:
                recs.append(SimpleNamespace(level=level, M=M, executed=0, status=1,
                                            res_before=res_before, res_after=res_before))
                stop = _lib.SOLVE_CONVERGED
                break
            meff = min(M, max(budget - total, 0))
            if meff == 0:
                recs.append(SimpleNamespace(level=level, M=M, executed=0, status=0,
                                            res_before=res_before, res_after=res_before))
                stop = _lib.SOLVE_BUDGET
                break
            if total + meff > hist_cap:
                break
            res, executed, status = res_before, 0, 0
            for k in range(meff):
                if k > 0 and res <= tol:
                    status = 1
                    break
                X = self.op.update(X, r, om[off[level] + k])
                r, s = self.op.residual(X, B)
                res = math.sqrt(s) / baseline
                executed += 1
                if history is not None:
                    history[total + executed - 1] = res
                if not math.isfinite(res):
                    status = 2
                    break
            if status == 0 and res <= tol:
                status = 1
            recs.append(SimpleNamespace(level=level, M=M, executed=executed, status=status,
                                        res_before=res_before, res_after=res))
            total += executed
            if status == 2:
                stop = _lib.SOLVE_DIVERGED
                break
            if res <= tol:
                stop = _lib.SOLVE_CONVERGED
                break
            if total >= budget:
                stop = _lib.SOLVE_BUDGET
                break
            if res_before > 0 and res > 0:
                prev = res / res_before
            if mode == _lib.SOLVE_HEURISTIC:
                if math.isfinite(prev):
                    level = O.next_level(prev, level, t_hi, t_lo)
            elif mode == _lib.SOLVE_INCREASING:
                level = min(level + 1, top)
            res_before = res
        x.interior[:] = X
        out = SimpleNamespace(cycles=len(recs), stop=stop, result_in_alt=0, next_level=level,
                              res_next=res_before, prev_ratio=prev, sweeps=total)
        return out, recs


CASES = [
    # family, n, controller, tol, relative, budget
    ("1d3", 100, "heuristic", 1e-8, True, 10**9),
    ("1d3", 60, "increasing", 1e-9, False, 10**9),
    ("2d5", 24, "heuristic", 1e-8, True, 10**9),
    ("2d5", 20, "heuristic", 1e-10, True, 150),       # budget cut inside a cycle
    ("1d3", 24, "fixed:5", 1e-12, False, 70),
    ("3d7", 8, "heuristic", 1e-8, True, 10**9),
]


@pytest.mark.parametrize("pause", [None, (3, 10000), (1, 10000)])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}_{c[1]}_{c[2]}_{c[5]}")
def test_report_equals_oracle(case, pause, monkeypatch):
    fam, n, ctrl, tol, relative, budget = case
    op = O.stencil(fam, n)
    b = O.uniform_rhs(5, op.n)
    if ctrl == "heuristic":
        controller, oc, fixed = Heuristic(), "heuristic", None
    elif ctrl == "increasing":
        controller, oc, fixed = Increasing(), "increasing", None
    else:
        m = int(ctrl.split(":")[1])
        controller, oc, fixed = FixedM(m), "fixed", m
    if pause:
        monkeypatch.setattr(solver, "_SOLVE_MAX_CYCLES", pause[0])
        monkeypatch.setattr(solver, "_SOLVE_HIST_CAP", pause[1])
    A = FakeDeviceOp(op)
    x = _Field(np.zeros(op.n))
    bf = _Field(b)
    norm = "relative_l2" if relative else "absolute_l2"
    rule = StoppingRule(norm, tol, budget)
    baseline = math.sqrt(A.residual_sq(x, bf)) if relative else 1.0
    rep = solver._solve_on_device(A, bf, x, _Field(np.zeros(op.n)), controller, rule, 512, True,
                                  baseline, 0.0)
    ref = O.Oracle(op, b).solve(np.zeros(op.n), controller=oc, tol=tol, relative=relative,
                                max_iterations=budget, fixed_M=fixed)
    assert rep.converged == ref.converged
    assert rep.total_iterations == ref.total
    assert [(c.cycle, c.level, c.M, c.executed) for c in rep.cycles] == \
        [(c.cycle, c.level, c.M, c.executed) for c in ref.cycles]
    # residual norms: the OpenMP oracle's reduction order is not fixed -> 1e-12
    close = lambda a, b: a == b or abs(a - b) <= 1e-12 * max(abs(a), abs(b))
    for c, rc in zip(rep.cycles, ref.cycles):
        assert close(c.residual_before, rc.res_before) and close(c.residual_after, rc.res_after)
        assert close(c.average_rate, rc.rate) or abs(c.average_rate - rc.rate) < 1e-9
    assert [k for k, _ in rep.residual_history] == [k for k, _ in ref.history]
    assert all(close(a, b) for (_, a), (_, b) in zip(rep.residual_history, ref.history))
    assert np.array_equal(rep.x, ref.x)
    if pause and pause[0] == 1:
        assert A.launches >= len(rep.cycles)


def test_divergence_raises_like_the_host_loop():
    """A cycle with a non-finite residual ends the device loop; the host raises
    SolveDivergedError with the reference's diagnostic keys (solver.py:235-239)."""
    from paper_2011_06636_b200.solver import SolveDivergedError
    op = O.stencil("1d3", 50)
    b = np.full(op.n, 1e306)
    A = FakeDeviceOp(op)
    x = _Field(np.zeros(op.n))
    rule = StoppingRule("absolute_l2", 1e-8, 10**9)
    with pytest.raises(SolveDivergedError) as e:
        solver._solve_on_device(A, _Field(b), x, _Field(np.zeros(op.n)), Heuristic(), rule, 512,
                                True, 1.0, 0.0)
    d = e.value.diagnostics
    assert set(d) == {"cycle", "sweep", "omega", "level", "M"}
    with pytest.raises(O.OracleDiverged) as ref:
        O.Oracle(op, b).solve(np.zeros(op.n), controller="heuristic", tol=1e-8, relative=False)
    # the oracle counts sweeps over the whole solve, the diagnostics per cycle
    assert d["omega"] == ref.value.omega
