"""SRJ cycles on the device, level-selection controllers and the solve driver.

Same names, signatures, semantics and errors as the reference solver
(reference solver.py:24-331); the difference is where the sweeps run.  Each
cycle is ONE call into libsrj (`srj_run_cycle`): the sm_100a kernel applies up
to M weighted-Jacobi sweeps in the scheme's application order, evaluates the
stopping rule before every sweep on a device-reduced residual norm, and the
host reads back one small struct (executed, status, res_after) -- plus the
per-sweep residuals only when `record_history` is set.  Scheme selection
(Heuristic / Increasing / FixedM / Jacobi / Cjm) stays on the host, except that
for the temporally blocked kernels `solve` runs the Heuristic / Increasing /
FixedM loop on the device (srj_solve) with the same decisions.

Parity contract: identical scheme sequence, executed counts and
iterates (bitwise) to the reference; residual norms differ from OpenBLAS ddot
only in summation order (~1e-15 relative).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .operators import DeviceOperator, Field, StencilOperator
from .problems import ABSOLUTE_L2, RELATIVE_L2, SOLUTION_DIFF_INF, ProblemInstance
from .sparse import device_operator
from .schemes import (MAX_LEVEL, ORDER_GRID_SIZE, SrjScheme, generate_srj_scheme,
                      scheme_for_level)

T_HI_DEFAULT = 0.4
T_LO_DEFAULT = 0.2

JACOBI_SCHEME = SrjScheme(M=1, omegas=(1.0,), application_order=(0,))


@dataclass(frozen=True)
class StoppingRule:
    norm: str
    tolerance: float
    max_iterations: int

    def __post_init__(self):
        if self.tolerance <= 0.0:
            raise ValueError("tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be positive")


class ResidualKnown:
    """Internal `SolverState.cached_r` marker of the solve loop: the residual of
    `x` is `current_residual` (the device path never needs the vector r)."""

    __slots__ = ()

    def __repr__(self):
        return "ResidualKnown"


RESIDUAL_KNOWN = ResidualKnown()


class LazyResidual:
    """r = b - A x of a run_cycle result, materialised on first access of
    `SolverState.cached_r` (reference solver.py:205-210,270 keep that vector).
    One device matvec plus one subtraction: bit-identical to the reference's
    `b - csr.dot(x)`."""

    __slots__ = ("_A", "_b", "_x", "_as_numpy")

    def __init__(self, A, b, x, as_numpy: bool):
        self._A, self._b, self._x, self._as_numpy = A, b, x, as_numpy

    def materialize(self):
        A = self._A
        y = A.matvec(A.field(self._x))
        r = self._b.interior - y
        return r.cpu().numpy() if self._as_numpy else r


@dataclass
class SolverState:
    x: object
    level: int = 0
    prev_residual_ratio: float | None = None
    cycle_index: int = 0
    total_iterations: int = 0
    residual_history: list[tuple[int, float]] = field(default_factory=list)
    current_residual: float | None = None
    cached_r: object | None = None
    converged: bool = False


def _get_cached_r(self):
    r = self.__dict__.get("_cached_r")
    if isinstance(r, LazyResidual):
        r = r.materialize()
        self.__dict__["_cached_r"] = r
    elif isinstance(r, ResidualKnown):
        return None
    return r


def _set_cached_r(self, value):
    self.__dict__["_cached_r"] = value


SolverState.cached_r = property(_get_cached_r, _set_cached_r)


def _residual_known(state) -> bool:
    """Whether `state` carries the residual of its x (without materialising a
    LazyResidual); works for the reference's own SolverState too."""
    if "_cached_r" in getattr(state, "__dict__", {}):
        return state.__dict__["_cached_r"] is not None
    return getattr(state, "cached_r", None) is not None


@dataclass(frozen=True)
class CycleStats:
    cycle: int
    level: int
    M: int
    executed: int
    residual_before: float
    residual_after: float
    average_rate: float

    @property
    def ratio(self) -> float:
        return self.residual_after / self.residual_before


@dataclass
class SolveReport:
    converged: bool
    total_iterations: int
    cycles: list[CycleStats]
    wall_time: float
    x: object
    residual_history: list[tuple[int, float]]


class SolveDivergedError(RuntimeError):
    """A sweep produced non-finite values (application-order failure)."""

    def __init__(self, diagnostics: dict):
        super().__init__(f"solve diverged: {diagnostics}")
        self.diagnostics = diagnostics


# ---------------------------------------------------------------------------
# Controllers (reference solver.py:96-122)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Heuristic:
    t_hi: float = T_HI_DEFAULT
    t_lo: float = T_LO_DEFAULT


@dataclass(frozen=True)
class Increasing:
    pass


@dataclass(frozen=True)
class FixedM:
    M: int


@dataclass(frozen=True)
class Jacobi:
    pass


@dataclass(frozen=True)
class Cjm:
    scheme: SrjScheme


Controller = Heuristic | Increasing | FixedM | Jacobi | Cjm


def heuristic_next_level(ratio: float, level: int, t_hi: float = T_HI_DEFAULT,
                         t_lo: float = T_LO_DEFAULT) -> int:
    """Algorithm 1: raise above t_hi, lower strictly between t_lo and t_hi,
    otherwise keep (ratio == t_hi keeps); clamp to the ladder."""
    if ratio < 0.0:
        raise ValueError("residual ratio must be nonnegative")
    if ratio > t_hi:
        level += 1
    elif t_lo < ratio < t_hi:
        level -= 1
    return min(max(level, 0), MAX_LEVEL)


def average_convergence_rate(r_before: float, r_after: float, M: int) -> float:
    if r_before <= 0.0 or r_after <= 0.0:
        raise ValueError("residuals must be positive")
    if M < 1:
        raise ValueError("M must be positive")
    return -math.log(r_after / r_before) / M


# ---------------------------------------------------------------------------
# Device plumbing
# ---------------------------------------------------------------------------

class _OmegaCache:
    """Ordered omegas of each scheme, resident in HBM (one upload per scheme)."""

    def __init__(self):
        self._by_device: dict = {}

    def get(self, scheme: SrjScheme, device):
        import torch
        key = (str(device), scheme.M, scheme.omegas, scheme.application_order)
        table = self._by_device
        t = table.get(key)
        if t is None:
            t = torch.tensor(scheme.ordered_omegas(), dtype=torch.float64, device=device)
            if len(table) > 512:
                table.clear()
            table[key] = t
        return t


_OMEGAS = _OmegaCache()


class _LevelTables:
    """Ordered omegas of every scheme a device-resident solve may pick, resident
    in HBM: levels 0..MAX_LEVEL concatenated (Heuristic, Increasing) or one
    fixed scheme (FixedM), with int32 offsets (srj_solve_args)."""

    def __init__(self):
        self._cache: dict = {}

    def get(self, schemes: tuple, device):
        import torch
        key = (str(device), tuple((s.M, s.omegas, s.application_order) for s in schemes))
        t = self._cache.get(key)
        if t is None:
            om = [w for s in schemes for w in s.ordered_omegas()]
            off = np.concatenate([[0], np.cumsum([s.M for s in schemes])]).astype(np.int32)
            t = (torch.tensor(om, dtype=torch.float64, device=device),
                 torch.tensor(off, dtype=torch.int32, device=device))
            if len(self._cache) > 64:
                self._cache.clear()
            self._cache[key] = t
        return t


_LEVEL_TABLES = _LevelTables()
_SOLVE_HIST_CAP = 1 << 20   # sweeps one srj_solve call may record (then it pauses)
_SOLVE_MAX_CYCLES = 4096


def _device_solve_ok(A, controller, stopping: StoppingRule, cycle_hook) -> bool:
    return (cycle_hook is None and stopping.norm in (ABSOLUTE_L2, RELATIVE_L2)
            and isinstance(controller, (Heuristic, Increasing, FixedM))
            and isinstance(A, StencilOperator) and A.solve_supported())


def _solve_on_device(A: StencilOperator, b: Field, x: Field, x_alt: Field, controller,
                     stopping: StoppingRule, order_grid: int, record_history: bool,
                     baseline: float, t0: float) -> SolveReport:
    """solve_fields with the controller loop on the device (srj_solve): the
    same cycles, levels, stopping and report as the host loop below, one
    launch per solve instead of one per cycle."""
    if isinstance(controller, FixedM):
        schemes = (generate_srj_scheme(controller.M, order_grid),)
        mode, t_hi, t_lo = _lib.SOLVE_FIXED, 0.0, 0.0
    else:
        schemes = tuple(scheme_for_level(l, order_grid) for l in range(MAX_LEVEL + 1))
        if isinstance(controller, Heuristic):
            mode, t_hi, t_lo = _lib.SOLVE_HEURISTIC, controller.t_hi, controller.t_lo
        else:
            mode, t_hi, t_lo = _lib.SOLVE_INCREASING, 0.0, 0.0
    omegas_all, level_off = _LEVEL_TABLES.get(schemes, A.device)
    # the first cycle's incoming residual, as the host loop computes it
    res_now = math.sqrt(A.residual_sq(x, b)) / baseline
    history: list[tuple[int, float]] = [(0, res_now)] if record_history else []
    hist = np.empty(_SOLVE_HIST_CAP, dtype=np.float64) if record_history else None
    cycles: list[CycleStats] = []
    total, cycle_index, level, prev = 0, 0, 0, math.nan
    while True:
        out, recs = A.solve_device(x, x_alt, b, omegas_all, level_off, mode, level, t_hi, t_lo,
                                   res_now, prev, stopping.max_iterations - total,
                                   stopping.tolerance, baseline, _SOLVE_MAX_CYCLES,
                                   _SOLVE_HIST_CAP, hist)
        done = 0
        for rec in recs:
            scheme = schemes[rec.level]
            executed = int(rec.executed)
            if rec.status == _lib.CYCLE_DIVERGED:
                raise SolveDivergedError({
                    "cycle": cycle_index, "sweep": executed,
                    "omega": scheme.ordered_omegas()[executed - 1],
                    "level": scheme.level, "M": scheme.M,
                })
            if record_history:
                history.extend((total + k + 1, float(hist[done + k])) for k in range(executed))
            rb, ra = float(rec.res_before), float(rec.res_after)
            if executed > 0:
                if rb > 0.0 and ra > 0.0:
                    rate = average_convergence_rate(rb, ra, executed)
                else:
                    rate = math.inf
                cycles.append(CycleStats(
                    cycle=cycle_index, level=scheme.level if scheme.level is not None else -1,
                    M=scheme.M, executed=executed, residual_before=rb, residual_after=ra,
                    average_rate=rate))
            total += executed
            done += executed
            cycle_index += 1
        if out.result_in_alt:
            x, x_alt = x_alt, x
        if out.stop != _lib.SOLVE_PAUSED:
            break
        level, res_now, prev = int(out.next_level), float(out.res_next), float(out.prev_ratio)
    return SolveReport(
        converged=out.stop == _lib.SOLVE_CONVERGED, total_iterations=total, cycles=cycles,
        wall_time=time.perf_counter() - t0, x=x.interior, residual_history=history,
    )


def _l2_norm_parts(norm: str) -> None:
    if norm not in (ABSOLUTE_L2, RELATIVE_L2, SOLUTION_DIFF_INF):
        raise ValueError(f"unknown norm {norm!r}")


def _diff_cycle(A, b, x, x_alt, state, scheme, stopping, record_history, x_out_kind):
    """One cycle under the solution-difference infinity norm, step for step
    reference solver.py:200-203,216-273 with diff_norm true; the sweep loop is
    srj_run_cycle_diffinf (norm bit-identical: a max)."""
    res_now = state.current_residual
    res_before = res_now
    history = list(state.residual_history) if record_history else state.residual_history
    M = scheme.M
    tol = stopping.tolerance if stopping is not None else -1.0
    budget = (stopping.max_iterations - state.total_iterations) if stopping is not None else M
    # the first sweep's norm becomes res_before when none is known (:242-243)
    hist = np.empty(M, dtype=np.float64) if (record_history or res_now is None) else None
    omegas = _OMEGAS.get(scheme, A.device)
    out = A.run_cycle_diffinf(x, x_alt, b, omegas, M, tol, res_now, budget, hist)
    executed = int(out.executed)
    if out.status == _lib.CYCLE_DIVERGED:
        raise SolveDivergedError({
            "cycle": state.cycle_index, "sweep": executed,
            "omega": scheme.ordered_omegas()[executed - 1], "level": scheme.level, "M": scheme.M,
        })
    if executed > 0:
        res_now = float(out.res_after)
        if res_before is None:
            res_before = float(hist[0])
    if record_history and executed:
        base = state.total_iterations
        history.extend((base + k + 1, float(hist[k])) for k in range(executed))
    res_after = res_now if res_now is not None else float("nan")
    if res_before is None:
        res_before = res_after
    converged = stopping is not None and res_now is not None and res_now <= stopping.tolerance
    if executed > 0 and res_before > 0.0 and res_after > 0.0:
        rate = average_convergence_rate(res_before, res_after, executed)
        ratio = res_after / res_before
    else:
        rate = math.inf if executed > 0 else 0.0
        ratio = state.prev_residual_ratio
    result, other = (x_alt, x) if out.result_in_alt else (x, x_alt)
    stats = CycleStats(
        cycle=state.cycle_index, level=scheme.level if scheme.level is not None else -1,
        M=scheme.M, executed=executed, residual_before=res_before, residual_after=res_after,
        average_rate=rate)
    new_state = SolverState(
        x=x_out_kind(result), level=scheme.level if scheme.level is not None else state.level,
        prev_residual_ratio=ratio if executed > 0 else state.prev_residual_ratio,
        cycle_index=state.cycle_index + 1, total_iterations=state.total_iterations + executed,
        residual_history=history, current_residual=res_now, cached_r=None, converged=converged)
    return new_state, stats, result, other


def _device_cycle(A: DeviceOperator, b: Field, x: Field, x_alt: Field, state: SolverState,
                  scheme: SrjScheme, stopping: StoppingRule | None, baseline: float,
                  record_history: bool, x_out_kind, norm: str = ABSOLUTE_L2):
    """One cycle on (x, x_alt); returns (new_state, stats, result_field, other_field).

    Follows reference solver.py:187-273 step by step; the sweep loop itself
    (:216-243) is the device call.
    """
    if norm == SOLUTION_DIFF_INF:
        return _diff_cycle(A, b, x, x_alt, state, scheme, stopping, record_history, x_out_kind)
    if _residual_known(state) and state.current_residual is not None:
        res_now = float(state.current_residual)
    else:
        res_now = math.sqrt(A.residual_sq(x, b)) / baseline
    res_before = res_now
    history = list(state.residual_history) if record_history else state.residual_history
    if record_history and not history:
        history.append((state.total_iterations, res_now))

    M = scheme.M
    tol = stopping.tolerance if stopping is not None else -1.0
    budget = (stopping.max_iterations - state.total_iterations) if stopping is not None else M
    hist = np.empty(M, dtype=np.float64) if record_history else None
    omegas = _OMEGAS.get(scheme, A.device)
    out = A.run_cycle(x, x_alt, b, omegas, M, tol, baseline, res_before, budget, hist)
    executed = int(out.executed)
    if out.status == _lib.CYCLE_DIVERGED:
        ordered = scheme.ordered_omegas()
        raise SolveDivergedError({
            "cycle": state.cycle_index, "sweep": executed, "omega": ordered[executed - 1],
            "level": scheme.level, "M": scheme.M,
        })
    res_after = float(out.res_after) if executed > 0 else res_before
    converged = stopping is not None and res_after <= stopping.tolerance
    if record_history:
        base = state.total_iterations
        history.extend((base + k + 1, float(hist[k])) for k in range(executed))

    if executed > 0 and res_before > 0.0 and res_after > 0.0:
        rate = average_convergence_rate(res_before, res_after, executed)
        ratio = res_after / res_before
    else:
        rate = math.inf if executed > 0 else 0.0
        ratio = state.prev_residual_ratio

    result, other = (x_alt, x) if out.result_in_alt else (x, x_alt)
    stats = CycleStats(
        cycle=state.cycle_index, level=scheme.level if scheme.level is not None else -1,
        M=scheme.M, executed=executed, residual_before=res_before, residual_after=res_after,
        average_rate=rate,
    )
    new_state = SolverState(
        x=x_out_kind(result), level=scheme.level if scheme.level is not None else state.level,
        prev_residual_ratio=ratio if executed > 0 else state.prev_residual_ratio,
        cycle_index=state.cycle_index + 1,
        total_iterations=state.total_iterations + executed,
        residual_history=history, current_residual=res_after,
        cached_r=RESIDUAL_KNOWN, converged=converged,
    )
    return new_state, stats, result, other


def _field_view(f: Field):
    return f.interior


def run_cycle(A: StencilOperator, b, state: SolverState, scheme: SrjScheme,
              stopping: StoppingRule | None = None, baseline: float = 1.0,
              norm: str = ABSOLUTE_L2, record_history: bool = True,
              ) -> tuple[SolverState, CycleStats]:
    """Apply one scheme cycle and return the advanced state plus its stats.

    The input state is not modified (its x is copied into a fresh device
    ping-pong pair); numpy inputs give numpy outputs.
    """
    A = device_operator(A)
    if stopping is not None and norm != stopping.norm:
        norm = stopping.norm
    _l2_norm_parts(norm)
    as_numpy = isinstance(state.x, np.ndarray)
    bf = b if isinstance(b, Field) else A.field(b)
    x = A.field(state.x)
    x_alt = A.new_field()

    def kind(f: Field):
        return f.interior.cpu().numpy() if as_numpy else f.interior

    new_state, stats, _, _ = _device_cycle(A, bf, x, x_alt, state, scheme, stopping,
                                           baseline, record_history, kind, norm)
    if norm != SOLUTION_DIFF_INF:
        new_state.cached_r = LazyResidual(A, bf, new_state.x, as_numpy)
    return new_state, stats


def _next_scheme(controller: Controller, state: SolverState, order_grid: int) -> SrjScheme:
    if isinstance(controller, (Heuristic, Increasing)):
        return scheme_for_level(state.level, order_grid)
    if isinstance(controller, FixedM):
        return generate_srj_scheme(controller.M, order_grid)
    if isinstance(controller, Jacobi):
        return JACOBI_SCHEME
    if isinstance(controller, Cjm):
        return controller.scheme
    raise TypeError(f"unknown controller {controller!r}")


def solve(problem: ProblemInstance, controller: Controller, stopping: StoppingRule,
          order_grid: int = ORDER_GRID_SIZE, record_history: bool = True,
          out=None) -> SolveReport:
    """Full solve under a controller and stopping rule (reference solver.py:289-331).

    b and x0 are staged into HBM once; the iterate then ping-pongs between two
    device buffers for the whole solve with no per-cycle copies.  The report's
    x has the kind of x0: numpy array, CPU tensor (copied back through pinned
    memory) or CUDA tensor (no copy).  `out` (extension, optional): a
    preallocated torch tensor of n float64 values (e.g. pinned host memory)
    that receives the solution and becomes the report's x, so repeated solves
    do not allocate a fresh host buffer each time.
    """
    t0 = time.perf_counter()
    A = device_operator(problem.A)
    _l2_norm_parts(stopping.norm)
    b = A.field(problem.b)
    x = A.field(problem.x0)
    rep = solve_fields(A, b, x, A.new_field(), controller, stopping, order_grid, record_history)
    if out is not None:
        if out.numel() != A.n:
            raise ValueError(f"out holds {out.numel()} values, the operator {A.n}")
        out.view(-1).copy_(rep.x.reshape(-1))
        rep.x = out
    else:
        rep.x = _like(problem.x0, rep.x)
    rep.wall_time = time.perf_counter() - t0
    return rep


def _like(template, x_dev):
    if isinstance(template, np.ndarray):
        return x_dev.cpu().numpy()
    if not template.is_cuda:
        import torch
        out = torch.empty(x_dev.shape, dtype=x_dev.dtype, pin_memory=True)
        out.copy_(x_dev)
        return out
    return x_dev


def solve_fields(A: StencilOperator, b: Field, x: Field, x_alt: Field, controller: Controller,
                 stopping: StoppingRule, order_grid: int = ORDER_GRID_SIZE,
                 record_history: bool = True, cycle_hook=None,
                 device_loop: bool = True) -> SolveReport:
    """`solve` on device-resident Fields (no staging): x holds x0 on entry and
    both x and x_alt are overwritten.  The report's x is a CUDA view of
    whichever buffer holds the final iterate.  `cycle_hook(stats)` is called
    after every cycle (bench instrumentation; forces the host loop).  Where the
    operator supports it (srj_op_solve_supported) and the controller is
    Heuristic / Increasing / FixedM, the controller loop runs on the device
    (`device_loop`, srj_solve): one launch per solve, same report."""
    t0 = time.perf_counter()
    _l2_norm_parts(stopping.norm)
    baseline = 1.0
    if stopping.norm == RELATIVE_L2:
        baseline = math.sqrt(A.residual_sq(x, b))
        if baseline == 0.0:
            raise ValueError("initial residual is zero; relative norm undefined")
    if device_loop and _device_solve_ok(A, controller, stopping, cycle_hook):
        return _solve_on_device(A, b, x, x_alt, controller, stopping, order_grid, record_history,
                                baseline, t0)
    state = SolverState(x=x.interior, level=0)
    cycles: list[CycleStats] = []
    converged = False
    while True:
        scheme = _next_scheme(controller, state, order_grid)
        state, stats, x, x_alt = _device_cycle(A, b, x, x_alt, state, scheme, stopping,
                                               baseline, record_history, _field_view,
                                               stopping.norm)
        if cycle_hook is not None:
            cycle_hook(stats)
        if stats.executed > 0:
            cycles.append(stats)
        if state.converged:
            converged = True
            break
        if state.total_iterations >= stopping.max_iterations:
            break
        if isinstance(controller, Heuristic):
            ratio = state.prev_residual_ratio
            if ratio is not None and math.isfinite(ratio):
                state.level = heuristic_next_level(ratio, state.level,
                                                   controller.t_hi, controller.t_lo)
        elif isinstance(controller, Increasing):
            state.level = min(state.level + 1, MAX_LEVEL)
    return SolveReport(
        converged=converged, total_iterations=state.total_iterations, cycles=cycles,
        wall_time=time.perf_counter() - t0, x=x.interior, residual_history=state.residual_history,
    )
