"""SRJ CPU oracle -- TEST INFRASTRUCTURE ONLY.

An independent CPU restatement of the reference solve path, used as the parity
checker by tests/, by __graft_entry__.smoke() and as bench.py's CPU baseline
(`cpu_baseline.kind = "port"`).  The product never imports this module.

Pinned (tests/test_oracle.py) against fixtures produced by running the
reference itself (tests/golden/make_golden.py) and against the reference's own
golden CSVs (pkg/results/*.csv).

Restated reference code (paths under /root/reference/pkg/src/srj):
  chebyshev.py:82-94,117-120  roots, lambda*, lambda_max       -> cheb_roots, lambda_star, lambda_max
  schemes.py:31-35,72-138     ladder, omegas, stability order   -> LADDER, omegas, stability_order, scheme
  solver.py:125-149           heuristic, average rate           -> next_level, avg_rate
  solver.py:177-273           run_cycle                         -> Oracle.cycle
  solver.py:289-331           solve                             -> Oracle.solve
  sparse.py:20-44,84-93       operator, inv_diag, sweep         -> StencilCPU (C kernels in srj_oracle.c)
  rng.py:25-40                SplitMix64                        -> splitmix_uniforms
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libsrj_oracle.so")

# ---------------------------------------------------------------- schemes

LADDER = (1, 2, 3, 5, 7, 10, 14, 19, 26, 35, 47, 63, 84, 111, 147,
          194, 256, 338, 446, 589, 778, 1027, 1356, 1790, 2362)
TOP = len(LADDER) - 1


def cheb_roots(M):
    j = np.arange(M)
    return np.cos(np.pi * (2 * j + 1) / (2 * M))


def lambda_star(M):
    return math.cosh(math.acosh(3.0) / M)


def lambda_max(M):
    s = lambda_star(M)
    return (3.0 - s) / (1.0 + s)


def omegas(M):
    s = lambda_star(M)
    return (s + 1.0) / (2.0 * (s - cheb_roots(M)))


def _pairing(units):
    # recursive strongest/weakest pairing (schemes.py:78-85)
    if len(units) <= 2:
        return units
    h = len(units) // 2
    joined = [units[i] + units[-1 - i] for i in range(h)]
    return _pairing(joined) + ([units[h]] if len(units) % 2 else [])


def stability_order(w, grid_size=512):
    M = len(w)
    if M == 1:
        return (0,)
    desc = sorted(range(M), key=lambda j: -w[j])
    order = tuple(j for u in _pairing([[j] for j in desc]) for j in u)
    grid = np.linspace(-1.0, lambda_max(M), grid_size)
    run = np.zeros_like(grid)
    peak = 0.0
    for j in order:
        run += np.log(np.maximum(np.abs(1.0 - w[j] * (1.0 - grid)), 1e-300))
        peak = max(peak, float(run.max()))
    if not np.isfinite(peak) or peak > 700.0:
        raise ValueError(f"no stable ordering for M={M}")
    return order


_SCHEMES = {}


def scheme(M):
    """(ordered omegas, level) of the length-M SRJ scheme."""
    if M not in _SCHEMES:
        w = tuple(float(v) for v in omegas(M))
        order = stability_order(np.asarray(w))
        _SCHEMES[M] = (tuple(w[j] for j in order), LADDER.index(M) if M in LADDER else None)
    return _SCHEMES[M]


def cjm_scheme(M, lam_lo, lam_hi):
    """Ordered omegas of the CJM comparator (schemes.py:141-160)."""
    mid = 0.5 * (lam_hi + lam_lo)
    half = 0.5 * (lam_hi - lam_lo)
    w = tuple(float(1.0 / (1.0 - v)) for v in mid + half * cheb_roots(M))
    order = stability_order(np.asarray(w))
    return tuple(w[j] for j in order)


def next_level(ratio, level, t_hi=0.4, t_lo=0.2):
    if ratio > t_hi:
        level += 1
    elif t_lo < ratio < t_hi:
        level -= 1
    return min(max(level, 0), TOP)


def avg_rate(before, after, M):
    return -math.log(after / before) / M


def splitmix_uniforms(seed, n):
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uniform_rhs(seed, n):
    return 2.0 * splitmix_uniforms(seed, n) - 1.0

# ---------------------------------------------------------------- operators


_lib = None


def clib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run `make -C oracle`")
        L = ctypes.CDLL(LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.oracle_residual.restype = ctypes.c_double
        L.oracle_residual.argtypes = [ctypes.c_int, i64, i64, i64, ctypes.c_double,
                                      dp, dp, dp, dp, dp, dp]
        L.oracle_update.argtypes = [ctypes.c_int, i64, i64, i64, ctypes.c_double,
                                    dp, dp, dp, dp, dp, ctypes.c_double, dp]
        L.oracle_matvec.argtypes = [ctypes.c_int, i64, i64, i64, ctypes.c_double,
                                    dp, dp, dp, dp, dp]
        L.oracle_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


FAMILY_CODE = {"1d3": 1, "2d5": 2, "3d7": 3, "2d5var": 4, "3d7var": 6, "1d3var": 7}


@dataclass
class StencilCPU:
    """Structured Dirichlet operator evaluated by srj_oracle.c."""

    family: str
    nx: int
    ny: int = 1
    nz: int = 1
    dx2: float = 0.0
    fx: np.ndarray | None = None
    fy: np.ndarray | None = None
    fz: np.ndarray | None = None

    @property
    def n(self):
        return self.nx * self.ny * self.nz

    def _args(self):
        return (FAMILY_CODE[self.family], self.nx, self.ny, self.nz, float(self.dx2),
                _p(self.fx), _p(self.fy), _p(self.fz))

    def residual(self, x, b):
        r = np.empty(self.n)
        s = clib().oracle_residual(*self._args(), _p(x), _p(b), _p(r))
        return r, s

    def update(self, x, r, w):
        out = np.empty(self.n)
        clib().oracle_update(*self._args(), _p(x), _p(r), float(w), _p(out))
        return out

    def matvec(self, x):
        y = np.empty(self.n)
        clib().oracle_matvec(*self._args(), _p(x), _p(y))
        return y


class CsrCPU:
    """General CSR operator: scipy's csr_matvec is the reference's own SpMV
    (solver.py:233 -> sparse.py:81), so the oracle calls it directly."""

    def __init__(self, csr):
        self.csr = csr
        self.n = csr.shape[0]
        self.inv_diag = 1.0 / csr.diagonal()

    def residual(self, x, b):
        r = b - self.csr.dot(x)
        return r, float(np.dot(r, r))

    def update(self, x, r, w):
        return x + w * (self.inv_diag * r)

    def matvec(self, x):
        return self.csr.dot(x)


def stencil(family, n, dx2=None, fx=None, fy=None, fz=None, dims=None):
    if dims is None:
        dims = {"1d3": (n, 1, 1), "2d5": (n, n, 1), "3d7": (n, n, n), "2d5var": (n, n, 1),
                "3d7var": (n, n, n), "1d3var": (n, 1, 1)}[family]
    dims = tuple(dims) + (1,) * (3 - len(dims))
    if dx2 is None:
        dx2 = (dims[0] + 1.0) ** 2

    def arr(a):
        return None if a is None else np.ascontiguousarray(a, dtype=np.float64)
    return StencilCPU(family, *dims, dx2=dx2, fx=arr(fx), fy=arr(fy), fz=arr(fz))


# ---------------------------------------------------------------- solver

@dataclass
class CycleRecord:
    cycle: int
    level: int
    M: int
    executed: int
    res_before: float
    res_after: float
    rate: float


@dataclass
class OracleReport:
    converged: bool
    total: int
    cycles: list
    x: np.ndarray
    history: list = field(default_factory=list)
    seconds: float = 0.0


class OracleDiverged(FloatingPointError):
    def __init__(self, sweep, omega):
        super().__init__(f"diverged at sweep {sweep} (omega {omega})")
        self.sweep, self.omega = sweep, omega


class Oracle:
    """Restatement of reference solver.run_cycle / solve for L2 norms."""

    def __init__(self, op: StencilCPU, b: np.ndarray):
        self.op = op
        self.b = np.ascontiguousarray(b, dtype=np.float64)

    def cycle(self, x, r, res_now, ordered, tol, budget, baseline, history, total):
        """solver.py:216-249 for an L2 norm; returns (x, r, res, executed, converged)."""
        executed = 0
        for w in ordered:
            if res_now <= tol:
                break
            if executed >= budget:
                break
            x = self.op.update(x, r, w)
            executed += 1
            r, s = self.op.residual(x, self.b)
            res_now = math.sqrt(s) / baseline
            if not math.isfinite(res_now) or not np.all(np.isfinite(x)):
                raise OracleDiverged(executed, w)
            if history is not None:
                history.append((total + executed, res_now))
        return x, r, res_now, executed, res_now <= tol

    def cycle_diff(self, x, res_now, ordered, tol, budget, history, total):
        """solver.py:200-203,216-249 with the solution-difference infinity norm;
        returns (x, res_now, executed, res_before)."""
        executed = 0
        res_before = res_now
        for w in ordered:
            if res_now is not None and res_now <= tol:
                break
            if executed >= budget:
                break
            r, _ = self.op.residual(x, self.b)
            x_new = self.op.update(x, r, w)
            res_now = float(np.max(np.abs(x_new - x)))
            x = x_new
            executed += 1
            if not math.isfinite(res_now) or not np.all(np.isfinite(x)):
                raise OracleDiverged(executed, w)
            if history is not None:
                history.append((total + executed, res_now))
            if res_before is None:
                res_before = res_now
        return x, res_now, executed, res_before

    def solve(self, x0, controller="heuristic", tol=1e-8, relative=True, max_iterations=10**9,
              max_cycles=None, fixed_M=None, record_history=True, t_hi=0.4, t_lo=0.2,
              ordered=None, diff=False):
        """controller: heuristic | increasing | fixed (fixed_M) | jacobi |
        custom (a fixed ordered-omega tuple, e.g. a CJM scheme).  diff: the
        solution-difference infinity norm (heuristic / jacobi controllers)."""
        t0 = time.perf_counter()
        x = np.ascontiguousarray(x0, dtype=np.float64).copy()
        if diff:
            return self._solve_diff(x, controller, tol, max_iterations, record_history, t_hi,
                                    t_lo, t0)
        r, s = self.op.residual(x, self.b)
        baseline = 1.0
        if relative:
            baseline = math.sqrt(s)
            if baseline == 0.0:
                raise ValueError("initial residual is zero")
        res = math.sqrt(s) / baseline
        history = [(0, res)] if record_history else None
        level, total, cycles, ratio_prev = 0, 0, [], None
        converged = False
        while True:
            if controller in ("heuristic", "increasing"):
                M = LADDER[level]
            elif controller == "fixed":
                M = fixed_M
            elif controller == "custom":
                M = len(ordered)
            else:  # jacobi
                M = 1
            if controller == "jacobi":
                seq, lvl = (1.0,), None
            elif controller == "custom":
                seq, lvl = tuple(ordered), None
            else:
                seq, lvl = scheme(M)
            before = res
            x, r, res, executed, conv = self.cycle(x, r, res, seq, tol,
                                                   max_iterations - total, baseline,
                                                   history, total)
            total += executed
            if executed > 0:
                rate = avg_rate(before, res, executed) if before > 0 and res > 0 else math.inf
                cycles.append(CycleRecord(len(cycles), lvl if lvl is not None else -1, M,
                                          executed, before, res, rate))
                ratio_prev = res / before if before > 0 and res > 0 else ratio_prev
            if conv:
                converged = True
                break
            if total >= max_iterations:
                break
            if max_cycles is not None and len(cycles) >= max_cycles:
                break
            if controller == "heuristic":
                if ratio_prev is not None and math.isfinite(ratio_prev):
                    level = next_level(ratio_prev, level, t_hi, t_lo)
            elif controller == "increasing":
                level = min(level + 1, TOP)
        return OracleReport(converged, total, cycles, x, history or [],
                            time.perf_counter() - t0)

    def _solve_diff(self, x, controller, tol, max_iterations, record_history, t_hi, t_lo, t0):
        """solve() under the solution-difference norm (solver.py:289-331 with
        baseline 1 and no initial residual)."""
        history = [] if record_history else None
        level, total, cycles, ratio_prev, res = 0, 0, [], None, None
        converged = False
        while True:
            if controller == "jacobi":
                seq, lvl, M = (1.0,), None, 1
            else:
                M = LADDER[level]
                seq, lvl = scheme(M)
            x, res_now, executed, before = self.cycle_diff(x, res, seq, tol,
                                                           max_iterations - total, history,
                                                           total)
            after = res_now if res_now is not None else float("nan")
            if before is None:
                before = after
            total += executed
            if executed > 0:
                ok = before > 0 and after > 0
                cycles.append(CycleRecord(len(cycles), lvl if lvl is not None else -1, M,
                                          executed, before, after,
                                          avg_rate(before, after, executed) if ok else math.inf))
                if ok:
                    ratio_prev = after / before
            res = res_now
            if res is not None and res <= tol:
                converged = True
                break
            if total >= max_iterations:
                break
            if controller == "heuristic" and ratio_prev is not None and math.isfinite(ratio_prev):
                level = next_level(ratio_prev, level, t_hi, t_lo)
        return OracleReport(converged, total, cycles, x, history or [],
                            time.perf_counter() - t0)


def sweep_count_sample(op: StencilCPU, b, sweeps: int, omega_seq=None):
    """Bounded CPU baseline sample: `sweeps` SRJ sweeps with per-sweep residual
    norms (the reference's per-sweep work), returns seconds."""
    x = np.zeros(op.n)
    r, s = op.residual(x, b)
    seq = omega_seq or scheme(LADDER[10])[0]
    t0 = time.perf_counter()
    for k in range(sweeps):
        x = op.update(x, r, seq[k % len(seq)])
        r, s = op.residual(x, b)
    return time.perf_counter() - t0
