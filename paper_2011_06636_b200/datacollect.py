"""Convergence-data collection for the level-selection thresholds (SURVEY
§8 f1), with the trials batched on the GPU.

Reference: datacollect.py (`_run_trial` :79-117, `collect` :120-131,
`collect_until` :134-147, `aggregate` :156-180, `fit_thresholds` :211-265).
A trial walks the 1D Dirichlet Poisson problem (b = 1, x0 = 0) under a random
level policy: at every step each admissible action's cycle runs from the same
snapshot, one data point per candidate, then one action chosen by the trial's
SplitMix64 stream is followed.  Here all live trials advance in lockstep and a
whole collection step -- every candidate cycle of every trial -- is ONE launch
of `srj_batch_cycles_1d` (one CTA per candidate, iterate in shared memory).
Iterates are bit-identical to the reference; rates and ratios differ only by
the residual norms' summation order (~1e-15), so the walks (levels, actions,
step counts) are identical.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from statistics import NormalDist

import numpy as np

from . import _lib
from .reports import fmt, read_csv, write_csv
from .rng import SplitMix64, derive_seed
from .schemes import LEVEL_TABLE_M, MAX_LEVEL, scheme_for_level
from .solver import average_convergence_rate

ACTIONS = ("increase", "keep", "decrease")
_DELTA = {"increase": 1, "keep": 0, "decrease": -1}
DEFAULT_SIZES = (2, 5, 10, 20, 30, 40, 50, 60, 70, 80, 90, 100, 200, 300, 400)
DEFAULT_TOL = 1e-8
DEFAULT_N_SET = 10_000
INCONCLUSIVE = "inconclusive"
MAX_STEPS_PER_TRIAL = 10_000
MAX_MISBANDED_FRACTION = 0.25


@dataclass(frozen=True)
class DataPoint:
    action: str
    avg_rate: float
    level: int
    prev_ratio: float
    trial: int = 0
    step: int = 0
    res_before: float = math.nan
    res_after: float = math.nan


@dataclass(frozen=True)
class ActionStats:
    mean: float
    ci_halfwidth: float
    count: int


@dataclass(frozen=True)
class ClusterSummary:
    level_bucket: int
    mean_ratio: float
    best_action: str
    actions: dict


class ThresholdFitError(ValueError):
    def __init__(self, message: str, violations):
        super().__init__(message)
        self.violations = violations


def admissible(level: int) -> tuple[str, ...]:
    return tuple(a for a in ACTIONS
                 if not (a == "increase" and level >= MAX_LEVEL)
                 and not (a == "decrease" and level <= 0))


# ---------------------------------------------------------------------------
# Batched trials
# ---------------------------------------------------------------------------

class _Trial:
    __slots__ = ("ident", "N", "rng", "level", "cur", "res", "ratio", "step", "points", "done",
                 "base")

    def __init__(self, ident, N, seed, base):
        self.ident, self.N, self.rng = ident, N, SplitMix64(seed)
        self.level, self.cur, self.base = 0, 0, base
        self.res, self.ratio, self.step = None, None, 0
        self.points, self.done = [], False

    def slot(self, s):
        return self.base + s * self.N


class BatchedTrials:
    """Device pools for a set of trials: every level's ordered omegas (one
    upload), the right-hand sides (ones) and four iterate slots per trial
    (current + up to three candidates)."""

    SLOTS = 4

    def __init__(self, specs, device=None):
        import torch
        self.torch = torch
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        omegas, self.omega_off = [], []
        off = 0
        for level in range(MAX_LEVEL + 1):
            w = scheme_for_level(level).ordered_omegas()
            self.omega_off.append(off)
            omegas.extend(w)
            off += len(w)
        self.omegas = torch.tensor(omegas, dtype=torch.float64, device=self.device)
        sizes = sorted({N for _, N, _ in specs})
        self.b_off = {}
        pos = 0
        for N in sizes:
            self.b_off[N] = pos
            pos += N
        self.b = torch.ones(max(pos, 1), dtype=torch.float64, device=self.device)
        self.trials = []
        base = 0
        for ident, N, seed in specs:
            self.trials.append(_Trial(ident, N, seed, base))
            base += self.SLOTS * N
        self.x = torch.zeros(max(base, 1), dtype=torch.float64, device=self.device)
        self.max_n = max(sizes) if sizes else 1

    def _launch(self, jobs):
        """jobs: list of (trial, level, in_slot, out_slot) -> host sum r^2 per job."""
        torch = self.torch
        arr = (_lib.BatchJob * len(jobs))()
        for j, (t, level, si, so) in enumerate(jobs):
            arr[j] = _lib.BatchJob(t.N, LEVEL_TABLE_M[level], self.omega_off[level], t.slot(si),
                                   t.slot(so), self.b_off[t.N])
        raw = torch.frombuffer(bytearray(ctypes.string_at(arr, ctypes.sizeof(arr))),
                               dtype=torch.uint8).to(self.device)
        out = torch.empty(len(jobs), dtype=torch.float64, device=self.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        rc = _lib.lib().srj_batch_cycles_1d(
            ctypes.c_void_p(raw.data_ptr()), len(jobs), int(self.max_n),
            ctypes.c_void_p(self.omegas.data_ptr()), ctypes.c_void_p(self.x.data_ptr()),
            ctypes.c_void_p(self.b.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            self.device.index if self.device.index is not None else 0, stream)
        if rc != _lib.SRJ_OK:
            raise _lib.SrjLibraryError(f"srj_batch_cycles_1d failed (status {rc})")
        return out.cpu().numpy()

    def run(self, target_tol: float):
        """Advance every trial to completion (reference _run_trial semantics)."""
        live = list(self.trials)
        # cycle 0 at level 0 from x0 = 0: ||b - A 0|| = ||1|| = sqrt(N)
        sums = self._launch([(t, 0, 0, 1) for t in live])
        for t, s in zip(live, sums):
            before, after = math.sqrt(float(t.N)), math.sqrt(s)
            t.cur, t.res = 1, after
            t.ratio = after / before if (before > 0.0 and after > 0.0) else None
        while live:
            jobs, plan = [], []
            for t in live:
                t.step += 1
                if (t.step > MAX_STEPS_PER_TRIAL or (t.res is not None and t.res < target_tol)
                        or t.ratio is None or not math.isfinite(t.ratio)):
                    t.done = True
                    continue
                acts = admissible(t.level)
                free = [s for s in range(self.SLOTS) if s != t.cur]
                cands = []
                for a, so in zip(acts, free):
                    cands.append((a, so, len(jobs)))
                    jobs.append((t, t.level + _DELTA[a], t.cur, so))
                plan.append((t, acts, cands))
            live = [t for t in live if not t.done]
            if not jobs:
                break
            sums = self._launch(jobs)
            for t, acts, cands in plan:
                outcome, step_points, finite = {}, [], True
                for a, so, j in cands:
                    after = math.sqrt(sums[j])
                    M = LEVEL_TABLE_M[t.level + _DELTA[a]]
                    if t.res > 0.0 and after > 0.0:
                        rate = average_convergence_rate(t.res, after, M)
                        ratio = after / t.res
                    else:
                        rate, ratio = math.inf, t.ratio
                    if not math.isfinite(rate):
                        finite = False
                        break
                    outcome[a] = (so, after, ratio)
                    step_points.append(DataPoint(action=a, avg_rate=rate, level=t.level,
                                                 prev_ratio=t.ratio, trial=t.ident, step=t.step,
                                                 res_before=t.res, res_after=after))
                if not finite:
                    t.done = True
                    continue
                t.points.extend(step_points)
                chosen = acts[t.rng.randint(len(acts))]
                t.cur, t.res, t.ratio = outcome[chosen]
                t.level += _DELTA[chosen]
            live = [t for t in live if not t.done]
        return [p for t in self.trials for p in t.points]


def collect(sizes, trials_per_size: int, target_tol: float = DEFAULT_TOL, seed: int = 0,
            device=None) -> list[DataPoint]:
    """`trials_per_size` random-policy trials per size (reference :120-131),
    all trials batched together."""
    if not sizes:
        raise ValueError("need at least one problem size")
    specs, trial = [], 0
    for si, N in enumerate(sizes):
        for t in range(trials_per_size):
            trial += 1
            specs.append((trial, N, derive_seed(seed, si, t)))
    return BatchedTrials(specs, device).run(target_tol)


def collect_until(sizes, min_points: int, target_tol: float = DEFAULT_TOL, seed: int = 0,
                  device=None, rounds_per_batch: int = 8) -> list[DataPoint]:
    """Round-robin trials over the sizes until at least `min_points` exist
    (reference :134-147).  Rounds are batched speculatively; points of rounds
    past the one that reaches `min_points` are discarded, so the result is the
    reference's exactly."""
    if not sizes:
        raise ValueError("need at least one problem size")
    points: list[DataPoint] = []
    round_idx, trial = 0, 0
    while len(points) < min_points:
        specs = []
        for r in range(round_idx, round_idx + rounds_per_batch):
            for si, N in enumerate(sizes):
                trial += 1
                specs.append((trial, N, derive_seed(seed, si, r)))
        by_trial: dict[int, list[DataPoint]] = {}
        for p in BatchedTrials(specs, device).run(target_tol):
            by_trial.setdefault(p.trial, []).append(p)
        idx = 0
        for _ in range(rounds_per_batch):
            for _ in sizes:
                ident = specs[idx][0]
                points.extend(by_trial.get(ident, []))
                idx += 1
            round_idx += 1
            if len(points) >= min_points:
                return points
    return points


# ---------------------------------------------------------------------------
# Aggregation and threshold fit (host; reference :150-265)
# ---------------------------------------------------------------------------

def _z(confidence: float) -> float:
    return 1.96 if confidence == 0.95 else NormalDist().inv_cdf(0.5 * (1.0 + confidence))


def _stats(rates) -> ActionStats:
    k = len(rates)
    mean = sum(rates) / k
    if k < 2:
        return ActionStats(mean=mean, ci_halfwidth=math.inf, count=k)
    var = sum((r - mean) ** 2 for r in rates) / (k - 1)
    return ActionStats(mean=mean, ci_halfwidth=math.sqrt(var / k), count=k)


def _summarize(chunk, level: int, z: float) -> ClusterSummary:
    stats = {}
    for a in ACTIONS:
        rates = [p.avg_rate for p in chunk if p.action == a]
        if rates:
            s = _stats(rates)
            stats[a] = ActionStats(s.mean, z * s.ci_halfwidth, s.count)
    best = INCONCLUSIVE
    if len(stats) >= 2:
        top = max(stats, key=lambda a: stats[a].mean)
        floor = stats[top].mean - stats[top].ci_halfwidth
        if all(floor > s.mean + s.ci_halfwidth for a, s in stats.items() if a != top):
            best = top
    return ClusterSummary(level_bucket=level,
                          mean_ratio=sum(p.prev_ratio for p in chunk) / len(chunk),
                          best_action=best, actions=stats)


def aggregate(points, n_set: int = DEFAULT_N_SET, confidence: float = 0.95):
    """Per level, sort by (prev_ratio, rate, action, trial, step) and cut into
    clusters of n_set points (a tail of >= n_set/10 survives)."""
    if not points:
        raise ValueError("no data points to aggregate")
    z = _z(confidence)
    out = []
    for level in sorted({p.level for p in points}):
        group = sorted((p for p in points if p.level == level),
                       key=lambda p: (p.prev_ratio, p.avg_rate, p.action, p.trial, p.step))
        for lo in range(0, len(group), n_set):
            chunk = group[lo:lo + n_set]
            if len(chunk) >= n_set or len(chunk) >= n_set / 10:
                out.append(_summarize(chunk, level, z))
    return out


def fit_thresholds(clusters) -> tuple[float, float]:
    """(t_hi, t_lo): band boundaries keep < decrease < increase over the
    conclusive clusters placed to minimise misbanded clusters (at most a
    quarter), ties broken by the widest gaps; midpoints of the gaps."""
    conclusive = [c for c in clusters if c.best_action != INCONCLUSIVE]
    for a in ACTIONS:
        if not any(c.best_action == a for c in conclusive):
            raise ValueError(f"no conclusive cluster labeled '{a}'")
    ordered = sorted(conclusive, key=lambda c: (c.mean_ratio, c.level_bucket))
    band = {"keep": 0, "decrease": 1, "increase": 2}
    labels = [band[c.best_action] for c in ordered]
    n = len(ordered)
    # prefix counts of "not keep" and "not decrease", suffix of "not increase"
    not_k = np.concatenate([[0], np.cumsum([lab != 0 for lab in labels])])
    not_d = np.concatenate([[0], np.cumsum([lab != 1 for lab in labels])])
    not_i = np.concatenate([[0], np.cumsum([lab != 2 for lab in labels])])
    best, fallback = None, None
    for i in range(n + 1):
        for j in range(i, n + 1):
            mis = int(not_k[i] + (not_d[j] - not_d[i]) + (not_i[n] - not_i[j]))
            if fallback is None or (mis, i, j) < fallback:
                fallback = (mis, i, j)
            keeps = [c.mean_ratio for c in ordered[:i] if c.best_action == "keep"]
            decs = [c.mean_ratio for c in ordered[i:j] if c.best_action == "decrease"]
            incs = [c.mean_ratio for c in ordered[j:] if c.best_action == "increase"]
            if not (keeps and decs and incs):
                continue
            margin = (min(decs) - max(keeps)) + (min(incs) - max(decs))
            cand = (mis, -margin, i, j, 0.5 * (max(decs) + min(incs)),
                    0.5 * (max(keeps) + min(decs)))
            if best is None or cand < best:
                best = cand
    if best is None or best[0] > MAX_MISBANDED_FRACTION * n:
        mis, i, j = fallback if best is None else (best[0], best[2], best[3])
        wrong = ([c for c in ordered[:i] if c.best_action != "keep"]
                 + [c for c in ordered[i:j] if c.best_action != "decrease"]
                 + [c for c in ordered[j:] if c.best_action != "increase"])
        detail = ", ".join(f"(level={c.level_bucket}, ratio={c.mean_ratio:.4g}, "
                           f"best={c.best_action})" for c in wrong)
        raise ThresholdFitError(
            f"action bands are not ratio-ordered keep < decrease < increase "
            f"({mis}/{n} clusters misbanded): {detail}", wrong)
    return best[4], best[5]


# ---------------------------------------------------------------------------
# File formats (reference :271-320)
# ---------------------------------------------------------------------------

POINTS_HEADER = ["trial", "step", "action", "avg_rate", "level", "prev_ratio"]
CLUSTERS_HEADER = ["level", "mean_ratio", "best_action"] + [
    f"{a}_{f}" for a in ACTIONS for f in ("mean", "ci", "count")]


def write_points_csv(fh, points) -> None:
    write_csv(fh, POINTS_HEADER, ((p.trial, p.step, p.action, p.avg_rate, p.level, p.prev_ratio)
                                  for p in points))


def read_points_csv(path: str):
    header, rows = read_csv(path)
    if header != POINTS_HEADER:
        raise ValueError(f"{path}: unexpected columns {header}")
    return [DataPoint(trial=int(r[0]), step=int(r[1]), action=r[2], avg_rate=float(r[3]),
                      level=int(r[4]), prev_ratio=float(r[5])) for r in rows]


def write_clusters_csv(fh, clusters) -> None:
    rows = []
    for c in clusters:
        row = [c.level_bucket, c.mean_ratio, c.best_action]
        for a in ACTIONS:
            s = c.actions.get(a)
            row += [s.mean, s.ci_halfwidth, s.count] if s else ["", "", 0]
        rows.append(row)
    write_csv(fh, CLUSTERS_HEADER, rows)


def write_thresholds(path: str, t_hi: float, t_lo: float) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"t_hi={fmt(t_hi)}\nt_lo={fmt(t_lo)}\n")


def read_thresholds(path: str) -> tuple[float, float]:
    values = {}
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                key, _, val = line.partition("=")
                values[key.strip()] = float(val)
    if "t_hi" not in values or "t_lo" not in values:
        raise ValueError(f"{path}: expected t_hi= and t_lo= lines")
    return values["t_hi"], values["t_lo"]
