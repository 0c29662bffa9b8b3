"""SRJ relaxation schedules: the host-side producer of the omega sequence the
device sweeps consume.

A scheme of length M carries one factor per Chebyshev root,
omega_j = (lambda* + 1) / (2 (lambda* - x_j)) (reference schemes.py:72-75),
each used exactly once per cycle (Q = 1), applied in a stability order that
pairs the strongest remaining over-relaxation with the weakest
under-relaxation recursively (reference schemes.py:78-120).  The order is
certified on a uniform grid over [-1, lambda_max(M)]: every running partial
amplification product must stay below e^700.

The omegas are produced bit-identically to the reference so that device
iterates match the CPU reference bit for bit; `ordered_omegas` is what is
uploaded to HBM (one contiguous fp64 array per scheme).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .chebyshev import cheb_roots, lambda_max, lambda_star

MAX_SCHEME_LENGTH = 10_000
ORDER_GRID_SIZE = 512

# Pinned 25-level ladder of scheme lengths (reference schemes.py:31-34).
LEVEL_TABLE_M = (
    1, 2, 3, 5, 7, 10, 14, 19, 26, 35, 47, 63, 84, 111, 147,
    194, 256, 338, 446, 589, 778, 1027, 1356, 1790, 2362,
)
MAX_LEVEL = len(LEVEL_TABLE_M) - 1

_LOG_OVERFLOW = 700.0  # e^700 is close to the float64 overflow threshold


@dataclass(frozen=True)
class SrjScheme:
    """Factors in root order plus the order in which a cycle applies them.

    omegas[j] belongs to the j-th descending Chebyshev root and
    application_order[k] names the factor used by sweep k.
    """

    M: int
    omegas: tuple[float, ...]
    application_order: tuple[int, ...]
    level: int | None = None

    def ordered_omegas(self) -> tuple[float, ...]:
        return tuple(self.omegas[j] for j in self.application_order)


def srj_omegas(M: int) -> np.ndarray:
    """omega_j over the descending roots x_j of T_M."""
    ls = lambda_star(M)
    x = cheb_roots(M)
    return (ls + 1.0) / (2.0 * (ls - x))


def _fold_pairs(ranked: list[int]) -> list[int]:
    """Recursive strongest/weakest pairing, flattened.

    At each round the unit list is folded in half (unit i joined with unit
    -1-i); an odd middle unit is set aside and emitted after everything the
    deeper rounds produce, innermost rounds' middles first.
    """
    units = [[j] for j in ranked]
    trailing: list[list[int]] = []
    while len(units) > 2:
        half = len(units) // 2
        middle = [units[half]] if len(units) % 2 else []
        units = [units[i] + units[len(units) - 1 - i] for i in range(half)]
        trailing = middle + trailing
    return [j for unit in units + trailing for j in unit]


def certify_order(omegas, order, M: int, grid_size: int) -> float:
    """Largest log partial product of |1 - w (1 - lambda)| over the grid."""
    grid = np.linspace(-1.0, lambda_max(M), grid_size)
    w = np.asarray(omegas)[np.asarray(order)]
    logs = np.log(np.maximum(np.abs(1.0 - w[:, None] * (1.0 - grid[None, :])), 1e-300))
    running = np.cumsum(logs, axis=0)
    return float(running.max())


def order_for_stability(scheme: SrjScheme, grid_size: int = ORDER_GRID_SIZE) -> tuple[int, ...]:
    if grid_size < 64:
        raise ValueError("grid_size must be at least 64")
    omegas = np.asarray(scheme.omegas)
    M = len(omegas)
    if M == 1:
        return (0,)
    ranked = sorted(range(M), key=lambda j: -omegas[j])  # stable: ties keep root order
    order = tuple(_fold_pairs(ranked))
    peak = certify_order(omegas, order, M, grid_size)
    if not np.isfinite(peak) or peak > _LOG_OVERFLOW:
        raise ValueError(f"no stable ordering certified for M={M} (peak e^{peak:.0f})")
    return order


@lru_cache(maxsize=256)
def generate_srj_scheme(M: int, grid_size: int = ORDER_GRID_SIZE) -> SrjScheme:
    if not 1 <= M <= MAX_SCHEME_LENGTH:
        raise ValueError(f"scheme length M={M} out of range [1, {MAX_SCHEME_LENGTH}]")
    omegas = tuple(float(w) for w in srj_omegas(M))
    level = LEVEL_TABLE_M.index(M) if M in LEVEL_TABLE_M else None
    draft = SrjScheme(M=M, omegas=omegas, application_order=tuple(range(M)), level=level)
    return SrjScheme(M=M, omegas=omegas,
                     application_order=order_for_stability(draft, grid_size), level=level)


def scheme_for_level(level: int, grid_size: int = ORDER_GRID_SIZE) -> SrjScheme:
    if not 0 <= level <= MAX_LEVEL:
        raise ValueError(f"level {level} outside [0, {MAX_LEVEL}]")
    return generate_srj_scheme(LEVEL_TABLE_M[level], grid_size)


@lru_cache(maxsize=256)
def generate_cjm_scheme(M: int, lam_lo: float, lam_hi: float,
                        grid_size: int = ORDER_GRID_SIZE) -> SrjScheme:
    """Chebyshev factors 1/(1 - lambda_j) for roots mapped onto [lam_lo, lam_hi]
    (comparator controller; reference schemes.py:141-160)."""
    if not 1 <= M <= MAX_SCHEME_LENGTH:
        raise ValueError(f"scheme length M={M} out of range [1, {MAX_SCHEME_LENGTH}]")
    if not (-1.0 <= lam_lo < lam_hi < 1.0):
        raise ValueError(f"invalid eigenvalue interval [{lam_lo}, {lam_hi}]")
    centre = 0.5 * (lam_hi + lam_lo)
    radius = 0.5 * (lam_hi - lam_lo)
    lam = centre + radius * cheb_roots(M)
    omegas = tuple(float(1.0 / (1.0 - v)) for v in lam)
    draft = SrjScheme(M=M, omegas=omegas, application_order=tuple(range(M)))
    return SrjScheme(M=M, omegas=omegas, application_order=order_for_stability(draft, grid_size))
