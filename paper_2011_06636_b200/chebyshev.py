"""Chebyshev quantities the SRJ scheme family is built from (host side).

Only what the solve path consumes lives here: the Chebyshev roots, the anchor
point lambda* where T_M(lambda*) = 3, the captured eigenvalue bound
lambda_max(M), and G_M(lambda) = T_M(f(lambda)) / 3 for diagnostics.

Parity: `cheb_roots`, `lambda_star` and `lambda_max` must produce the same
float64 bits as the reference (they feed the relaxation factors that the
device sweeps consume), so the floating-point expressions are evaluated in the
same order as the published formulas:
  - roots  x_j = cos(pi (2j+1) / (2M))        (reference chebyshev.py:82-87)
  - lambda* = cosh(acosh(3) / M)              (reference chebyshev.py:90-94)
  - lambda_max = (3 - lambda*) / (1 + lambda*) (reference chebyshev.py:117-120)
"""

from __future__ import annotations

import math

import numpy as np

ACOSH3 = math.acosh(3.0)


def cheb_roots(M: int) -> np.ndarray:
    """Roots of T_M, descending: cos(pi (2j+1) / (2M)) for j = 0..M-1."""
    if M < 1:
        raise ValueError("degree must be positive")
    odd = 2 * np.arange(M) + 1
    return np.cos(np.pi * odd / (2 * M))


def lambda_star(M: int) -> float:
    """lambda* > 1 with T_M(lambda*) = 3."""
    if M < 1:
        raise ValueError("degree must be positive")
    return math.cosh(ACOSH3 / M)


def lambda_max(M: int) -> float:
    """Largest Jacobi eigenvalue with |G_M| <= 1/3."""
    ls = lambda_star(M)
    return (3.0 - ls) / (1.0 + ls)


def cheb_eval(M: int, x):
    """T_M(x): trigonometric form inside [-1, 1], hyperbolic form outside."""
    if M < 0:
        raise ValueError("degree must be nonnegative")
    arr = np.atleast_1d(np.asarray(x, dtype=float))
    out = np.empty_like(arr)
    inner = np.abs(arr) <= 1.0
    out[inner] = np.cos(M * np.arccos(arr[inner]))
    outer = ~inner
    a = np.abs(arr[outer])
    excess = a - 1.0
    acosh = np.log1p(excess + np.sqrt(excess * (2.0 + excess)))
    sign = np.where(arr[outer] < 0.0, (-1.0) ** M, 1.0)
    out[outer] = sign * np.cosh(M * acosh)
    return float(out[0]) if np.ndim(x) == 0 else out


def amplification_eval(M: int, lam):
    """G_M(lambda) = T_M(((lambda*+1) lambda + (lambda*-1)) / 2) / 3."""
    ls = lambda_star(M)
    lam = np.asarray(lam, dtype=float)
    arg = ((ls + 1.0) * lam + (ls - 1.0)) / 2.0
    val = cheb_eval(M, arg if arg.ndim else float(arg))
    return val / 3.0
