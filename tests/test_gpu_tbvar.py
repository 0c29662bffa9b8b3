"""Variable-coefficient temporal blocking (srj_tbvar.cu) vs the reference and the oracle.

The 2D variable-coefficient golden cases run with every sweeps-per-pass
setting (1: the single-sweep tile kernel k_cycle2d<1>; 2-6: k_tbvar_cycle,
larger requests clamp to 6), and multi-tile grids with random positive faces
are swept cycle by cycle against oracle sweeps with every stop position inside
a pass (rollback) exercised.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import _parity as P
from test_gpu_parity import device_solve, rows_of

pytestmark = pytest.mark.gpu

NAMES_VAR = [c["name"] for c in P.cases(lambda c: c["family"] == "2d5var" and "diverged" not in c)]


@pytest.mark.parametrize("spp", [1, 2, 3, 4, 5, 6, 8])
@pytest.mark.parametrize("name", NAMES_VAR)
def test_varcoef_cycle_kernels_match_reference(name, spp):
    c = P.case(name)
    rep = device_solve(c, record_history="history" in c, sweeps_per_pass=spp)
    P.assert_trace_matches(c, rows_of(rep), rep.total_iterations, rep.converged, x=rep.x,
                           history=rep.residual_history if "history" in c else None)


def _oracle_sweeps(op, x, b, omegas, baseline):
    xs, res = [x], []
    for w in omegas:
        r, s = op.residual(xs[-1], b)
        res.append(math.sqrt(s) / baseline)
        xs.append(op.update(xs[-1], r, w))
    _, s = op.residual(xs[-1], b)
    res.append(math.sqrt(s) / baseline)
    return xs, res


@pytest.mark.parametrize("dims,kernel", [((130, 90), 6), ((64, 41), 6), ((58, 200), 6),
                                         ((2, 2), 6), ((400, 1), 6), ((33, 17), 0)])
def test_tbvar_cycle_bitwise_vs_oracle(dims, kernel):
    """kernel 6: k_tbvar_cycle; odd nx (no 16-byte TMA row pitch for any tile
    kernel) falls back to the generic row walker k_cycle (0)."""
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny = dims
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(nx * 1000 + ny)
    fx = rng.uniform(0.5, 30.0, (ny, nx + 1))
    fy = rng.uniform(0.5, 30.0, (ny + 1, nx))
    A = srj.StencilOperator("2d5var", dims, face_x=fx, face_y=fy, device=dev)
    assert A.describe()["cycle_kernel"] == kernel
    op = O.StencilCPU("2d5var", nx, ny, 1, 0.0, fx, fy)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    omegas = rng.uniform(0.4, 2.6, 11)
    baseline = 3.0
    xs, res = _oracle_sweeps(op, x0, b, omegas, baseline)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    bf = A.field(b)
    # no stop: 11 sweeps (a full pass + a 5-sweep pass); then every stop k
    for stop in [None] + list(range(1, 11)):
        if stop is None:
            tol = 0.0
        else:
            tol = res[stop] * (1.0 + 1e-9)  # margin above the norm-order difference
            if any(r <= tol * (1.0 + 1e-9) for r in res[:stop]):
                continue
        x = A.field(x0)
        x_alt = A.new_field()
        hist = np.zeros(len(omegas))
        out = A.run_cycle(x, x_alt, bf, om, len(omegas), tol, baseline, res[0], 10**9, hist)
        k = len(omegas) if stop is None else stop
        assert out.executed == k, (stop, out.executed)
        got = (x_alt if out.result_in_alt else x).interior.cpu().numpy()
        assert np.array_equal(got, xs[k]), (stop, np.max(np.abs(got - xs[k])))
        np.testing.assert_allclose(hist[:k], res[1:k + 1], rtol=1e-12)
        np.testing.assert_allclose(out.res_after, res[k], rtol=1e-12)
