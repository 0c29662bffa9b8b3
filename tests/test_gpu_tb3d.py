"""3D temporal blocking (srj_tb3d.cu) against the reference traces and the oracle.

The 3D golden cases run with both cycle kernels (sweeps_per_pass 1: the plane
ring k_cycle3d; 2, the default: the z-wavefront k_tb3d_cycle), and a
multi-tile, non-cubic grid is swept cycle by cycle against oracle sweeps with
every stop position inside a pass (rollback) exercised.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import _parity as P
from test_gpu_parity import device_solve, rows_of

pytestmark = pytest.mark.gpu

NAMES_3D = [c["name"] for c in P.cases(lambda c: c["family"] == "3d7" and "diverged" not in c)]


@pytest.mark.parametrize("spp", [1, 2])
@pytest.mark.parametrize("name", NAMES_3D)
def test_3d_cycle_kernels_match_reference(name, spp):
    c = P.case(name)
    rep = device_solve(c, record_history="history" in c, sweeps_per_pass=spp)
    P.assert_trace_matches(c, rows_of(rep), rep.total_iterations, rep.converged, x=rep.x,
                           history=rep.residual_history if "history" in c else None)


def _oracle_sweeps(op, x, b, omegas, baseline):
    """x_k and the relative residual of x_k for k = 0..len(omegas)."""
    xs, res = [x], []
    for w in omegas:
        r, s = op.residual(xs[-1], b)
        res.append(math.sqrt(s) / baseline)
        xs.append(op.update(xs[-1], r, w))
    _, s = op.residual(xs[-1], b)
    res.append(math.sqrt(s) / baseline)
    return xs, res


@pytest.mark.parametrize("dims", [(130, 40, 12), (64, 17, 5), (62, 33, 3)])
def test_tb3d_cycle_bitwise_vs_oracle(dims):
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny, nz = dims
    dev = torch.device("cuda", 0)
    A = srj.StencilOperator("3d7", dims, dx2=7.0, device=dev)
    A.set_sweeps_per_pass(2)
    info = A.describe()
    assert info["cycle_kernel"] == 5, info  # k_tb3d_cycle
    op = O.StencilCPU("3d7", nx, ny, nz, dx2=7.0)
    rng = np.random.default_rng(nx * 1000 + ny * 10 + nz)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    omegas = rng.uniform(0.4, 2.6, 9)
    baseline = 3.0
    xs, res = _oracle_sweeps(op, x0, b, omegas, baseline)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    bf = A.field(b)
    # no stop: all 9 sweeps (4 full passes + a 1-sweep pass), then every stop
    # position k = 1..8 (odd k stops inside a pass: rollback)
    for stop in [None] + list(range(1, 9)):
        if stop is None:
            tol = 0.0
        else:
            # a margin well above the device/oracle norm difference (~1e-16)
            tol = res[stop] * (1.0 + 1e-9)
            if any(r <= tol * (1.0 + 1e-9) for r in res[:stop]):  # stops earlier
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
