"""Constant-coefficient 2D temporal blocking (srj_tb.cu) vs the oracle, cycle by cycle.

Both tile variants (S = 4 ring for <= 4 sweeps per pass, S = 6 ring for 5-6)
on multi-tile, non-square, single-row and odd-nx grids, with every stop
position inside a pass (rollback) exercised; the golden solves in
test_gpu_parity.py cover the reference traces.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle_sweeps(op, x, b, omegas, baseline):
    xs, res = [x], []
    for w in omegas:
        r, s = op.residual(xs[-1], b)
        res.append(math.sqrt(s) / baseline)
        xs.append(op.update(xs[-1], r, w))
    _, s = op.residual(xs[-1], b)
    res.append(math.sqrt(s) / baseline)
    return xs, res


@pytest.mark.parametrize("spp", [4, 6])
@pytest.mark.parametrize("dims,kernel", [((130, 90), 1), ((64, 41), 1), ((2, 300), 1),
                                         ((400, 1), 1), ((33, 17), 0)])
def test_tb2d_cycle_bitwise_vs_oracle(dims, kernel, spp):
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny = dims
    dev = torch.device("cuda", 0)
    A = srj.StencilOperator("2d5", dims, dx2=5.0, device=dev)
    A.set_sweeps_per_pass(spp)
    assert A.describe()["cycle_kernel"] == kernel
    op = O.StencilCPU("2d5", nx, ny, 1, 5.0)
    rng = np.random.default_rng(nx * 1000 + ny + spp)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    omegas = rng.uniform(0.4, 2.6, 13)
    baseline = 3.0
    xs, res = _oracle_sweeps(op, x0, b, omegas, baseline)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    bf = A.field(b)
    for stop in [None] + list(range(1, 13)):
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


@pytest.mark.parametrize("family", ["2d5", "2d5var"])
def test_negative_zero_start(family):
    """x0 holding -0.0 entries (and b zero there): the TB kernels skip the
    reference's leading `0 +`, so at most the sign of a zero may differ --
    the values equal the oracle's."""
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny = 66, 70
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    if family == "2d5var":
        fx = rng.uniform(0.5, 30.0, (ny, nx + 1))
        fy = rng.uniform(0.5, 30.0, (ny + 1, nx))
        A = srj.StencilOperator(family, (nx, ny), face_x=fx, face_y=fy, device=dev)
        op = O.StencilCPU(family, nx, ny, 1, 0.0, fx, fy)
    else:
        A = srj.StencilOperator(family, (nx, ny), dx2=5.0, device=dev)
        op = O.StencilCPU(family, nx, ny, 1, 5.0)
    x0 = np.where(rng.random(A.n) < 0.5, -0.0, 0.0)
    b = np.where(rng.random(A.n) < 0.97, 0.0, rng.uniform(-1, 1, A.n))
    omegas = rng.uniform(0.4, 2.6, 6)
    xs = [x0]
    for w in omegas:
        r, _ = op.residual(xs[-1], b)
        xs.append(op.update(xs[-1], r, w))
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    x, x_alt = A.field(x0), A.new_field()
    out = A.run_cycle(x, x_alt, A.field(b), om, 6, 0.0, 1.0, 1.0, 10**9, None)
    got = (x_alt if out.result_in_alt else x).interior.cpu().numpy()
    assert np.array_equal(got, xs[6])  # -0.0 == +0.0


@pytest.mark.parametrize("family", ["2d5", "2d5var"])
def test_subnormal_products_start(family):
    """x0 with subnormal entries, so that c_off * x is subnormal in the first
    sweep (the TB kernels' `fma(p, -4, y)` diagonal and the dropped
    leading `0 +` are exact only for normal-or-zero products).  Records the
    behaviour: the iterates must equal the oracle's to within one unit in the
    last place of the result scale (they are bit-identical unless a subnormal
    product changes a rounding)."""
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny = 66, 70
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    kw = {}
    if family == "2d5var":
        fx = rng.uniform(0.5, 3.0, (ny, nx + 1))
        fy = rng.uniform(0.5, 3.0, (ny + 1, nx))
        A = srj.StencilOperator(family, (nx, ny), face_x=fx, face_y=fy, device=dev)
        op = O.StencilCPU(family, nx, ny, 1, 0.0, fx, fy)
    else:
        A = srj.StencilOperator(family, (nx, ny), dx2=5.0, device=dev)
        op = O.StencilCPU(family, nx, ny, 1, 5.0)
    assert A.describe()["tb_supported"]
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n) * 1e-310          # subnormal start
    omegas = rng.uniform(0.4, 1.6, 6)
    xs, res = _oracle_sweeps(op, x0, b, omegas, 1.0)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    x = A.field(x0)
    x_alt = A.new_field()
    out = A.run_cycle(x, x_alt, A.field(b), om, len(omegas), 0.0, 1.0, res[0], 10**9,
                      np.zeros(len(omegas)))
    got = (x_alt if out.result_in_alt else x).interior.cpu().numpy()
    want = xs[len(omegas)]
    scale = np.max(np.abs(want))
    assert np.max(np.abs(got - want)) <= 2.0 ** -52 * scale, np.max(np.abs(got - want))
