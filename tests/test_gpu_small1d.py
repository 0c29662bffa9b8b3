"""1D cycle kernels vs the oracle: the single-CTA register-resident kernel
(n <= 4096, BASELINE config 1), the single-CTA shared-memory kernel (n <= 8192)
and the generic row walker above it, swept
cycle by cycle with every stop position, plus a residual-only evaluation.
The 1D golden solves (test_gpu_parity.py) already run through the small kernel.
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


@pytest.mark.parametrize("n,kernel", [(1, 8), (2, 8), (127, 8), (200, 8), (1000, 8), (1024, 8),
                                      (2048, 8), (4096, 8), (4097, 7), (8192, 7), (8193, 0),
                                      (20000, 0)])
def test_1d_cycle_bitwise_vs_oracle(n, kernel):
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    dev = torch.device("cuda", 0)
    A = srj.StencilOperator("1d3", (n,), device=dev)
    assert A.describe()["cycle_kernel"] == kernel
    op = O.stencil("1d3", n)
    rng = np.random.default_rng(n)
    b = rng.uniform(-1, 1, n)
    x0 = rng.uniform(-1, 1, n)
    omegas = rng.uniform(0.4, 2.6, 7)
    baseline = 2.0
    xs, res = _oracle_sweeps(op, x0, b, omegas, baseline)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    bf = A.field(b)
    assert math.isclose(math.sqrt(A.residual_sq(A.field(x0), bf)) / baseline, res[0],
                        rel_tol=1e-12)
    for stop in [None] + list(range(1, 7)):
        if stop is None:
            tol = 0.0
        else:
            tol = res[stop] * (1.0 + 1e-9)
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
