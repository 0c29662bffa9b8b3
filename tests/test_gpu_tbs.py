"""Skewed-tile 2D temporal blocking (srj_tbs.cu) vs the oracle, cycle by cycle.

Grids with several strips, several segments per strip, more than one tile per
CTA, single rows / columns, and every stop position inside a pass (rollback);
the kernel is forced with SRJ_TB_SKEW=1 (small grids default to the square
tiles).  Whole solves: the golden traces and the full-size C2 fixture run it
by default where the plan picks it (tests/test_gpu_fullsize.py).
"""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture()
def force_skew():
    old = os.environ.get("SRJ_TB_SKEW")
    os.environ["SRJ_TB_SKEW"] = "1"
    yield
    if old is None:
        os.environ.pop("SRJ_TB_SKEW", None)
    else:
        os.environ["SRJ_TB_SKEW"] = old


def _oracle_sweeps(op, x, b, omegas, baseline):
    xs, res = [x], []
    for w in omegas:
        r, s = op.residual(xs[-1], b)
        res.append(math.sqrt(s) / baseline)
        xs.append(op.update(xs[-1], r, w))
    _, s = op.residual(xs[-1], b)
    res.append(math.sqrt(s) / baseline)
    return xs, res


@pytest.mark.parametrize("spp", [5, 6])
@pytest.mark.parametrize("dims,stops", [((130, 250), "all"), ((64, 41), "all"), ((2, 300), "all"),
                                        ((400, 1), "all"), ((52, 96), "all"), ((104, 84), "some"),
                                        ((300, 500), "some"), ((1100, 1100), "few")])
def test_tbs_cycle_bitwise_vs_oracle(dims, stops, spp, force_skew):
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny = dims
    dev = torch.device("cuda", 0)
    A = srj.StencilOperator("2d5", dims, dx2=5.0, device=dev)
    A.set_sweeps_per_pass(spp)
    info = A.describe()
    assert info["cycle_kernel"] == 11, info
    op = O.StencilCPU("2d5", nx, ny, 1, 5.0)
    rng = np.random.default_rng(nx * 1000 + ny + spp)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    omegas = rng.uniform(0.4, 2.6, 13)
    baseline = 3.0
    xs, res = _oracle_sweeps(op, x0, b, omegas, baseline)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    bf = A.field(b)
    stop_list = {"all": list(range(1, 13)), "some": [1, 5, 6, 7, 12], "few": [4, 9]}[stops]
    for stop in [None] + stop_list:
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


@pytest.mark.parametrize("name", ["c2_64", "c2_128", "c2_256", "budget_midcycle_2d", "tiny_2d_n2"])
@pytest.mark.parametrize("device_loop", [True, False])
def test_tbs_golden_solves(name, device_loop, force_skew):
    """Reference-run golden 2D solves through the skewed kernel: the device
    controller loop and the per-cycle host loop."""
    import torch

    import _parity as P
    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200 import solver
    c = P.case(name)
    dev = torch.device("cuda", 0)
    fam, n, b, _, _ = P.case_inputs(c)
    A = P.case_operator(c, device=dev)
    assert A.describe()["cycle_kernel"] == 11
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = solver.solve_fields(A, A.field(b), A.new_field(), A.new_field(), srj.Heuristic(), rule,
                              device_loop=device_loop)
    rows = [(q.cycle, q.level, q.M, q.executed, q.residual_before, q.residual_after,
             q.average_rate) for q in rep.cycles]
    P.assert_trace_matches(c, rows, rep.total_iterations, rep.converged, x=rep.x.cpu().numpy())


@pytest.mark.parametrize("seed", range(16))
def test_tbs_random_shapes_bitwise(seed, force_skew):
    """Random even-nx grids (strips with one to fourteen column pairs in the grid,
    one to eight tiles per strip, segments cut at random places by the packing),
    5 or 6 sweeps per pass, one random stop: bit for bit against oracle sweeps."""
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    rng = np.random.default_rng(1000 + seed)
    nx = 2 * int(rng.integers(1, 360))
    ny = int(rng.integers(1, 720))
    spp = int(rng.integers(5, 7))
    M = int(rng.integers(7, 20))
    dev = torch.device("cuda", 0)
    dx2 = float(rng.uniform(1.0, 400.0))
    A = srj.StencilOperator("2d5", (nx, ny), dx2=dx2, device=dev)
    A.set_sweeps_per_pass(spp)
    assert A.describe()["cycle_kernel"] == 11
    op = O.StencilCPU("2d5", nx, ny, 1, dx2)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    omegas = rng.uniform(0.4, 2.6, M)
    baseline = 2.0
    xs, res = _oracle_sweeps(op, x0, b, omegas, baseline)
    om = torch.tensor(omegas, dtype=torch.float64, device=dev)
    bf = A.field(b)
    for stop in (None, int(rng.integers(1, M))):
        tol = 0.0
        if stop is not None:
            tol = res[stop] * (1.0 + 1e-9)
            if any(r <= tol * (1.0 + 1e-9) for r in res[:stop]):
                continue
        x, x_alt = A.field(x0), A.new_field()
        hist = np.zeros(M)
        out = A.run_cycle(x, x_alt, bf, om, M, tol, baseline, res[0], 10**9, hist)
        k = M if stop is None else stop
        assert out.executed == k, (nx, ny, spp, stop, out.executed)
        got = (x_alt if out.result_in_alt else x).interior.cpu().numpy()
        assert np.array_equal(got, xs[k]), (nx, ny, spp, stop, np.max(np.abs(got - xs[k])))
        np.testing.assert_allclose(hist[:k], res[1:k + 1], rtol=1e-12)


def test_skew_kernel_is_chosen_by_region_rows():
    """Default choice (no override): the skewed tiles where they compute fewer
    region rows per CTA and pass than the square ones -- 1024^2 and the C2 grid,
    not 256^2 -- and never for <= 4 sweeps per pass."""
    import torch

    import paper_2011_06636_b200 as srj
    assert "SRJ_TB_SKEW" not in os.environ
    dev = torch.device("cuda", 0)
    for n, want in ((256, 1), (1024, 11), (2048, 11)):
        A = srj.StencilOperator("2d5", (n, n), device=dev)
        assert A.describe()["cycle_kernel"] == want, (n, A.describe())
        A.set_sweeps_per_pass(4)
        assert A.describe()["cycle_kernel"] == 1
