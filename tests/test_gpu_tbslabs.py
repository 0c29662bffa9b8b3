"""Temporally blocked slabs (srj_tb_pass + deep ghost rows / planes) on the GPU.

Several extended slabs of one grid live on cuda:0 (virtual ranks) and exchange
their deep ghost rows (2D: TB_GHOST = 6 rows, 3D: TB3_GHOST = 2 planes) by
device copies before each pass.  Iterates
must be bit-identical to the reference for every slab count, the scheme
sequence identical; the pass kernel alone is checked against the oracle.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import _parity as P

pytestmark = pytest.mark.gpu

CASES = ["c2_64", "c2_37", "c4_32", "c4_64", "budget_midcycle_2d"]
CASES_3D = ["c3_16", "c3_32", "c3_48", "poisson3d_24_ones", "fixed2362_3d"]


def _rows(rep):
    return [(c.cycle, c.level, c.M, c.executed, c.residual_before, c.residual_after,
             c.average_rate) for c in rep.cycles]


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_tb_row_slabs_match_reference(name, world, overlap):
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import (LocalTbExchanger, TbSlabSolver,
                                                   local_tb_slabs)
    c = P.case(name)
    fam, n, b, fx, fy = P.case_inputs(c)
    if n % 2:
        pytest.skip("temporal blocking needs an even row length")
    if n // world < 6:
        pytest.skip("slabs need at least TB_GHOST rows")
    slabs = local_tb_slabs(fam, (n, n), world, range(world), torch.device("cuda", 0),
                           face_x=fx, face_y=fy)
    solver = TbSlabSolver(slabs, LocalTbExchanger(world), overlap=overlap)
    solver.load(b=b)
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = solver.solve(srj.Heuristic(), rule, record_history=False)
    P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged, x=solver.gather())


@pytest.mark.parametrize("family", ["2d5", "2d5var"])
def test_tb_pass_owned_rows_vs_oracle(family):
    """One srj_tb_pass of h sweeps over owned rows [lo, hi) of a grid whose
    outer rows stand in for ghost rows: owned rows equal the oracle's sweeps,
    rows outside are never written, the per-sweep sums are the owned r^2."""
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny, lo, hi = 130, 90, 6, 77
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11)
    kw = {}
    if family == "2d5var":
        fx = rng.uniform(0.5, 30.0, (ny, nx + 1))
        fy = rng.uniform(0.5, 30.0, (ny + 1, nx))
        A = srj.StencilOperator(family, (nx, ny), face_x=fx, face_y=fy, device=dev)
        op = O.StencilCPU(family, nx, ny, 1, 0.0, fx, fy)
    else:
        A = srj.StencilOperator(family, (nx, ny), dx2=5.0, device=dev)
        op = O.StencilCPU(family, nx, ny, 1, 5.0)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    for h in (1, 4, 6):
        omegas = rng.uniform(0.4, 2.6, h)
        xs, sq = [x0], []
        for w in omegas:
            r, _ = op.residual(xs[-1], b)
            sq.append(float(np.sum(r.reshape(ny, nx)[lo:hi] ** 2)))
            xs.append(op.update(xs[-1], r, w))
        x = A.field(x0)
        sentinel = np.full(A.n, 123.0)
        x_alt = A.field(sentinel)
        om = torch.tensor(omegas, dtype=torch.float64, device=dev)
        sums = torch.zeros(h, dtype=torch.float64, device=dev)
        A.tb_pass(x, x_alt, A.field(b), om.data_ptr(), h, lo, hi, sums.data_ptr())
        got = x_alt.interior.cpu().numpy().reshape(ny, nx)
        want = xs[h].reshape(ny, nx)
        assert np.array_equal(got[lo:hi], want[lo:hi]), h
        assert np.all(got[:lo] == 123.0) and np.all(got[hi:] == 123.0), h
        np.testing.assert_allclose(sums.cpu().numpy(), sq, rtol=1e-12)
        assert all(math.isfinite(v) for v in sq)


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name", CASES_3D)
def test_tb_z_slabs_match_reference(name, world, overlap):
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import (LocalTbExchanger, TbSlabSolver,
                                                   local_tb_slabs)
    c = P.case(name)
    fam, n, b, _, _ = P.case_inputs(c)
    assert fam == "3d7"
    if n % 2:
        pytest.skip("temporal blocking needs an even row length")
    if n // world < 2:
        pytest.skip("slabs need at least TB3_GHOST planes")
    slabs = local_tb_slabs(fam, (n, n, n), world, range(world), torch.device("cuda", 0))
    assert all(s.A.describe()["cycle_kernel"] == 5 for s in slabs)
    solver = TbSlabSolver(slabs, LocalTbExchanger(world), overlap=overlap)
    solver.load(b=b)
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    ctrl = c["controller"]
    controller = srj.FixedM(int(ctrl.split(":")[1])) if ctrl.startswith("fixed:") else srj.Heuristic()
    rep = solver.solve(controller, rule, record_history=False)
    P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged, x=solver.gather())


@pytest.mark.parametrize("dims,lo,hi", [((130, 40, 14), 2, 12), ((64, 70, 9), 0, 7),
                                        ((62, 33, 6), 2, 6)])
def test_tb3_pass_owned_planes_vs_oracle(dims, lo, hi):
    """One 3D srj_tb_pass of h <= 2 sweeps over owned planes [lo, hi): owned
    planes equal the oracle's sweeps, planes outside are never written, the
    per-sweep sums are the owned r^2."""
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    nx, ny, nz = dims
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(nx + ny + nz)
    A = srj.StencilOperator("3d7", dims, dx2=5.0, device=dev)
    op = O.StencilCPU("3d7", nx, ny, nz, 5.0)
    b = rng.uniform(-1, 1, A.n)
    x0 = rng.uniform(-1, 1, A.n)
    pl = nx * ny
    for h in (1, 2):
        omegas = rng.uniform(0.4, 2.6, h)
        xs, sq = [x0], []
        for w in omegas:
            r, _ = op.residual(xs[-1], b)
            sq.append(float(np.sum(r[lo * pl:hi * pl] ** 2)))
            xs.append(op.update(xs[-1], r, w))
        x = A.field(x0)
        x_alt = A.field(np.full(A.n, 123.0))
        om = torch.tensor(omegas, dtype=torch.float64, device=dev)
        sums = torch.zeros(h, dtype=torch.float64, device=dev)
        A.tb_pass(x, x_alt, A.field(b), om.data_ptr(), h, lo, hi, sums.data_ptr())
        got = x_alt.interior.cpu().numpy()
        assert np.array_equal(got[lo * pl:hi * pl], xs[h][lo * pl:hi * pl]), h
        assert np.all(got[:lo * pl] == 123.0) and np.all(got[hi * pl:] == 123.0), h
        np.testing.assert_allclose(sums.cpu().numpy(), sq, rtol=1e-12)


@pytest.mark.parametrize("name", ["c2_64", "c4_64", "c3_32"])
def test_tb_slabs_with_reserved_sms(name):
    """Pass kernels that leave SMs free for NCCL (overlapped exchange on real
    multi-GPU runs) give the same iterates."""
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import (LocalTbExchanger, TbSlabSolver,
                                                   local_tb_slabs)
    c = P.case(name)
    fam, n, b, fx, fy = P.case_inputs(c)
    shape = (n, n, n) if fam == "3d7" else (n, n)
    slabs = local_tb_slabs(fam, shape, 2, range(2), torch.device("cuda", 0), face_x=fx, face_y=fy)
    for s in slabs:
        s.A.set_reserved_sms(100)
    solver = TbSlabSolver(slabs, LocalTbExchanger(2), overlap=True)
    solver.load(b=b)
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = solver.solve(srj.Heuristic(), rule, record_history=False)
    P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged, x=solver.gather())


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("name,world", [("c2_64", 3), ("c4_64", 2), ("c3_32", 3)])
def test_tb_slabs_graph_replay_matches_reference(name, world, graphs):
    """The cycle's forward work captured in a CUDA graph and replayed (the
    default with virtual ranks) gives the reference's trace and iterate, and
    so does the eager path."""
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import (LocalTbExchanger, TbSlabSolver,
                                                   local_tb_slabs)
    c = P.case(name)
    fam, n, b, fx, fy = P.case_inputs(c)
    shape = (n, n, n) if fam == "3d7" else (n, n)
    slabs = local_tb_slabs(fam, shape, world, range(world), torch.device("cuda", 0),
                           face_x=fx, face_y=fy)
    solver = TbSlabSolver(slabs, LocalTbExchanger(world), graphs=graphs)
    solver.load(b=b)
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = solver.solve(srj.Heuristic(), rule, record_history=False)
    P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged, x=solver.gather())
    if graphs:
        assert solver._graph_cache, "no cycle was replayed from a graph"


def test_tb_pass_rejects_more_sweeps_than_the_ring(monkeypatch):
    """SRJ_TB_VARIANT=0 pins the S = 4 ring: a 6-sweep srj_tb_pass must fail
    (bad argument) instead of silently running 4 sweeps (advisor finding)."""
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200._lib import SrjLibraryError
    monkeypatch.setenv("SRJ_TB_VARIANT", "0")
    dev = torch.device("cuda", 0)
    A = srj.StencilOperator("2d5", (64, 40), device=dev)
    x, xa, b = A.new_field(), A.new_field(), A.new_field()
    om = torch.ones(6, dtype=torch.float64, device=dev)
    sums = torch.zeros(6, dtype=torch.float64, device=dev)
    with pytest.raises(SrjLibraryError):
        A.tb_pass(x, xa, b, om.data_ptr(), 6, 0, 40, sums.data_ptr())
    A.tb_pass(x, xa, b, om.data_ptr(), 4, 0, 40, sums.data_ptr())  # within the ring: fine


@pytest.mark.parametrize("name", ["c2_64", "c4_64", "c3_32"])
def test_nccl_native_slab_cycle_single_rank(name, tmp_path):
    """The native multi-GPU path (NcclTbExchanger: libsrj's own NCCL
    communicator; srj_slab_cycle_forward issues snapshot, passes with their
    deep-halo exchanges, residual and the all-gather as one C call per cycle)
    on a one-rank job: NCCL loads, the communicator initialises, and the solve
    reproduces the reference.  (Several ranks need several GPUs; the exchange
    offsets are the srj_slab_exchange_plan the virtual-rank tests copy by.)"""
    import torch
    import torch.distributed as dist

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200 import _lib
    from paper_2011_06636_b200.distributed import (NcclTbExchanger, TbSlabSolver,
                                                   local_tb_slabs)
    assert _lib.lib().srj_nccl_available() == 1, _lib.lib().srj_nccl_last_error()
    c = P.case(name)
    fam, n, b, fx, fy = P.case_inputs(c)
    shape = (n, n, n) if fam == "3d7" else (n, n)
    dev = torch.device("cuda", 0)
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0,
                                world_size=1)
    try:
        ex = NcclTbExchanger(dev)
        slabs = local_tb_slabs(fam, shape, 1, [0], dev, face_x=fx, face_y=fy)
        solver = TbSlabSolver(slabs, ex, overlap=False)
        solver.load(b=b)
        rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
        rep = solver.solve(srj.Heuristic(), rule, record_history=False)
        P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged,
                               x=solver.gather())
        ex.close()
    finally:
        if own:
            dist.destroy_process_group()
