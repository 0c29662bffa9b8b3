"""Slab-decomposed solve: protocol tests on CPU (gloo world_size 2 and
in-process virtual ranks) with a numpy slab engine standing in for libsrj.

The engine below restates the per-point arithmetic (ascending CSR columns,
separately rounded) on a slab whose ghost planes are filled by the
exchanger, so the distributed iterates must be bit-identical to the
single-domain oracle and the scheme sequence identical to the reference trace.
"""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch

import _parity as P
from oracle import srj_oracle as O


class NumpySlabEngine:
    """CPU stand-in for DeviceEngine.apply on Fields living in CPU tensors."""

    overlap = True

    def apply(self, slab, xin, xout, w, z0, z1, out, slot):
        lay = slab.layout
        fam = lay.family
        buf = xin.buf.numpy()
        b = slab.b.interior.numpy()
        if fam == "3d7":
            nx, ny = lay.shape[0], lay.shape[1]
            nzl = slab.count
            X = np.pad(buf.reshape(nzl + 2, ny, nx), ((0, 0), (1, 1), (1, 1)))
            B = b.reshape(nzl, ny, nx)
            c = -1.0 * slab.A.dx2
            d = 6.0 * slab.A.dx2
            zs = slice(z0 + 1, z1 + 1)
            ctr = X[zs, 1:-1, 1:-1]
            y = 0.0 + c * X[z0:z1, 1:-1, 1:-1]
            y = y + c * X[zs, :-2, 1:-1]
            y = y + c * X[zs, 1:-1, :-2]
            y = y + d * ctr
            y = y + c * X[zs, 1:-1, 2:]
            y = y + c * X[zs, 2:, 1:-1]
            y = y + c * X[z0 + 2:z1 + 2, 1:-1, 1:-1]
            r = B[z0:z1] - y
            inv = 1.0 / d
            if xout is not None:
                xo = xout.interior.numpy().reshape(nzl, ny, nx)
                xo[z0:z1] = ctr + w * (inv * r)
        else:  # 2d5 row slab
            nx = lay.shape[0]
            nyl = slab.count
            X = np.pad(buf.reshape(nyl + 2, nx), ((0, 0), (1, 1)))
            B = b.reshape(nyl, nx)
            c = -1.0 * slab.A.dx2
            d = 4.0 * slab.A.dx2
            rs = slice(z0 + 1, z1 + 1)
            ctr = X[rs, 1:-1]
            y = 0.0 + c * X[z0:z1, 1:-1]
            y = y + c * X[rs, :-2]
            y = y + d * ctr
            y = y + c * X[rs, 2:]
            y = y + c * X[z0 + 2:z1 + 2, 1:-1]
            r = B[z0:z1] - y
            inv = 1.0 / d
            if xout is not None:
                xo = xout.interior.numpy().reshape(nyl, nx)
                xo[z0:z1] = ctr + w * (inv * r)
        out.fill_(float(np.sum(r * r)))


def _rows(rep):
    return [(c.cycle, c.level, c.M, c.executed, c.residual_before, c.residual_after,
             c.average_rate) for c in rep.cycles]


def _check(c, rep, x):
    P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged, x=x)


CASES = ["c3_16", "c2_32", "c2_37", "budget_midcycle_2d"]


def _shape(c):
    n = c["n"]
    return (n, n, n) if c["family"] == "3d7" else (n, n)


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("name", CASES)
def test_virtual_ranks_match_reference(name, world):
    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import LocalExchanger, SlabSolver, local_slabs
    c = P.case(name)
    fam, n, b, _, _ = P.case_inputs(c)
    slabs = local_slabs(fam, _shape(c), world, range(world), torch.device("cpu"))
    solver = SlabSolver(slabs, LocalExchanger(world), NumpySlabEngine())
    solver.load(b=b)
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = solver.solve(srj.Heuristic(), rule)
    _check(c, rep, solver.gather())


def test_layout_spans_cover_the_grid():
    from paper_2011_06636_b200.distributed import SlabLayout
    for planes in (1, 2, 7, 64, 1024):
        for world in range(1, min(planes, 9) + 1):
            lay = SlabLayout("3d7", (4, 4, planes), world)
            spans = [lay.span(r) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(cnt for _, cnt in spans) == planes
            assert all(s1 + c1 == s2 for (s1, c1), (s2, _) in zip(spans, spans[1:]))
            assert max(cnt for _, cnt in spans) - min(cnt for _, cnt in spans) <= 1
    with pytest.raises(ValueError):
        SlabLayout("1d3", (100,), 2)
    with pytest.raises(ValueError):
        SlabLayout("3d7", (4, 4, 3), 4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, result_path):
    import torch.distributed as dist

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import SlabSolver, TorchExchanger, local_slabs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = P.case(name)
        fam, n, b, _, _ = P.case_inputs(c)
        slabs = local_slabs(fam, _shape(c), world, [rank], torch.device("cpu"))
        solver = SlabSolver(slabs, TorchExchanger(), NumpySlabEngine())
        solver.load(b=b)
        rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
        rep = solver.solve(srj.Heuristic(), rule)
        x = solver.gather()
        if rank == 0:
            np.savez(result_path, x=x, rows=np.array(_rows(rep), dtype=float),
                     total=rep.total_iterations, converged=rep.converged)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c3_16", "c2_37"])
def test_gloo_world2_matches_reference(name, tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    z = np.load(out)
    c = P.case(name)
    rows = [tuple(r) for r in z["rows"]]
    P.assert_trace_matches(c, rows, int(z["total"]), bool(z["converged"]), x=z["x"])


def test_oracle_and_slab_norms_agree():
    # the gathered per-sweep norms equal the oracle's to summation-order noise
    from paper_2011_06636_b200.distributed import LocalExchanger, SlabSolver, local_slabs
    n = 10
    b = O.uniform_rhs(3, n ** 3)
    slabs = local_slabs("3d7", (n, n, n), 3, range(3), torch.device("cpu"))
    solver = SlabSolver(slabs, LocalExchanger(3), NumpySlabEngine())
    solver.load(b=b)
    r0 = solver.residual_norm()
    _, s = O.stencil("3d7", n).residual(np.zeros(n ** 3), b)
    assert math.isclose(r0, math.sqrt(s), rel_tol=1e-13)
