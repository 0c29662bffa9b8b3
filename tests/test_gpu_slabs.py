"""Slab-decomposed solve on the GPU with virtual ranks (GPU).

Several slabs of one grid live on cuda:0 and exchange ghost planes by device
copies (LocalExchanger); the kernels are libsrj's srj_sweep_planes, including
the interior/boundary split used to overlap the halo exchange.  Iterates must
be bit-identical to the reference for every slab count (1..4), and the
scheme sequence identical.
"""

from __future__ import annotations

import numpy as np
import pytest

import _parity as P

pytestmark = pytest.mark.gpu

CASES = ["c3_16", "c3_19", "c3_32", "c2_64", "c2_37", "c4_32", "budget_midcycle_2d",
         "fixed2362_3d"]


def _shape(c):
    n = c["n"]
    return (n, n, n) if c["family"] == "3d7" else (n, n)


def _rows(rep):
    return [(c.cycle, c.level, c.M, c.executed, c.residual_before, c.residual_after,
             c.average_rate) for c in rep.cycles]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_virtual_rank_slabs_match_reference(name, world):
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import LocalExchanger, SlabSolver, local_slabs
    c = P.case(name)
    fam, n, b, fx, fy = P.case_inputs(c)
    slabs = local_slabs(fam, _shape(c), world, range(world), torch.device("cuda", 0),
                        face_x=fx, face_y=fy)
    solver = SlabSolver(slabs, LocalExchanger(world))
    solver.load(b=b)
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    ctrl = c["controller"]
    controller = srj.FixedM(int(ctrl.split(":")[1])) if ctrl.startswith("fixed:") else srj.Heuristic()
    rep = solver.solve(controller, rule, record_history=False)
    P.assert_trace_matches(c, _rows(rep), rep.total_iterations, rep.converged, x=solver.gather())


def test_slab_rhs_generated_on_device_matches_global():
    import torch

    from paper_2011_06636_b200.distributed import LocalExchanger, SlabSolver, local_slabs
    from paper_2011_06636_b200.rng import uniform_rhs
    n = 24
    slabs = local_slabs("3d7", (n, n, n), 3, range(3), torch.device("cuda", 0))
    solver = SlabSolver(slabs, LocalExchanger(3))
    solver.load(seed=7)
    got = np.concatenate([s.b.interior.cpu().numpy() for s in slabs])
    assert np.array_equal(got, uniform_rhs(7, n ** 3))
