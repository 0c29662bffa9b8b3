"""Parity at the BASELINE sizes (C2 2048^2, C4 4096^2 variable coefficient,
C3 512^3): a heuristic solve of the config, capped by a sweep budget that cuts
a cycle mid-way, on the device default kernels vs the OpenMP oracle on the
host -- identical scheme levels, executed counts and sweep totals, the final
iterate bit for bit, residuals to 1e-12.  (The full solves take minutes to
hours on the CPU, so the prefix is what the oracle can check here; the
reduced-size golden traces cover whole solves.)
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,budget", [("c2", 600), ("c4", 250), ("c3", 80)])
def test_baseline_size_prefix_matches_oracle(config, budget):
    import torch

    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    dev = torch.device("cuda", 0)
    prob = srj.config_problem(config, device=dev)
    A = prob.A
    rule = srj.StoppingRule("relative_l2", 1e-8, budget)
    rep = srj.solve(prob, srj.Heuristic(), rule, record_history=False)
    n = A.shape[0]
    if A.family == "2d5var":
        op = O.stencil("2d5var", n, fx=A.face_x, fy=A.face_y)
    else:
        op = O.stencil(A.family, n)
    orc = O.Oracle(op, np.asarray(prob.b)).solve(np.zeros(A.n), controller="heuristic", tol=1e-8,
                                                 max_iterations=budget, record_history=False)
    assert rep.total_iterations == orc.total == budget
    assert [c.level for c in rep.cycles] == [c.level for c in orc.cycles]
    assert [c.executed for c in rep.cycles] == [c.executed for c in orc.cycles]
    np.testing.assert_allclose([c.residual_after for c in rep.cycles],
                               [c.res_after for c in orc.cycles], rtol=1e-12)
    assert np.array_equal(np.asarray(rep.x), orc.x)
