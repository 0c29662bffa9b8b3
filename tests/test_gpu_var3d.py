"""3D variable-coefficient kernels against the reference's traces (GPU).

The reference-run golden cases c3v_* (tests/golden/make_golden.py --var:
SparseMatrix.from_coo of the 7-point harmonic-face operator solved by the
reference) through both device kernels: the one-sweep plane ring
(k_cycle3dv, default) and the two-sweep z-wavefront (k_tb3v_cycle,
sweeps_per_pass = 2), with the device-resident controller loop and the host
loop; identical scheme sequence, bit-identical iterate.
"""

from __future__ import annotations

import numpy as np
import pytest

import _parity as P

pytestmark = pytest.mark.gpu

CASES = ["c3v_12", "c3v_20", "c3v_31", "c3v_32", "c3v_24_budget"]


@pytest.mark.parametrize("device_loop", [True, False])
@pytest.mark.parametrize("spp", [1, 2])
@pytest.mark.parametrize("name", CASES)
def test_var3d_kernels_match_reference(name, spp, device_loop):
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.solver import solve_fields
    c = P.case(name)
    fam, n, b, _, _ = P.case_inputs(c)
    dev = torch.device("cuda", 0)
    A = P.case_operator(c, device=dev)
    A.set_sweeps_per_pass(spp)
    info = A.describe()
    if n % 2 == 0:
        assert info["cycle_kernel"] == (10 if spp == 2 else 9), info
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = solve_fields(A, A.field(b), A.field(np.zeros(A.n)), A.new_field(), srj.Heuristic(), rule,
                       record_history=False, device_loop=device_loop)
    rows = [(s.cycle, s.level, s.M, s.executed, s.residual_before, s.residual_after,
             s.average_rate) for s in rep.cycles]
    P.assert_trace_matches(c, rows, rep.total_iterations, rep.converged, x=rep.x.cpu().numpy())
