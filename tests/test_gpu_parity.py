"""Device path vs the reference's own traces and the pinned oracle (GPU).

Every golden case (tests/golden/traces.json, produced by running the
reference) is solved through the drop-in API (`solve`) on the B200: the
scheme sequence, executed counts and total sweeps must be identical, the final
iterate bit-identical, and residuals equal to 1e-12 relative.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import _parity as P

pytestmark = pytest.mark.gpu


def device_solve(c, record_history=True, sweeps_per_pass=None, tb_kind=None):
    import torch

    import paper_2011_06636_b200 as srj
    dev = torch.device("cuda", 0)
    if P.is_csr(c):
        csr, b, x0 = P.csr_inputs(c)
        A = srj.SparseMatrix(csr, device=dev)
        n = A.n
    else:
        fam, n, b, _, _ = P.case_inputs(c)
        A = P.case_operator(c, device=dev)
        x0 = np.zeros(A.n)
    if sweeps_per_pass:
        A.set_sweeps_per_pass(sweeps_per_pass)
    if tb_kind:
        A.set_temporal_kernel(tb_kind)
    p = srj.ProblemInstance(A=A, b=b, x0=x0, stopping_norm=c["norm"])
    ctrl = c["controller"]
    if ctrl == "heuristic":
        controller = srj.Heuristic()
    elif ctrl == "increasing":
        controller = srj.Increasing()
    elif ctrl == "jacobi":
        controller = srj.Jacobi()
    elif ctrl.startswith("fixed:"):
        controller = srj.FixedM(int(ctrl.split(":")[1]))
    elif ctrl.startswith("cjm:"):
        mu = float(np.cos(np.pi / (n + 1)))
        controller = srj.Cjm(srj.generate_cjm_scheme(int(ctrl.split(":")[1]), -mu, mu))
    elif ctrl == "blowup":
        controller = srj.Cjm(srj.SrjScheme(M=2, omegas=(1e200, 1.0), application_order=(0, 1)))
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    return srj.solve(p, controller, rule, record_history=record_history)


def rows_of(rep):
    return [(c.cycle, c.level, c.M, c.executed, c.residual_before, c.residual_after,
             c.average_rate) for c in rep.cycles]


NAMES = [c["name"] for c in P.cases(lambda c: "diverged" not in c)]


@pytest.mark.parametrize("name", NAMES)
def test_device_solve_matches_reference(name):
    c = P.case(name)
    rep = device_solve(c, record_history="history" in c)
    P.assert_trace_matches(c, rows_of(rep), rep.total_iterations, rep.converged, x=rep.x,
                           history=rep.residual_history if "history" in c else None)


def test_device_divergence_matches_reference():
    import paper_2011_06636_b200 as srj
    c = P.case("blowup_diverges")
    with pytest.raises(srj.SolveDivergedError) as exc:
        device_solve(c)
    d = exc.value.diagnostics
    want = c["diverged"]
    assert (d["cycle"], d["sweep"], d["omega"], d["level"], d["M"]) == \
        (want["cycle"], want["sweep"], want["omega"], want["level"], want["M"])


def test_run_cycle_snapshots_match_reference():
    import paper_2011_06636_b200 as srj
    snaps = {s["name"]: s for s in P.traces()["run_cycle"]}
    s = snaps["budget3_level3_n50"]
    p = srj.poisson_1d(50)
    st = srj.SolverState(x=p.x0.copy())
    rule = srj.StoppingRule(norm="absolute_l2", tolerance=1e-30, max_iterations=3)
    new, stats = srj.run_cycle(p.A, p.b, st, srj.scheme_for_level(3), stopping=rule)
    assert stats.executed == s["executed"] == 3 and new.converged == s["converged"]
    assert np.array_equal(new.x, np.asarray(s["x"]))
    assert np.array_equal(st.x, np.zeros(50))  # input state untouched
    assert math.isclose(stats.residual_after, s["res_after"], rel_tol=P.RES_RTOL)

    s = snaps["chain_level5_level6_n30"]
    p = srj.poisson_1d(30)
    s2, c2 = srj.run_cycle(p.A, p.b, srj.SolverState(x=p.x0.copy()), srj.scheme_for_level(5))
    s3, c3 = srj.run_cycle(p.A, p.b, s2, srj.scheme_for_level(6))
    assert [c2.executed, c3.executed] == s["executed"]
    assert np.array_equal(s3.x, np.asarray(s["x"]))
    for got, want in zip([(c2.residual_before, c2.residual_after),
                          (c3.residual_before, c3.residual_after)], s["res"]):
        assert math.isclose(got[0], want[0], rel_tol=P.RES_RTOL)
        assert math.isclose(got[1], want[1], rel_tol=P.RES_RTOL)
    assert len(s3.residual_history) == len(s["history"])
    for (i1, r1), (i2, r2) in zip(s3.residual_history, s["history"]):
        assert i1 == i2 and math.isclose(r1, r2, rel_tol=P.RES_RTOL)


def test_solve_is_deterministic_on_device():
    c = P.case("c2_64")
    a = device_solve(c)
    b = device_solve(c)
    assert a.total_iterations == b.total_iterations
    assert np.array_equal(a.x, b.x)
    assert [r.residual_after for r in a.cycles] == [r.residual_after for r in b.cycles]


# --------------------------------------------------------------------------
# Temporal blocking (several sweeps per pass, rollback on a mid-pass stop)
# --------------------------------------------------------------------------

TB_NAMES = [c["name"] for c in P.cases(lambda c: c["family"] == "2d5" and "diverged" not in c)]


@pytest.mark.parametrize("spp", [1, 2, 3, 5, 6, 8])
@pytest.mark.parametrize("name", TB_NAMES)
def test_temporal_blocking_matches_reference(name, spp):
    c = P.case(name)
    rep = device_solve(c, record_history="history" in c, sweeps_per_pass=spp)
    P.assert_trace_matches(c, rows_of(rep), rep.total_iterations, rep.converged, x=rep.x,
                           history=rep.residual_history if "history" in c else None)


def test_standalone_sweep_and_norm_helpers_match_oracle():
    """a6: weighted_jacobi_sweep / matvec / residual norms / diff_inf on device."""
    import paper_2011_06636_b200 as srj
    from oracle import srj_oracle as O
    c = P.case("tridiag_500_seed0")
    csr, b, _ = P.csr_inputs(c)
    A = srj.SparseMatrix(csr)
    x = O.uniform_rhs(9, A.n)
    orc = O.CsrCPU(csr)
    r, s = orc.residual(x, b)
    assert np.array_equal(srj.weighted_jacobi_sweep(A, x, b, 0.7), orc.update(x, r, 0.7))
    assert np.array_equal(srj.matvec(A, x), csr.dot(x))
    assert math.isclose(srj.residual_l2(A, x, b), math.sqrt(s), rel_tol=1e-13)
    S = srj.StencilOperator("3d7", (9, 9, 9))
    xs = O.uniform_rhs(3, S.n)
    bs = O.uniform_rhs(4, S.n)
    ref = O.stencil("3d7", 9)
    rr, _ = ref.residual(xs, bs)
    assert np.array_equal(srj.weighted_jacobi_sweep(S, xs, bs, 1.3), ref.update(xs, rr, 1.3))
    assert np.array_equal(srj.matvec(S, xs), ref.matvec(xs))
    assert srj.diff_inf(xs, bs) == float(np.max(np.abs(xs - bs)))
    with pytest.raises(ValueError):
        srj.matvec(S, xs[:-1])


def test_solve_into_preallocated_out():
    """solve(out=...) writes the solution into the caller's buffer (pinned host
    or device) and returns it as the report's x; values identical to the
    default return path."""
    import torch

    c = P.case("c2_64")
    ref = device_solve(c, record_history=False)
    import paper_2011_06636_b200 as srj
    fam, n, b, _, _ = P.case_inputs(c)
    A = srj.StencilOperator(fam, (n, n))
    p = srj.ProblemInstance(A=A, b=b, x0=np.zeros(A.n), stopping_norm=c["norm"])
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    for out in (torch.empty(A.n, dtype=torch.float64, pin_memory=True),
                torch.empty(A.n, dtype=torch.float64, device="cuda")):
        rep = srj.solve(p, srj.Heuristic(), rule, record_history=False, out=out)
        assert rep.x is out
        assert np.array_equal(out.cpu().numpy(), ref.x)
    with pytest.raises(ValueError):
        srj.solve(p, srj.Heuristic(), rule, out=torch.empty(3, dtype=torch.float64))
