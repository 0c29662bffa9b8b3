"""Reference-style duck-typed operators at the drop-in boundary.

The reference's run_cycle needs only `A.inv_diag` and `A.scipy_csr()`
(reference solver.py:192-193,209,233) and ProblemInstance only `A.n`
(problems.py:37-39).  `sparse.device_operator` wraps any such object: a CSR
that is exactly a Dirichlet stencil goes to the structured kernels, anything
else to the general CSR kernel with the object's own inv_diag.  The GPU tests
pass plain wrappers (not DeviceOperators) through `solve` / `run_cycle` and
match the reference-run traces bit for bit; `SolverState.cached_r` is the
reference's r = b - A x vector, materialised on access.
"""

from __future__ import annotations

import types

import numpy as np
import pytest

import _parity as P
import paper_2011_06636_b200 as srj
from paper_2011_06636_b200.operators import StencilOperator
from paper_2011_06636_b200.sparse import SparseMatrix, device_operator


def duck(csr, inv_diag=None):
    """The minimal operator surface the reference's solver touches."""
    inv = 1.0 / csr.diagonal() if inv_diag is None else inv_diag
    return types.SimpleNamespace(n=csr.shape[0], inv_diag=inv, scipy_csr=lambda: csr)


@pytest.mark.parametrize("family,dims", [("1d3", (37,)), ("2d5", (19, 19)), ("3d7", (7, 7, 7))])
def test_stencil_csr_routes_to_structured_kernels(family, dims):
    ref = StencilOperator(family, dims)          # dx2 = (n+1)^2, reference layout
    op = device_operator(duck(ref.scipy_csr()))
    assert isinstance(op, StencilOperator)
    assert op.family == family and op.shape == dims and op.dx2 == ref.dx2


def test_non_stencil_csr_routes_to_csr_kernel():
    ref = StencilOperator("2d5", (12, 12))
    csr = ref.scipy_csr().copy()
    csr.data[0] *= 1.5                            # one diagonal changed
    op = device_operator(duck(csr))
    assert isinstance(op, SparseMatrix) and op.n == 144
    # a rectangular 2D grid is not detectable as a stencil: CSR path
    op = device_operator(duck(StencilOperator("2d5", (12, 5)).scipy_csr()))
    assert isinstance(op, SparseMatrix)
    # inv_diag not equal to 1/diag: the operator's own inv_diag is used as is
    csr = StencilOperator("1d3", (9,)).scipy_csr()
    inv = np.full(9, 0.25)
    op = device_operator(duck(csr, inv))
    assert isinstance(op, SparseMatrix) and np.array_equal(op.inv_diag, inv)


def test_wrapped_operator_is_cached_per_object():
    d = duck(StencilOperator("3d7", (5, 5, 5)).scipy_csr())
    assert device_operator(d) is device_operator(d)


def test_objects_without_the_operator_surface_are_refused():
    with pytest.raises(TypeError):
        device_operator(types.SimpleNamespace(n=4))


def test_csr_stored_order_is_kept():
    """csr_matvec sums in stored column order, so the wrap keeps a
    non-canonical CSR exactly as stored (no sort, no duplicate merge)."""
    import scipy.sparse
    csr = scipy.sparse.csr_matrix((np.array([2.0, -1.0, -1.0, 2.0]), np.array([1, 0, 1, 0]),
                                   np.array([0, 2, 4])), shape=(2, 2))
    csr.has_sorted_indices = False
    op = device_operator(duck(csr, np.array([1.0, 0.5])))
    assert isinstance(op, SparseMatrix)
    assert list(op.col_idx) == [1, 0, 1, 0]


# --------------------------------------------------------------------- GPU

def _controller(c, n):
    ctrl = c["controller"]
    if ctrl == "heuristic":
        return srj.Heuristic()
    if ctrl.startswith("fixed:"):
        return srj.FixedM(int(ctrl.split(":")[1]))
    if ctrl == "jacobi":
        return srj.Jacobi()
    if ctrl == "increasing":
        return srj.Increasing()
    raise KeyError(ctrl)


def _case_csr(c):
    if P.is_csr(c):
        return P.csr_inputs(c)
    fam, n, b, fx, fy = P.case_inputs(c)
    dims = {"1d3": (n,), "2d5": (n, n), "3d7": (n, n, n)}[fam]
    return StencilOperator(fam, dims).scipy_csr(), b, np.zeros(len(b))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fem_disk", "fem_airfoil_med", "c3_16", "c2_37", "c1_seed0",
                                  "tridiag_500_seed0", "poisson3d_24_ones"])
def test_duck_operator_solve_matches_reference(name):
    c = P.case(name)
    csr, b, x0 = _case_csr(c)
    A = duck(csr)
    p = types.SimpleNamespace(A=A, b=b, x0=x0)   # reference ProblemInstance surface
    rule = srj.StoppingRule(c["norm"], c["tol"], c.get("max_iterations", 10**9))
    rep = srj.solve(p, _controller(c, A.n), rule, record_history=False)
    rows = [(s.cycle, s.level, s.M, s.executed, s.residual_before, s.residual_after,
             s.average_rate) for s in rep.cycles]
    P.assert_trace_matches(c, rows, rep.total_iterations, rep.converged, x=rep.x)


@pytest.mark.gpu
@pytest.mark.parametrize("structured", [True, False])
def test_run_cycle_cached_r_is_the_residual_vector(structured):
    """state.cached_r == b - A x bitwise (reference solver.py:233,270), and
    feeding the state back continues exactly like a fresh residual."""
    ref = StencilOperator("2d5", (24, 24))
    csr = ref.scipy_csr()
    if not structured:
        csr = csr.copy()
        csr.data[csr.data > 0] *= 1.25            # still SPD, no longer a stencil
    A = duck(csr)
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, A.n)
    st = srj.SolverState(x=np.zeros(A.n))
    s1, _ = srj.run_cycle(A, b, st, srj.scheme_for_level(4))
    assert st.cached_r is None                   # input state untouched
    r = s1.cached_r
    assert isinstance(r, np.ndarray)
    assert np.array_equal(r, b - csr.dot(s1.x))
    s2, c2 = srj.run_cycle(A, b, s1, srj.scheme_for_level(5))
    s2b, c2b = srj.run_cycle(A, b, srj.SolverState(x=s1.x.copy()), srj.scheme_for_level(5))
    assert np.array_equal(s2.x, s2b.x)
    assert c2.residual_before == s1.current_residual
    assert np.array_equal(s2.cached_r, b - csr.dot(s2.x))


def test_reference_sparse_matrix_is_accepted():
    """The reference's own SparseMatrix (when /root/reference is mounted, as in
    the build container) wraps to the structured kernel for its Poisson
    generators and to the CSR kernel for its tridiagonal generator."""
    import importlib
    import os
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    sys.path.insert(0, src)
    try:
        ref = importlib.import_module("srj")
        p3 = ref.poisson_3d(6)
        op = device_operator(p3.A)
        assert isinstance(op, StencilOperator) and op.family == "3d7" and op.dx2 == 49.0
        p1 = ref.poisson_1d(40)
        assert isinstance(device_operator(p1.A), StencilOperator)
        t = ref.random_tridiagonal(30, 2)
        op = device_operator(t.A)
        assert isinstance(op, SparseMatrix) and np.array_equal(op.inv_diag, t.A.inv_diag)
    finally:
        sys.path.remove(src)
        for k in [k for k in sys.modules if k == "srj" or k.startswith("srj.")]:
            del sys.modules[k]
