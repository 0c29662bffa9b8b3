"""Host-side drop-in logic (CPU): schemes, Chebyshev quantities, controllers,
RNG and problem/operator metadata against the reference's own values."""

from __future__ import annotations

import math

import numpy as np
import pytest

import _parity as P
import paper_2011_06636_b200 as srj
from paper_2011_06636_b200 import chebyshev as ch
from paper_2011_06636_b200 import schemes as sc
from paper_2011_06636_b200.rng import SplitMix64, derive_seed, uniform_rhs, uniforms_counter


def test_scheme_ladder_matches_reference_bitwise():
    z = P.schemes_npz()
    assert len(srj.LEVEL_TABLE_M) == 25 and srj.MAX_LEVEL == 24
    for level in range(25):
        s = srj.scheme_for_level(level)
        assert s.M == srj.LEVEL_TABLE_M[level] and s.level == level
        assert np.array_equal(np.array(s.omegas), z[f"omegas_{level}"])
        assert s.application_order == tuple(int(v) for v in z[f"order_{level}"])


def test_scheme_properties():
    # Table 2 style facts: M=1 is omega = 2/3; largest factor applied first
    assert srj.generate_srj_scheme(1).omegas == pytest.approx((2.0 / 3.0,))
    for M in (2, 5, 47, 2362):
        s = srj.generate_srj_scheme(M)
        assert sorted(s.application_order) == list(range(M))
        assert s.ordered_omegas()[0] == max(s.omegas)
        # omegas descend with the roots; each is 1/(1 - lambda_j) of a G_M root
        assert all(a > b for a, b in zip(s.omegas, s.omegas[1:]))
        lam = 1.0 - 1.0 / np.asarray(s.omegas)
        assert np.max(np.abs(ch.amplification_eval(M, lam))) < 1e-6
    with pytest.raises(ValueError):
        srj.generate_srj_scheme(0)
    with pytest.raises(ValueError):
        srj.scheme_for_level(25)
    with pytest.raises(ValueError):
        sc.order_for_stability(srj.generate_srj_scheme(5), grid_size=10)


def test_chebyshev_closed_forms():
    assert ch.lambda_star(1) == pytest.approx(3.0)
    assert ch.lambda_max(1) == pytest.approx(0.0)
    assert np.allclose(ch.cheb_roots(2), [math.sqrt(0.5), -math.sqrt(0.5)])
    assert ch.cheb_eval(3, 0.5) == pytest.approx(4 * 0.125 - 3 * 0.5)
    assert ch.cheb_eval(4, 1.5) == pytest.approx(8 * 1.5**4 - 8 * 1.5**2 + 1)
    for M in (1, 3, 10, 84):
        assert ch.amplification_eval(M, 1.0) == pytest.approx(1.0)


def test_heuristic_rules_match_reference_tests():
    h = srj.heuristic_next_level
    assert h(0.5, 3) == 4 and h(0.3, 5) == 4 and h(0.1, 5) == 5 and h(0.3, 0) == 0
    assert h(0.4, 7) == 7 and h(0.9, srj.MAX_LEVEL) == srj.MAX_LEVEL
    assert h(0.2, 7) == 7  # exactly t_lo keeps
    assert h(0.35, 3, t_hi=0.3, t_lo=0.15) == 4 and h(0.2, 3, t_hi=0.3, t_lo=0.15) == 2
    with pytest.raises(ValueError):
        h(-0.2, 3)


def test_average_rate_and_stopping_rule_validation():
    r = srj.average_convergence_rate
    assert r(1.0, math.exp(-1.0), 1) == pytest.approx(1.0)
    assert r(1.0, 1.0, 7) == 0.0
    for bad in ((0.0, 1.0, 1), (1.0, -1.0, 1), (1.0, 1.0, 0)):
        with pytest.raises(ValueError):
            r(*bad)
    with pytest.raises(ValueError):
        srj.StoppingRule("relative_l2", 0.0, 10)
    with pytest.raises(ValueError):
        srj.StoppingRule("relative_l2", 1e-8, 0)


def test_splitmix_streams():
    for seed in (0, 1, 2**64 - 1):
        g = SplitMix64(seed)
        seq = np.array(g.uniforms(1000))
        assert np.array_equal(seq, uniforms_counter(seed, 1000))
        assert np.array_equal(uniforms_counter(seed, 10, start=990), seq[990:])
    assert np.array_equal(uniform_rhs(5, 100), 2.0 * uniforms_counter(5, 100) - 1.0)
    assert derive_seed(1, 2) != derive_seed(1, 3)


@pytest.mark.parametrize("family,shape", [("1d3", (7,)), ("2d5", (5, 4)), ("3d7", (3, 4, 5))])
def test_stencil_operator_csr_matches_reference_layout(family, shape):
    import scipy.sparse
    A = srj.StencilOperator(family, shape)
    csr = A.scipy_csr()
    n = A.n
    assert csr.shape == (n, n)
    dense = csr.toarray()
    assert np.array_equal(dense, dense.T)
    dx2 = (shape[0] + 1.0) ** 2
    d = {"1d3": 2.0, "2d5": 4.0, "3d7": 6.0}[family]
    assert np.all(np.diag(dense) == d * dx2)
    assert np.all(A.inv_diag == 1.0 / (d * dx2))
    off = dense - np.diag(np.diag(dense))
    assert set(np.unique(off)) <= {0.0, -dx2}
    if family == "3d7":
        import sys
        sys.path.insert(0, "/root/reference/pkg/src")
        try:
            from srj.problems import poisson_3d
        except ImportError:
            return
        nn = shape[0]
        if shape == (nn, nn, nn):
            ref = poisson_3d(nn).A.scipy_csr()
            assert (abs(ref - scipy.sparse.csr_matrix(dense)) > 0).nnz == 0


def test_poisson_3d_operator_equals_reference_csr():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from srj.problems import poisson_1d as ref1
        from srj.problems import poisson_3d as ref3
    except ImportError:
        pytest.skip("reference not mounted")
    for ours, ref in ((srj.poisson_3d(5), ref3(5)), (srj.poisson_1d(9), ref1(9))):
        a = ours.A.scipy_csr().toarray()
        b = ref.A.scipy_csr().toarray()
        assert np.array_equal(a, b)
        assert np.array_equal(ours.A.inv_diag, ref.A.inv_diag)
        assert np.array_equal(ours.b, ref.b) and ours.stopping_norm == ref.stopping_norm
        assert ours.cjm_bounds == pytest.approx(ref.cjm_bounds)


def test_varcoef_definition_is_deterministic_and_symmetric():
    from paper_2011_06636_b200.problems import gaussian_field, harmonic_faces
    g1, g2 = gaussian_field(16, 3), gaussian_field(16, 3)
    assert np.array_equal(g1, g2) and g1.shape == (18, 18)
    assert 0.3 < np.std(gaussian_field(64, 0)) < 3.0  # unit-variance field, smoothed
    fx, fy = harmonic_faces(np.exp(g1), 17.0 ** 2)
    assert fx.shape == (16, 17) and fy.shape == (17, 16) and np.all(fx > 0) and np.all(fy > 0)
    p = srj.diffusion_2d_varcoef(16, seed=3)
    dense = p.A.scipy_csr().toarray()
    assert np.array_equal(dense, dense.T)
    assert np.all(np.linalg.eigvalsh(dense) > 0)


def test_problem_instance_validation():
    A = srj.StencilOperator("1d3", (4,))
    with pytest.raises(ValueError):
        srj.ProblemInstance(A=A, b=np.ones(3), x0=np.zeros(4), stopping_norm="absolute_l2")
    with pytest.raises(ValueError):
        srj.ProblemInstance(A=A, b=np.ones(4), x0=np.zeros(4), stopping_norm="absolute_l2",
                            cjm_bounds=(0.5, 0.2))
    with pytest.raises(ValueError):
        srj.poisson_1d(0)
    with pytest.raises(ValueError):
        srj.StencilOperator("3d7", (4, 4))


def test_device_path_refuses_non_stencil_operators():
    import types
    p = srj.poisson_1d(4)
    csr_like = types.SimpleNamespace(A=types.SimpleNamespace(n=4), b=np.ones(4), x0=np.zeros(4))
    with pytest.raises(TypeError):
        srj.solve(csr_like, srj.Heuristic(), srj.StoppingRule("absolute_l2", 1e-6, 10))
    with pytest.raises(ValueError):
        srj.solve(p, srj.Heuristic(), srj.StoppingRule("max_norm", 1e-6, 10))


def test_sparse_matrix_contract_matches_reference():
    # constructor semantics of reference sparse.py:20-44 (no device needed)
    A = srj.SparseMatrix.from_coo(3, [0, 0, 1, 1, 2, 2, 0], [0, 1, 0, 1, 2, 1, 0],
                                  [1.0, -1.0, -1.0, 4.0, 2.0, 0.0, 1.0])
    assert A.n == 3 and A.nnz == 6
    assert list(A.row_ptr) == [0, 2, 4, 6]
    assert np.array_equal(A.diag, [2.0, 4.0, 2.0])  # duplicate (0,0) entries summed
    assert np.array_equal(A.inv_diag, 1.0 / np.array([2.0, 4.0, 2.0]))
    with pytest.raises(ValueError, match="square"):
        srj.SparseMatrix(np.ones((2, 3)))
    with pytest.raises(ValueError, match="symmetric"):
        srj.SparseMatrix.from_dense([[2.0, 1.0], [0.0, 2.0]])
    with pytest.raises(ValueError, match="diagonal"):
        srj.SparseMatrix.from_dense([[0.0, 1.0], [1.0, 2.0]])


def test_csr_generators_match_reference():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from srj.problems import laplace_2d_neumann, random_tridiagonal
    except ImportError:
        pytest.skip("reference not mounted")
    for ours, ref in ((srj.random_tridiagonal(9, 42), random_tridiagonal(9, 42)),
                      (srj.laplace_2d_neumann(6, 3), laplace_2d_neumann(6, 3))):
        a, b = ours.A.scipy_csr(), ref.A.scipy_csr()
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data)
        assert np.array_equal(ours.A.inv_diag, ref.A.inv_diag)
        assert np.array_equal(ours.b, ref.b) and np.array_equal(ours.x0, ref.x0)
        assert ours.stopping_norm == ref.stopping_norm and ours.cjm_bounds == ref.cjm_bounds
