"""Shared parity helpers: golden fixtures and trace comparison.

The fixtures in tests/golden/ were produced by running the reference itself
(tests/golden/make_golden.py).  Comparison rules (SURVEY §8a parity contract):
  - scheme levels, M, executed counts, cycle count, total sweeps: exact;
  - converged flag: exact;
  - iterate x: bit-identical (sha256 of the float64 bytes) -- the north star
    only asks for <= 1e-10 relative L2, which is also asserted;
  - residual norms: relative 1e-12 (only the summation order of sum r^2
    differs from OpenBLAS ddot).
"""

from __future__ import annotations

import hashlib
import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
RES_RTOL = 1e-12
X_REL_L2 = 1e-10

_cache = {}


def traces():
    if "traces" not in _cache:
        with open(os.path.join(GOLDEN, "traces.json")) as fh:
            _cache["traces"] = json.load(fh)
    return _cache["traces"]


def case(name):
    for c in traces()["cases"]:
        if c["name"] == name:
            return c
    raise KeyError(name)


def cases(filter_fn=None):
    return [c for c in traces()["cases"] if filter_fn is None or filter_fn(c)]


def schemes_npz():
    if "schemes" not in _cache:
        _cache["schemes"] = dict(np.load(os.path.join(GOLDEN, "schemes.npz")))
    return _cache["schemes"]


def sha(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


DIMS = {"1d3": 1, "1d3var": 1, "2d5": 2, "2d5var": 2, "3d7": 3, "3d7var": 3}


def case_faces(c) -> dict:
    """Face arrays of a variable-coefficient golden case (product-independent
    recipes: problems.gaussian_field* / harmonic_faces*), checked against the
    sha256 the golden script recorded; {} for constant coefficients."""
    import sys
    root = os.path.dirname(HERE)
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_2011_06636_b200 import problems as pr
    fam, n, seed = c["family"], c["n"], c.get("seed", 0)
    key = (fam, n, seed)
    if key in _cache:
        return _cache[key]
    dx2 = (n + 1.0) ** 2
    if fam == "2d5var":
        fx, fy = pr.harmonic_faces(np.exp(pr.gaussian_field(n, seed)), dx2)
        faces = {"face_x": fx, "face_y": fy}
    elif fam == "3d7var":
        fx, fy, fz = pr.harmonic_faces_3d(np.exp(pr.gaussian_field_3d(n, seed)), dx2)
        faces = {"face_x": fx, "face_y": fy, "face_z": fz}
    elif fam == "1d3var":
        faces = {"face_x": pr.harmonic_faces_1d(np.exp(pr.gaussian_field_1d(n, seed)), dx2)}
    else:
        faces = {}
    for k, v in faces.items():
        assert sha(v) == c[f"{k}_sha256"], (c["name"], k)
    _cache[key] = faces
    return faces


def case_inputs(c):
    """(family, n, b, face_x, face_y) for a golden case, built from the
    product-independent recipes (SplitMix64 rhs; config-4 faces).  3D
    variable coefficient: face_z from `case_faces`."""
    import sys
    root = os.path.dirname(HERE)
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_2011_06636_b200.rng import uniform_rhs

    fam, n = c["family"], c["n"]
    N = n ** DIMS[fam]
    b = np.ones(N) if c.get("rhs", "uniform") == "ones" else uniform_rhs(c.get("seed", 0), N)
    faces = case_faces(c)
    return fam, n, b, faces.get("face_x"), faces.get("face_y")


def case_operator(c, device=None):
    """The product's StencilOperator of a structured golden case."""
    import sys
    root = os.path.dirname(HERE)
    if root not in sys.path:
        sys.path.insert(0, root)
    from paper_2011_06636_b200.operators import StencilOperator
    fam, n = c["family"], c["n"]
    return StencilOperator(fam, (n,) * DIMS[fam], device=device, **case_faces(c))


def is_csr(c) -> bool:
    return c["family"].startswith("csr:")


def csr_inputs(c):
    """(scipy CSR, b, x0) of a general-CSR golden case: the product's
    generators (equal to the reference's, tests/test_host.py) or the committed
    FEM fixture written by make_golden.py."""
    import sys
    root = os.path.dirname(HERE)
    if root not in sys.path:
        sys.path.insert(0, root)
    import scipy.sparse

    import paper_2011_06636_b200 as srj
    fam = c["family"]
    if fam == "csr:laplace2d":
        p = srj.laplace_2d_neumann(c["n"], c["seed"])
    elif fam == "csr:tridiag":
        p = srj.random_tridiagonal(c["n"], c["seed"])
    elif fam == "csr:mesh":
        z = np.load(os.path.join(GOLDEN, c["fixture"]))
        n = len(z["b"])
        csr = scipy.sparse.csr_matrix((z["data"], z["indices"], z["indptr"]), shape=(n, n))
        return csr, z["b"], z["x0"]
    elif fam == "csr:dense1":
        return scipy.sparse.csr_matrix(np.array([[4.0]])), np.array([8.0]), np.array([0.0])
    else:
        raise KeyError(fam)
    return p.A.scipy_csr(), np.asarray(p.b), np.asarray(p.x0)


def golden_cycle_rows(c):
    """Per-cycle (cycle, level, M, executed) ints and the rows with residuals."""
    cyc = c["cycles"]
    if isinstance(cyc, dict):
        ints = [tuple(r) for r in cyc["ints"]]
        full = {r[0]: r[1:] for r in cyc["sampled"]}
        return ints, full
    ints = [tuple(r[:4]) for r in cyc]
    return ints, {k: r for k, r in enumerate(cyc)}


def assert_trace_matches(c, got_rows, total, converged, x=None, history=None):
    """got_rows: list of (cycle, level, M, executed, res_before, res_after, rate)."""
    ints, full = golden_cycle_rows(c)
    got_ints = [tuple(int(v) for v in r[:4]) for r in got_rows]
    assert len(got_ints) == len(ints), f"{c['name']}: {len(got_ints)} cycles vs {len(ints)}"
    if got_ints != ints:
        k = next(i for i, (a, b) in enumerate(zip(got_ints, ints)) if a != b)
        raise AssertionError(f"{c['name']}: cycle {k} differs: got {got_ints[k]} want {ints[k]}")
    assert total == c["total_iterations"], (c["name"], total, c["total_iterations"])
    assert converged == c["converged"], c["name"]
    for k, want in full.items():
        got = got_rows[k]
        for idx in (4, 5):
            assert math.isclose(got[idx], want[idx], rel_tol=RES_RTOL, abs_tol=0.0), \
                (c["name"], k, idx, got[idx], want[idx])
        if math.isfinite(want[6]) and want[6] != 0.0:
            # rate = -log(ratio)/executed amplifies the 1e-15 norm noise
            assert math.isclose(got[6], want[6], rel_tol=1e-8, abs_tol=1e-12), (c["name"], k)
    if x is not None:
        x = np.asarray(x, dtype=np.float64)
        if "x" in c:
            ref = np.asarray(c["x"])
            denom = max(np.linalg.norm(ref), 1e-300)
            assert np.linalg.norm(x - ref) / denom <= X_REL_L2, c["name"]
        assert sha(x) == c["x_sha256"], f"{c['name']}: iterate not bit-identical"
    if history is not None and "history" in c:
        want = c["history"]
        assert len(history) == len(want), c["name"]
        for (i1, r1), (i2, r2) in zip(history, want):
            assert i1 == i2
            assert math.isclose(r1, r2, rel_tol=RES_RTOL), (c["name"], i1, r1, r2)
