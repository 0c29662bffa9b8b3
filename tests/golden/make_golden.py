"""Generate the parity fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

Writes tests/golden/traces.json and tests/golden/schemes.npz.  Every number in
them comes from the unmodified reference package (/root/reference/pkg/src/srj)
solving the listed inputs through its public API (`solve`, `run_cycle`,
`scheme_for_level`); nothing is written by hand.  The inputs are built with the
reference's own generators where they exist (poisson_1d, poisson_3d) and with
`SparseMatrix.from_coo` for the 2D Dirichlet and variable-coefficient stencils
the reference has no generator for (their face arrays come from the product's
deterministic config-4 definition, `problems.gaussian_field`/`harmonic_faces`).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import srj  # noqa: E402  (the reference)
from srj.problems import ProblemInstance  # noqa: E402
from srj.sparse import SparseMatrix  # noqa: E402

from paper_2011_06636_b200.problems import (gaussian_field, gaussian_field_1d,  # noqa: E402
                                            gaussian_field_3d, harmonic_faces,
                                            harmonic_faces_1d, harmonic_faces_3d)
from paper_2011_06636_b200.rng import uniform_rhs  # noqa: E402

MAX_X_STORE = 4096
MAX_FULL_CYCLES = 2000   # longer traces keep every int column, residuals sampled


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def poisson_2d_ref(n: int) -> SparseMatrix:
    dx2 = (n + 1.0) ** 2
    ids = np.arange(n * n).reshape(n, n)
    rows, cols, vals = [ids.ravel()], [ids.ravel()], [np.full(n * n, 4.0 * dx2)]
    for a, b in ((ids[:, :-1], ids[:, 1:]), (ids[:-1, :], ids[1:, :])):
        rows += [a.ravel(), b.ravel()]
        cols += [b.ravel(), a.ravel()]
        vals += [np.full(a.size, -dx2)] * 2
    return SparseMatrix.from_coo(n * n, np.concatenate(rows), np.concatenate(cols),
                                 np.concatenate(vals))


def varcoef_2d_ref(n: int, seed: int):
    dx2 = (n + 1.0) ** 2
    fx, fy = harmonic_faces(np.exp(gaussian_field(n, seed)), dx2)
    ids = np.arange(n * n).reshape(n, n)
    diag = (((fx[:, :-1] + fx[:, 1:]) + fy[:-1, :]) + fy[1:, :]).ravel()
    rows, cols, vals = [ids.ravel()], [ids.ravel()], [diag]
    ix = -fx[:, 1:-1]
    iy = -fy[1:-1, :]
    for (a, b), v in (((ids[:, :-1], ids[:, 1:]), ix), ((ids[:-1, :], ids[1:, :]), iy)):
        rows += [a.ravel(), b.ravel()]
        cols += [b.ravel(), a.ravel()]
        vals += [v.ravel()] * 2
    A = SparseMatrix.from_coo(n * n, np.concatenate(rows), np.concatenate(cols),
                              np.concatenate(vals))
    return A, sha(fx), sha(fy)


def varcoef_3d_ref(n: int, seed: int):
    """3D 7-point variable-coefficient CSR for the reference: off-diagonals
    -face, diagonal (((((c_w + c_e) + c_s) + c_n) + c_b) + c_t) (srj.h)."""
    dx2 = (n + 1.0) ** 2
    fx, fy, fz = harmonic_faces_3d(np.exp(gaussian_field_3d(n, seed)), dx2)
    ids = np.arange(n ** 3).reshape(n, n, n)
    diag = (((((fx[:, :, :-1] + fx[:, :, 1:]) + fy[:, :-1, :]) + fy[:, 1:, :]) + fz[:-1])
            + fz[1:]).ravel()
    rows, cols, vals = [ids.ravel()], [ids.ravel()], [diag]
    for (a, b), v in (((ids[:, :, :-1], ids[:, :, 1:]), -fx[:, :, 1:-1]),
                      ((ids[:, :-1, :], ids[:, 1:, :]), -fy[:, 1:-1, :]),
                      ((ids[:-1], ids[1:]), -fz[1:-1])):
        rows += [a.ravel(), b.ravel()]
        cols += [b.ravel(), a.ravel()]
        vals += [v.ravel()] * 2
    A = SparseMatrix.from_coo(n ** 3, np.concatenate(rows), np.concatenate(cols),
                              np.concatenate(vals))
    return A, {"face_x_sha256": sha(fx), "face_y_sha256": sha(fy), "face_z_sha256": sha(fz)}


def varcoef_1d_ref(n: int, seed: int):
    dx2 = (n + 1.0) ** 2
    fx = harmonic_faces_1d(np.exp(gaussian_field_1d(n, seed)), dx2)
    ids = np.arange(n)
    rows = [ids, ids[:-1], ids[1:]]
    cols = [ids, ids[1:], ids[:-1]]
    vals = [fx[:-1] + fx[1:], -fx[1:-1], -fx[1:-1]]
    A = SparseMatrix.from_coo(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    return A, {"face_x_sha256": sha(fx)}


def build_csr(case):
    """General-CSR problems (§8 f2/f3) through the reference's own generators."""
    fam = case["family"]
    if fam == "csr:laplace2d":
        p = srj.laplace_2d_neumann(case["n"], case["seed"])
        return p, {}
    if fam == "csr:tridiag":
        return srj.random_tridiagonal(case["n"], case["seed"]), {}
    if fam == "csr:mesh":
        from srj.problems import assemble_fem_poisson, read_mesh
        p = assemble_fem_poisson(read_mesh(os.path.join("/root/reference/pkg/assets",
                                                        case["mesh"] + ".mesh")))
        csr = p.A.scipy_csr()
        path = os.path.join(HERE, f"fem_{case['mesh']}.npz")
        np.savez_compressed(path, indptr=csr.indptr, indices=csr.indices, data=csr.data,
                            b=p.b, x0=p.x0)
        return p, {"fixture": os.path.basename(path), "n": p.A.n}
    if fam == "csr:dense1":
        A = SparseMatrix.from_dense([[4.0]])
        return ProblemInstance(A=A, b=np.array([8.0]), x0=np.array([0.0]),
                               stopping_norm=case["norm"]), {}
    raise ValueError(fam)


def build(case):
    if case["family"].startswith("csr:"):
        return build_csr(case)
    fam, n, seed, rhs = case["family"], case["n"], case.get("seed", 0), case.get("rhs", "uniform")
    extra = {}
    if fam == "1d3":
        p = srj.poisson_1d(n)
        A = p.A
    elif fam == "3d7":
        p = srj.poisson_3d(n)
        A = p.A
    elif fam == "2d5":
        A = poisson_2d_ref(n)
    elif fam == "3d7var":
        A, extra = varcoef_3d_ref(n, seed)
    elif fam == "1d3var":
        A, extra = varcoef_1d_ref(n, seed)
    else:
        A, hx, hy = varcoef_2d_ref(n, seed)
        extra = {"face_x_sha256": hx, "face_y_sha256": hy}
    N = A.n
    b = np.ones(N) if rhs == "ones" else uniform_rhs(seed, N)
    return ProblemInstance(A=A, b=b, x0=np.zeros(N), stopping_norm=case["norm"]), extra


def controller_of(case):
    c = case["controller"]
    if c == "heuristic":
        return srj.Heuristic()
    if c == "increasing":
        return srj.Increasing()
    if c == "jacobi":
        return srj.Jacobi()
    if c.startswith("fixed:"):
        return srj.FixedM(int(c.split(":")[1]))
    if c.startswith("cjm:"):
        M = int(c.split(":")[1])
        return ("cjm", M)
    if c == "blowup":
        return srj.Cjm(srj.SrjScheme(M=2, omegas=(1e200, 1.0), application_order=(0, 1)))
    raise ValueError(c)


def cycles_record(cycles):
    rows = [[c.cycle, c.level, c.M, c.executed, c.residual_before, c.residual_after,
             c.average_rate] for c in cycles]
    if len(rows) <= MAX_FULL_CYCLES:
        return rows
    keep = set(range(0, len(rows), 97)) | set(range(len(rows) - 10, len(rows)))
    return {"count": len(rows),
            "ints": [[r[0], r[1], r[2], r[3]] for r in rows],
            "sampled": [[k] + rows[k] for k in sorted(keep)]}


def run_case(case):
    p, extra = build(case)
    ctrl = controller_of(case)
    if isinstance(ctrl, tuple):
        lo, hi = srj.poisson_1d(case["n"]).cjm_bounds
        ctrl = srj.Cjm(srj.generate_cjm_scheme(ctrl[1], lo, hi))
    rule = srj.StoppingRule(norm=case["norm"], tolerance=case["tol"],
                            max_iterations=case.get("max_iterations", 10**9))
    rec = dict(case)
    rec.update(extra)
    try:
        rep = srj.solve(p, ctrl, rule, record_history=True)
    except srj.SolveDivergedError as exc:
        rec["diverged"] = exc.diagnostics
        return rec
    rec.update({
        "converged": rep.converged,
        "total_iterations": rep.total_iterations,
        "cycles": cycles_record(rep.cycles),
        "x_sha256": sha(rep.x),
        "x_norm2": float(np.linalg.norm(rep.x)),
    })
    if p.A.n <= MAX_X_STORE:
        rec["x"] = [float(v) for v in rep.x]
    if case.get("history", False):
        rec["history"] = [[int(i), float(r)] for i, r in rep.residual_history]
    return rec


def run_cycle_cases():
    """Direct run_cycle snapshots (reference solver.py:177-273 semantics)."""
    out = []
    p = srj.poisson_1d(50)
    st = srj.SolverState(x=p.x0.copy())
    rule = srj.StoppingRule(norm="absolute_l2", tolerance=1e-30, max_iterations=3)
    s1, c1 = srj.run_cycle(p.A, p.b, st, srj.scheme_for_level(3), stopping=rule)
    out.append({"name": "budget3_level3_n50", "N": 50, "level": 3, "executed": c1.executed,
                "converged": s1.converged, "x": [float(v) for v in s1.x],
                "res_after": c1.residual_after})
    p = srj.poisson_1d(30)
    s2, c2 = srj.run_cycle(p.A, p.b, srj.SolverState(x=p.x0.copy()), srj.scheme_for_level(5))
    s3, c3 = srj.run_cycle(p.A, p.b, s2, srj.scheme_for_level(6))
    out.append({"name": "chain_level5_level6_n30", "N": 30, "levels": [5, 6],
                "executed": [c2.executed, c3.executed],
                "res": [[c2.residual_before, c2.residual_after],
                        [c3.residual_before, c3.residual_after]],
                "x": [float(v) for v in s3.x],
                "history": [[int(i), float(r)] for i, r in s3.residual_history]})
    return out


CASES = [
    # reference golden CSV recipes (pkg/results/*.csv, cli.py defaults: b = 1)
    {"name": "poisson1d_100_heuristic", "family": "1d3", "n": 100, "rhs": "ones",
     "norm": "absolute_l2", "tol": 1e-7, "controller": "heuristic", "max_iterations": 60000,
     "history": True},
    {"name": "poisson1d_100_increasing", "family": "1d3", "n": 100, "rhs": "ones",
     "norm": "absolute_l2", "tol": 1e-7, "controller": "increasing", "max_iterations": 60000},
    {"name": "poisson1d_100_cjm63", "family": "1d3", "n": 100, "rhs": "ones",
     "norm": "absolute_l2", "tol": 1e-7, "controller": "cjm:63", "max_iterations": 60000},
    {"name": "poisson1d_100_jacobi", "family": "1d3", "n": 100, "rhs": "ones",
     "norm": "absolute_l2", "tol": 1e-7, "controller": "jacobi", "max_iterations": 60000},
    {"name": "poisson3d_16_ones", "family": "3d7", "n": 16, "rhs": "ones",
     "norm": "relative_l2", "tol": 1e-8, "controller": "heuristic"},
    {"name": "poisson3d_24_ones", "family": "3d7", "n": 24, "rhs": "ones",
     "norm": "relative_l2", "tol": 1e-8, "controller": "heuristic"},
    {"name": "poisson3d_32_ones", "family": "3d7", "n": 32, "rhs": "ones",
     "norm": "relative_l2", "tol": 1e-8, "controller": "heuristic"},
    # BASELINE config 1 exactly, plus reduced 2D/3D/var-coef versions of configs 2-5
    {"name": "c1_seed0", "family": "1d3", "n": 1024, "seed": 0, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic", "history": True},
    {"name": "c1_seed1", "family": "1d3", "n": 1024, "seed": 1, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    {"name": "c1_seed42", "family": "1d3", "n": 1024, "seed": 42, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    {"name": "c2_32", "family": "2d5", "n": 32, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic", "history": True},
    {"name": "c2_37", "family": "2d5", "n": 37, "seed": 3, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c2_64", "family": "2d5", "n": 64, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c2_128", "family": "2d5", "n": 128, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c2_256", "family": "2d5", "n": 256, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c3_16", "family": "3d7", "n": 16, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic", "history": True},
    {"name": "c3_19", "family": "3d7", "n": 19, "seed": 5, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c3_32", "family": "3d7", "n": 32, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c3_48", "family": "3d7", "n": 48, "seed": 0, "norm": "relative_l2", "tol": 1e-8,
     "controller": "heuristic"},
    {"name": "c4_32", "family": "2d5var", "n": 32, "seed": 0, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic", "history": True},
    {"name": "c4_64", "family": "2d5var", "n": 64, "seed": 0, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    {"name": "c4_128", "family": "2d5var", "n": 128, "seed": 7, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    # edge cases the reference tests exercise (test_solver.py)
    {"name": "tiny_1d_n1", "family": "1d3", "n": 1, "rhs": "ones", "norm": "absolute_l2",
     "tol": 1e-12, "controller": "heuristic"},
    {"name": "tiny_2d_n2", "family": "2d5", "n": 2, "seed": 0, "norm": "relative_l2",
     "tol": 1e-10, "controller": "heuristic"},
    {"name": "tiny_3d_n2", "family": "3d7", "n": 2, "seed": 0, "norm": "relative_l2",
     "tol": 1e-10, "controller": "heuristic"},
    {"name": "budget_jacobi_50", "family": "1d3", "n": 100, "rhs": "ones",
     "norm": "absolute_l2", "tol": 1e-7, "controller": "jacobi", "max_iterations": 50},
    {"name": "budget_midcycle_2d", "family": "2d5", "n": 40, "seed": 2, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic", "max_iterations": 200},
    {"name": "fixed5_tol_tiny", "family": "1d3", "n": 24, "rhs": "ones", "norm": "absolute_l2",
     "tol": 1e-300, "controller": "fixed:5", "max_iterations": 70},
    {"name": "increasing_clamp", "family": "1d3", "n": 4, "rhs": "ones", "norm": "absolute_l2",
     "tol": 1e-300, "controller": "increasing", "max_iterations": 40},
    {"name": "fixed2362_3d", "family": "3d7", "n": 20, "seed": 9, "norm": "relative_l2",
     "tol": 1e-9, "controller": "fixed:2362"},
    {"name": "blowup_diverges", "family": "1d3", "n": 100, "rhs": "ones",
     "norm": "absolute_l2", "tol": 1e-7, "controller": "blowup"},
    # general CSR operators (§8 f3) and the solution-difference norm (§8 f2)
    {"name": "laplace2d_64_seed1", "family": "csr:laplace2d", "n": 64, "seed": 1,
     "norm": "solution_diff_inf", "tol": 1e-10, "controller": "heuristic", "history": True},
    {"name": "laplace2d_8_seed3", "family": "csr:laplace2d", "n": 8, "seed": 3,
     "norm": "solution_diff_inf", "tol": 1e-8, "controller": "heuristic", "max_iterations": 50000},
    {"name": "laplace2d_16_jacobi_budget", "family": "csr:laplace2d", "n": 16, "seed": 2,
     "norm": "solution_diff_inf", "tol": 1e-12, "controller": "jacobi", "max_iterations": 300},
    {"name": "tridiag_500_seed0", "family": "csr:tridiag", "n": 500, "seed": 0,
     "norm": "absolute_l2", "tol": 1e-7, "controller": "heuristic"},
    {"name": "tridiag_200_seed1_increasing", "family": "csr:tridiag", "n": 200, "seed": 1,
     "norm": "absolute_l2", "tol": 1e-7, "controller": "increasing"},
    {"name": "fem_disk", "family": "csr:mesh", "mesh": "disk", "n": 0,
     "norm": "absolute_l2", "tol": 1e-9, "controller": "heuristic"},
    {"name": "fem_airfoil_med", "family": "csr:mesh", "mesh": "airfoil_med", "n": 0,
     "norm": "absolute_l2", "tol": 1e-9, "controller": "heuristic"},
    {"name": "dense_1x1", "family": "csr:dense1", "n": 1, "norm": "absolute_l2", "tol": 1e-12,
     "controller": "jacobi"},
]


# north_star's 1D / 3D variable-coefficient stencils (round 2): merged into
# traces.json by `make_golden.py --var` without re-running the cases above
VAR_CASES = [
    {"name": "c3v_12", "family": "3d7var", "n": 12, "seed": 0, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic", "history": True},
    {"name": "c3v_20", "family": "3d7var", "n": 20, "seed": 3, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    {"name": "c3v_31", "family": "3d7var", "n": 31, "seed": 1, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    {"name": "c3v_32", "family": "3d7var", "n": 32, "seed": 0, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
    {"name": "c3v_24_budget", "family": "3d7var", "n": 24, "seed": 4, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic", "max_iterations": 150},
    {"name": "c1v_1024", "family": "1d3var", "n": 1024, "seed": 0, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic", "history": True},
    {"name": "c1v_100_s2", "family": "1d3var", "n": 100, "seed": 2, "norm": "relative_l2",
     "tol": 1e-8, "controller": "heuristic"},
]


def datacollect_cases():
    """Reference data collection (datacollect.py:79-147) and the threshold fit."""
    from srj import datacollect as dc

    def pack(points):
        return {"ints": [[p.trial, p.step, dc.ACTIONS.index(p.action), p.level] for p in points],
                "reals": [[p.avg_rate, p.prev_ratio, p.res_before, p.res_after] for p in points]}

    out = {
        "collect_10_t2_s5": pack(dc.collect([10], 2, target_tol=1e-8, seed=5)),
        "collect_5_30_t2_s7": pack(dc.collect([5, 30], 2, target_tol=1e-8, seed=7)),
        "until_5_10_200_s2": pack(dc.collect_until([5, 10], 200, target_tol=1e-6, seed=2)),
    }
    pts = dc.collect_until([10, 50], 40000, seed=3)
    clusters = dc.aggregate(pts, n_set=1000)
    t_hi, t_lo = dc.fit_thresholds(clusters)
    out["fit_10_50_40000_s3"] = {
        "count": len(pts), "t_hi": t_hi, "t_lo": t_lo,
        "clusters": [[c.level_bucket, c.mean_ratio, c.best_action] for c in clusters]}
    return out


def main_var():
    path = os.path.join(HERE, "traces.json")
    with open(path) as fh:
        traces = json.load(fh)
    names = {c["name"] for c in VAR_CASES}
    traces["cases"] = [c for c in traces["cases"] if c["name"] not in names]
    for case in VAR_CASES:
        print("running", case["name"], flush=True)
        traces["cases"].append(run_case(case))
    with open(path, "w") as fh:
        json.dump(traces, fh, separators=(",", ":"))
    print("merged", len(VAR_CASES), "cases into", path)


def main():
    traces = {"reference": "/root/reference (srj 0.1.0)", "numpy": np.__version__,
              "cases": [], "run_cycle": run_cycle_cases(), "datacollect": datacollect_cases()}
    for case in CASES:
        print("running", case["name"], flush=True)
        traces["cases"].append(run_case(case))
    with open(os.path.join(HERE, "traces.json"), "w") as fh:
        json.dump(traces, fh, separators=(",", ":"))
    arrays = {}
    for level in range(len(srj.LEVEL_TABLE_M)):
        s = srj.scheme_for_level(level)
        arrays[f"omegas_{level}"] = np.array(s.omegas)
        arrays[f"order_{level}"] = np.array(s.application_order, dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, "schemes.npz"), **arrays)
    print("wrote", HERE)


if __name__ == "__main__":
    if "--var" in sys.argv[1:]:
        main_var()
    else:
        main()
