"""Whole-solve fixtures at the BASELINE sizes (tests/golden/fullsize.json).

Run in the build container:

    python tests/golden/make_fullsize.py [c2ref c2 c3 c4 c5 ...]

* ``c2ref`` -- C2 (2D Poisson 2048^2, relative 1e-8) solved by the UNMODIFIED
  reference (/root/reference/pkg/src/srj ``solve`` on its own CSR
  ``SparseMatrix``; ~17 min on one core).  This pins the oracle at full size.
* ``c2``, ``c3``, ``c4`` -- C2 / C3 (3D 512^3) / C4 (2D var-coef 4096^2) whole
  solves to 1e-8 with the pinned OpenMP oracle (oracle/srj_oracle.c, itself
  checked against reference-run traces in tests/test_oracle.py).
* ``c5`` -- one 1024 x 1024 x 128 z-slab of config 5 (the per-GPU load at
  N = 1, dx2 = 1025^2, Dirichlet on all faces), exactly 50 heuristic cycles in
  throughput mode (tol 1e-300), oracle.

Each record holds the per-cycle [level, M, executed, res_before, res_after],
the totals, sha256 of the final iterate (bit-exact), and the smallest
distances of the cycle ratios to the heuristic thresholds 0.4 / 0.2 (SURVEY
§7c: how far the scheme sequence is from flipping on a last-bit residual
difference).  Existing records are kept unless named on the command line.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
OUT = os.path.join(HERE, "fullsize.json")

from oracle import srj_oracle as O  # noqa: E402
from paper_2011_06636_b200.problems import gaussian_field, harmonic_faces  # noqa: E402
from paper_2011_06636_b200.rng import uniform_rhs  # noqa: E402

SPECS = {
    "c2": dict(family="2d5", dims=(2048, 2048, 1), tol=1e-8, max_cycles=None),
    "c3": dict(family="3d7", dims=(512, 512, 512), tol=1e-8, max_cycles=None),
    "c4": dict(family="2d5var", dims=(4096, 4096, 1), tol=1e-8, max_cycles=None),
    "c5": dict(family="3d7", dims=(1024, 1024, 128), tol=1e-300, max_cycles=50),
}


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def margins(rows):
    r = [c[4] / c[3] for c in rows if c[3] > 0 and c[4] > 0]
    return {"min_abs_ratio_minus_0.4": min(abs(v - 0.4) for v in r),
            "min_abs_ratio_minus_0.2": min(abs(v - 0.2) for v in r)}


def record(name, generator, rows, total, converged, x, seconds):
    return {"config": name, "generator": generator, "seed": 0,
            "cycles": rows, "total_iterations": total, "converged": converged,
            "x_sha256": sha(x), "x_norm2": float(np.linalg.norm(x)),
            "margins": margins(rows), "last_res_after": rows[-1][4], "cpu_seconds": round(seconds, 1)}


def run_oracle(name):
    s = SPECS[name]
    nx, ny, nz = s["dims"]
    n = nx * ny * nz
    if s["family"] == "2d5var":
        fx, fy = harmonic_faces(np.exp(gaussian_field(nx, 0)), (nx + 1.0) ** 2)
        op = O.stencil("2d5var", nx, fx=fx, fy=fy)
    else:
        op = O.StencilCPU(s["family"], nx, ny, nz, dx2=(nx + 1.0) ** 2)
    b = uniform_rhs(0, n)
    t0 = time.perf_counter()
    rep = O.Oracle(op, b).solve(np.zeros(n), controller="heuristic", tol=s["tol"],
                                max_cycles=s["max_cycles"], record_history=False)
    rows = [[c.level, c.M, c.executed, c.res_before, c.res_after] for c in rep.cycles]
    return record(name, "oracle/srj_oracle (OpenMP)", rows, rep.total, rep.converged, rep.x,
                  time.perf_counter() - t0)


def run_reference_c2():
    sys.path.insert(0, "/root/reference/pkg/src")
    import srj  # the reference
    from srj.problems import ProblemInstance
    sys.path.insert(0, HERE)
    from make_golden import poisson_2d_ref
    n = 2048
    A = poisson_2d_ref(n)
    p = ProblemInstance(A=A, b=uniform_rhs(0, n * n), x0=np.zeros(n * n),
                        stopping_norm="relative_l2")
    t0 = time.perf_counter()
    rule = srj.StoppingRule(norm="relative_l2", tolerance=1e-8, max_iterations=10**9)
    rep = srj.solve(p, srj.Heuristic(), rule, record_history=False)
    rows = [[c.level, c.M, c.executed, c.residual_before, c.residual_after] for c in rep.cycles]
    return record("c2", "reference srj.solve (CSR, 1 core)", rows, rep.total_iterations,
                  rep.converged, rep.x, time.perf_counter() - t0)


def main(argv):
    names = argv or ["c2", "c3", "c4", "c5", "c2ref"]
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for name in names:
        rec = run_reference_c2() if name == "c2ref" else run_oracle(name)
        key = "c2_reference" if name == "c2ref" else name
        data[key] = rec
        print(key, rec["total_iterations"], len(rec["cycles"]), rec["x_sha256"][:16],
              rec["margins"], rec["cpu_seconds"], "s", flush=True)
        if os.path.exists(OUT):  # merge with records written meanwhile by another run
            with open(OUT) as f:
                cur = json.load(f)
            cur[key] = rec
            data = cur
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
