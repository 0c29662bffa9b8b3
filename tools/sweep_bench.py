"""Per-sweep timing of the cycle kernel at fixed scheme level (no early stop).

python tools/sweep_bench.py 2d5:512,2d5:2048,3d7:256 --level 20 --spp 1
Prints one JSON line per case: us/sweep, algorithmic GB/s, GLUP/s.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases")
    ap.add_argument("--level", type=int, default=20)
    ap.add_argument("--spp", type=int, default=0, help="sweeps per pass (0: operator default)")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.solver import _OMEGAS
    dev = torch.device("cuda", 0)
    bpu = {"1d3": 24, "2d5": 24, "3d7": 24, "2d5var": 40, "3d7var": 48, "1d3var": 32}
    for spec in a.cases.split(","):
        fam, n = spec.split(":")
        n = int(n)
        if fam in ("csr2d", "csr3d"):
            # the generic CSR kernel on a stencil matrix (bytes: x, b, x' + the
            # CSR row -- 8 B value + 4 B column per entry, 8 B row pointer -- and
            # 8 B inv_diag)
            st = srj.StencilOperator("2d5" if fam == "csr2d" else "3d7",
                                     (n, n) if fam == "csr2d" else (n, n, n))
            A = srj.SparseMatrix(st.scipy_csr(), device=dev)
            bpu[fam] = 24 + 12 * A.nnz / A.n + 16
            p = srj.ProblemInstance(A=A, b=srj.uniform_rhs(0, A.n), x0=np.zeros(A.n),
                                    stopping_norm="relative_l2")
        else:
            p = srj.baseline_problem(fam, n, seed=0, device=dev,
                                     rhs_on_device=(fam in ("1d3", "2d5", "3d7")))
        A = p.A
        if a.spp > 0:
            A.set_sweeps_per_pass(a.spp)
        b = A.field(p.b)
        x = A.new_field()
        xa = A.new_field()
        sch = srj.scheme_for_level(a.level)
        om = _OMEGAS.get(sch, dev)
        S = A.residual_sq(x, b)
        base = S ** 0.5
        times = []
        for r in range(a.reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            out = A.run_cycle(x, xa, b, om, sch.M, -1.0, base, 1.0, sch.M, None)
            e1.record()
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
            assert out.executed == sch.M or os.environ.get('SRJ_BENCH_NOASSERT'), out.executed
        ms = min(times)
        us = ms * 1e3 / out.executed
        print(json.dumps({"case": spec, "M": sch.M, "spp": a.spp, "us_per_sweep": us,
                          "GBps_alg": bpu[fam] * A.n / (us * 1e-6) / 1e9,
                          "GLUPs": A.n / (us * 1e-6) / 1e9, "launches": out.launches, "info": A.describe()}),
              flush=True)


if __name__ == "__main__":
    main()
