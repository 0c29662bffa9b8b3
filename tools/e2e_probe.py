"""Break down the e2e (host-buffer) C2 solve into staging, solve and readback.

    python tools/e2e_probe.py [--size 2048]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_06636_b200 as srj  # noqa: E402
from paper_2011_06636_b200.solver import solve_fields, _like  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=2048)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    prob = srj.baseline_problem("2d5", args.size, seed=0, device=dev, rhs_on_device=True)
    A = prob.A
    b_host = torch.empty(A.n, dtype=torch.float64, pin_memory=True)
    b_host.copy_(torch.as_tensor(prob.b))
    x0_host = torch.zeros(A.n, dtype=torch.float64, pin_memory=True)
    rule = srj.StoppingRule("relative_l2", 1e-8, 10**9)
    ctrl = srj.Heuristic()
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b = A.field(b_host)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x = A.field(x0_host)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rep = solve_fields(A, b, x, A.new_field(), ctrl, rule, record_history=False)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        out = _like(x0_host, rep.x)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        print(f"iter {it}: field(b) {1e3*(t1-t0):.2f} ms  field(x0) {1e3*(t2-t1):.2f} ms  "
              f"solve {1e3*(t3-t2):.2f} ms  readback {1e3*(t4-t3):.2f} ms  "
              f"cycles {len(rep.cycles)} sweeps {rep.total_iterations}", flush=True)
        del out


if __name__ == "__main__":
    main()
