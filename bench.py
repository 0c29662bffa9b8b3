"""SRJ solve benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
2D Poisson, 5-point stencil, 2048 x 2048 interior, Dirichlet, f ~ U[-1,1) from
SplitMix64(seed), x0 = 0, fp64, learned SRJ scheme selection (Heuristic 0.4/0.2)
until the relative residual <= 1e-8.  One step = one full solve.

  value     GLUP/s = points x sweeps / device time, inputs resident in HBM
  e2e       the same metric through the public API `solve()` with pinned host
            b/x0 in and x out (H2D + D2H inside the timed region)
  roofline  algorithmic bytes of the cycle kernel (24 B per point-sweep + 16 B
            per point for the end-of-cycle residual; 40 B + 32 B var-coef) / its
            event-timed duration vs the measured HBM copy bandwidth
            (MEASURED_PEAKS.json)
  cpu_baseline  the oracle port (oracle/srj_oracle.c, OpenMP) on a bounded
            sample of the same workload on this host's cores

`--impl reference` times the CPU port alone (the reference is pure Python and
cannot travel to the GPU box; its restatement is the oracle, pinned bit-exact
against it in tests/test_oracle.py).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_DESC = {
    "c2": "2D Poisson 5-pt 2048^2 Dirichlet, f~U[-1,1) SplitMix64, rel L2 1e-8, SRJ heuristic",
    "c3": "3D Poisson 7-pt 512^3 Dirichlet, f~U[-1,1) SplitMix64, rel L2 1e-8, SRJ heuristic",
    "c1": "1D Poisson 3-pt N=1024 Dirichlet, f~U[-1,1) SplitMix64, rel L2 1e-8, SRJ heuristic",
    "c4": "2D var-coef 5-pt 4096^2 harmonic faces k=exp(g), rel L2 1e-8, SRJ heuristic",
    "c5": "3D Poisson 7-pt 1024x1024x(128N) z-slabs over N GPUs, 50 heuristic cycles",
    "c3v": "3D var-coef 7-pt 512^3 harmonic faces k=exp(g), rel L2 1e-8, SRJ heuristic",
    "c1v": "1D var-coef 3-pt N=1024 harmonic faces k=exp(g), rel L2 1e-8, SRJ heuristic",
}
# x and b read, x written (+ the face arrays of the variable-coefficient
# families: 2D east/north 2, 3D x/y/z 3, 1D 1; the diagonal is recomputed)
BYTES_PER_UPDATE = {"1d3": 24, "2d5": 24, "3d7": 24, "2d5var": 40, "3d7var": 48, "1d3var": 32}
# end-of-cycle residual pass: reads x and b (+ the face arrays, var-coef)
RESIDUAL_BYTES = {"1d3": 16, "2d5": 16, "3d7": 16, "2d5var": 32, "3d7var": 40, "1d3var": 24}
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2
METRIC = {"default": "GLUP/s (SRJ point-updates/s); time-to-rel-residual 1e-8",
          "c5": "GLUP/s (SRJ point-updates/s), 50 heuristic cycles (throughput mode)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIG_DESC))
    ap.add_argument("--size", type=int, default=None, help="override the grid extent")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--sweeps-per-pass", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--planes-per-gpu", type=int, default=128, help="c5: z planes per GPU")
    ap.add_argument("--cycles", type=int, default=50, help="c5: heuristic cycles per step")
    ap.add_argument("--slabs", action="store_true",
                    help="c3/c4: use the slab solver even on one GPU (it is used for N > 1)")
    ap.add_argument("--host-loop", action="store_true",
                    help="run the controller loop on the host (one launch per cycle) even where "
                         "the device-resident solve exists")
    ap.add_argument("--no-tb-slabs", action="store_true",
                    help="slabs: one sweep per launch instead of temporally blocked passes")
    ap.add_argument("--exchange", default="torch", choices=["torch", "native"],
                    help="slabs at N > 1: deep-halo exchange over torch.distributed P2P, or "
                         "libsrj's own NCCL communicator with one srj_slab_cycle_forward call "
                         "per cycle (no exchange/compute split)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SRJ_BENCH_SHARE_DEVICE=1 (checking only): every rank on cuda:0, so the
    # N > 1 replica path (barriers, max over ranks, rank-0 line) runs on a
    # one-GPU box; replicas never wait on one another.  Never a bench number.
    if os.environ.get("SRJ_BENCH_SHARE_DEVICE") == "1":
        local = 0
    return rank, world, local


def init_dist(dev):
    """One process per GPU over NCCL; SRJ_BENCH_BACKEND=gloo pairs with
    SRJ_BENCH_SHARE_DEVICE for the one-GPU check of the N > 1 path."""
    import torch.distributed as dist
    if os.environ.get("SRJ_BENCH_BACKEND", "nccl") == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(os.environ["SRJ_BENCH_BACKEND"])


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()),
                 default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower() == "active"})
        pw = sorted(float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit())
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_median": pw[len(pw) // 2] if pw else None,
                "power_w_max": pw[-1] if pw else None}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_from_profile(config):
    """DRAM bytes (read + write) of one captured launch of the dominant kernel
    from `ncu --set full` (profiles/traffic.json), with that launch's
    algorithmic bytes for scale; None when no capture exists for the config."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            entry = json.load(fh).get(config)
    except Exception:
        return None
    if not entry:
        return None
    return {"traffic": entry["traffic"], "alg_bytes": entry["alg_bytes"],
            "ratio": entry["traffic_over_alg"], "launch": entry["launch"],
            "limiter": entry.get("limiter")}


def kernel_name(family, info):
    from paper_2011_06636_b200._lib import OpInfo
    return OpInfo.KERNELS.get(info.get("cycle_kernel"), "unknown")


def cpu_sample(family, n, seed, budget_s):
    """Bounded CPU sample: SRJ sweeps (update + residual + norm, the reference's
    per-sweep work) with the OpenMP oracle port on this host's cores."""
    import numpy as np

    from oracle import srj_oracle as O
    # every host thread this process may run on (torchrun sets OMP_NUM_THREADS=1)
    O.clib().oracle_set_threads(len(os.sched_getaffinity(0)))
    from paper_2011_06636_b200 import problems as pr
    fx = fy = fz = None
    dx2 = (n + 1.0) ** 2
    if family == "2d5var":
        fx, fy = pr.harmonic_faces(np.exp(pr.gaussian_field(n, seed)), dx2)
    elif family == "3d7var":
        fx, fy, fz = pr.harmonic_faces_3d(np.exp(pr.gaussian_field_3d(n, seed)), dx2)
    elif family == "1d3var":
        fx = pr.harmonic_faces_1d(np.exp(pr.gaussian_field_1d(n, seed)), dx2)
    op = O.stencil(family, n, fx=fx, fy=fy, fz=fz)
    b = O.uniform_rhs(seed, op.n)
    seq = O.scheme(O.LADDER[14])[0]
    x = np.zeros(op.n)
    r, s = op.residual(x, b)
    sweeps = 0
    t0 = time.perf_counter()
    while True:
        x = op.update(x, r, seq[sweeps % len(seq)])
        r, s = op.residual(x, b)
        sweeps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    out = {"value": op.n * sweeps / el / 1e9, "unit": "GLUP/s", "cores": O.clib().oracle_threads(),
           "kind": "port", "seconds": el,
           "sample": f"{sweeps} SRJ sweeps (update+residual+norm) of the {family} n={n} grid, "
                     f"{el:.1f} s, oracle/srj_oracle.c OpenMP"}
    out["host"] = host_info()
    return out


def host_info():
    """What the CPU numbers were measured on."""
    import platform

    import numpy as np
    info = {"nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS"),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "numpy": np.__version__, "python": platform.python_version()}
    try:
        import scipy
        info["scipy"] = scipy.__version__
    except Exception:
        info["scipy"] = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return info


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_stock_sample(family, n, seed, budget_s):
    """The UNMODIFIED reference (baseline/_ref, installed from /root/reference
    with pip --target; pure Python + numpy/scipy) timed through its own public
    `run_cycle` on a bounded sweep sample of the same grid: its CSR SparseMatrix
    (from_coo, the path its solve takes), one level-14 scheme cycle cut by the
    stopping rule's sweep budget.  Where the CSR does not fit (512^3 and up)
    or baseline/_ref is absent, returns the reason instead."""
    import numpy as np
    if not os.path.isdir(os.path.join(REF_DIR, "srj")):
        return {"unavailable": "baseline/_ref not installed"}
    npts = n ** {"1d3": 1, "1d3var": 1, "2d5": 2, "2d5var": 2, "3d7": 3, "3d7var": 3}[family]
    if npts > 20_000_000:
        return {"unavailable": f"reference CSR for {npts} points does not fit host memory "
                               "(SURVEY §8d: 512^3 needs a duck-typed operator)"}
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import srj as ref  # the reference package
    from srj.sparse import SparseMatrix

    from paper_2011_06636_b200.operators import StencilOperator
    from paper_2011_06636_b200.problems import baseline_problem
    # the reference's own CSR of the same operator (its constructor
    # canonicalises and checks symmetry, as for a user matrix)
    t_build = time.perf_counter()
    if family in ("1d3", "3d7"):
        gen = ref.poisson_1d if family == "1d3" else ref.poisson_3d
        A = gen(n).A
    else:
        prob = baseline_problem(family, n, seed)
        rows, cols, vals = prob.A.coo()
        A = SparseMatrix.from_coo(npts, rows, cols, vals)
    t_build = time.perf_counter() - t_build
    from paper_2011_06636_b200.rng import uniform_rhs
    b = uniform_rhs(seed, npts)
    st = ref.SolverState(x=np.zeros(npts))
    scheme = ref.scheme_for_level(14)
    # whole level-14 cycles (the last one cut by the stopping rule's sweep
    # budget) until the time budget is spent; one timed sweep sizes the cut
    t0 = time.perf_counter()
    ref.run_cycle(A, b, st, scheme, stopping=ref.StoppingRule("relative_l2", 1e-300, 1),
                  baseline=1.0, record_history=False)
    one = time.perf_counter() - t0
    want = max(1, int(budget_s / max(one, 1e-9)))
    done, cycles = 0, 0
    t0 = time.perf_counter()
    while done < want:
        k = min(scheme.M, want - done)
        st, stats = ref.run_cycle(A, b, st, scheme,
                                  stopping=ref.StoppingRule("relative_l2", 1e-300,
                                                            st.total_iterations + k),
                                  baseline=1.0, record_history=False)
        done += stats.executed
        cycles += 1
    el = time.perf_counter() - t0
    stats = type("S", (), {"executed": done})
    del StencilOperator
    return {"value": npts * stats.executed / el / 1e9, "unit": "GLUP/s", "cores": 1,
            "kind": "reference",
            "sample": f"{stats.executed} sweeps in {cycles} level-14 run_cycle calls of the stock "
                      f"reference (baseline/_ref, CSR of {npts} points, built in {t_build:.1f} s), "
                      f"{el:.1f} s; scipy csr_matvec is single-threaded",
            "seconds": el}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2011_06636_b200.problems import CONFIGS
    if args.config == "c5":  # per-GPU load of config 5 = a 512^3 cube of points
        family, n = "3d7", 512
    else:
        family, extent, _ = CONFIGS[args.config]
        n = args.size or extent
    for _ in range(args.warmup):
        cpu_sample(family, n, args.seed, min(2.0, args.cpu_seconds))
    vals = []
    samples = []
    for _ in range(args.steps):
        c = cpu_sample(family, n, args.seed, args.cpu_seconds / max(args.steps, 1))
        vals.append(c["value"])
        samples.append(c)
    v = sum(vals) / len(vals)
    npts = n ** {"1d3": 1, "1d3var": 1, "2d5": 2, "2d5var": 2, "3d7": 3, "3d7var": 3}[family]
    line = {
        "impl": "reference", "metric": METRIC.get(args.config, METRIC["default"]), "value": v,
        "unit": "GLUP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        # each step is a bounded sample of the workload's sweeps (see cpu_baseline)
        "ms_per_step": sum(c["seconds"] for c in samples) * 1e3 / len(samples),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (SplitMix64 f, seeded)",
        "config": {"workload": CONFIG_DESC[args.config], "n": npts, "grid": n,
                   "step": "a bounded sample of the workload's SRJ sweeps (update + residual + "
                           "norm, level-14 scheme) on the same grid, not a whole solve: the "
                           "sweep count of a solve is the GPU arm's (identical scheme "
                           "sequence, tests/test_gpu_fullsize.py), so compare point-update "
                           "rates (GLUP/s)"},
        "cpu_baseline": {"value": v, "unit": "GLUP/s", "cores": samples[-1]["cores"],
                         "kind": "port", "sample": samples[-1]["sample"],
                         "host": samples[-1].get("host"),
                         "reference_stock": reference_stock_sample(family, n, args.seed,
                                                                   min(args.cpu_seconds, 10.0))},
        "e2e": {"value": v, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_slabs(args, rank, world, local):
    """Slab-decomposed solves, one process per GPU.

    c5: 3D Poisson z-slabs of nx x ny x planes_per_gpu on each of N GPUs (N = 8:
    the 1024^3 grid of BASELINE config 5; N = 1: the 134M-point per-GPU load of
    config 3), a fixed 50 heuristic cycles in throughput mode (weak scaling).
    c3 / c4 at N > 1: the config's fixed grid split into N z-slabs (3D) or row
    slabs (2D variable coefficient), solved to the tolerance (strong scaling).
    Halo planes go over NCCL (torch.distributed P2P) overlapped with the
    interior planes' sweep; one all-gather of per-sweep partials per cycle."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import (LocalExchanger, LocalTbExchanger,
                                                   SlabSolver, TbSlabSolver, TorchExchanger,
                                                   TorchTbExchanger, local_slabs, local_tb_slabs,
                                                   tb_ghost)
    from paper_2011_06636_b200.problems import CONFIGS, gaussian_field, harmonic_faces
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        init_dist(dev)
    throughput = args.config == "c5"
    face_x = face_y = None
    if throughput:
        family = "3d7"
        nx = args.size or 1024
        shape = (nx, nx, args.planes_per_gpu * world)
        rule = srj.StoppingRule("relative_l2", 1e-300, 10**9)
        max_cycles = args.cycles
    else:
        family, extent, _ = CONFIGS[args.config]
        n = args.size or extent
        shape = (n, n, n) if family == "3d7" else (n, n)
        if family == "2d5var":
            face_x, face_y = harmonic_faces(np.exp(gaussian_field(n, args.seed)), (n + 1.0) ** 2)
        rule = srj.StoppingRule("relative_l2", args.tol, 10**9)
        max_cycles = None
    # slabs of at least tb_ghost rows (planes) with an even row length run the
    # temporally blocked pass kernel with deep ghost rows (2D: 6 rows, 3D: 2
    # planes); otherwise one sweep per launch with one-plane halos
    tb = (family in ("2d5", "2d5var", "3d7") and shape[0] % 2 == 0
          and shape[-1] // world >= tb_ghost(family) and not args.no_tb_slabs)
    if tb:
        slabs = local_tb_slabs(family, shape, world, [rank], dev, face_x=face_x, face_y=face_y)
        if world > 1 and args.exchange == "native":
            from paper_2011_06636_b200.distributed import NcclTbExchanger
            solver = TbSlabSolver(slabs, NcclTbExchanger(dev), overlap=False)
        else:
            solver = TbSlabSolver(slabs, TorchTbExchanger() if world > 1 else LocalTbExchanger(1))
    else:
        slabs = local_slabs(family, shape, world, [rank], dev, face_x=face_x, face_y=face_y)
        solver = SlabSolver(slabs, TorchExchanger() if world > 1 else LocalExchanger(1))
    ctrl = srj.Heuristic()
    stream = torch.cuda.current_stream(dev)

    def one():
        solver.load(seed=args.seed)
        return solver.solve(ctrl, rule, record_history=False, max_cycles=max_cycles)

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms, sweeps = [], []
    launches0 = solver.launches
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = one()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            sweeps.append(rep.total_iterations)
    launches_timed = solver.launches - launches0
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    n_global = int(np.prod(shape))
    value = n_global * sum(sweeps) / (total_ms * 1e-3) / 1e9

    # e2e: each rank stages its slab's b and x0 from pinned host memory and reads
    # its slab of the solution back (H2D + D2H inside the timed region)
    s0 = slabs[0]
    n_owned = s0.count * s0.nx if tb else s0.A.n  # TB slabs also hold ghost rows
    solver.load(seed=args.seed)
    b_host = torch.empty(s0.A.n, dtype=torch.float64, pin_memory=True)
    b_host.copy_(s0.b.interior)
    x0_host = torch.zeros(s0.A.n, dtype=torch.float64, pin_memory=True)
    x_out = torch.empty(n_owned, dtype=torch.float64, pin_memory=True)

    def one_e2e():
        s0.b.copy_(b_host)
        s0.x.buf.zero_()
        s0.x_alt.buf.zero_()
        s0.x.copy_(x0_host)
        r = solver.solve(ctrl, rule, record_history=False, max_cycles=max_cycles)
        x_out.copy_(r.x[0])
        return r

    one_e2e()  # untimed warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms, e2e_sweeps = [], []
    for _ in range(max(1, min(args.steps, 2))):
        t0 = time.perf_counter()
        r = one_e2e()
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_sweeps.append(r.total_iterations)
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_val = n_global * sum(e2e_sweeps) / (e2e_total * 1e-3) / 1e9
    per_gpu_bytes = float(BYTES_PER_UPDATE[family]) * n_owned * sum(sweeps)
    peak, peak_kind = measured_peak()
    achieved = per_gpu_bytes / (total_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC["c5"] if throughput else METRIC["default"],
        "value": value, "unit": "GLUP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if throughput else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (f = 2u-1 from SplitMix64(seed), generated per slab on device)",
        "config": {"workload": (f"3D Poisson 7-pt {shape[0]}x{shape[1]}x{shape[2]} z-slabs "
                                f"({args.planes_per_gpu} planes/GPU), {args.cycles} cycles")
                               if throughput else CONFIG_DESC[args.config],
                   "grid": list(shape), "sweeps_per_step": sweeps[-1], "cycles": len(rep.cycles),
                   "levels": [c.level for c in rep.cycles],
                   "executed": [c.executed for c in rep.cycles],
                   "time_to_tolerance_ms": None if throughput else total_ms / args.steps,
                   "parallelism": f"{'z' if family == '3d7' else 'row'}-slabs x{world}, " + (
                       f"deep NCCL halo P2P ({tb_ghost(family)} {'planes' if family == '3d7' else 'rows'}) "
                       "per temporally blocked pass" if tb else
                       "NCCL halo P2P overlapped with interior sweeps")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                     "kernel": (("srj::k_tb3d_cycle<true> slab passes (srj_tb_pass, 2 sweeps)"
                                 if family == "3d7" else
                                 "srj::k_tbvar_cycle / k_tb2d_cycle slab passes (srj_tb_pass)")
                                if tb else
                                ("srj::k_sweep3d" if family == "3d7" else "srj::k_sweep2d")
                                + " (slab sweep)") + ", whole step incl. exchange"},
        "e2e": {"value": e2e_val, "unit": "GLUP/s", "h2d_bytes_per_step": 16 * s0.A.n * world,
                "d2h_bytes_per_step": 8 * n_owned * world,
                "ms_per_step": e2e_total / len(e2e_ms)},
        "clocks": clocks.summary(),
        # counted by the slab solver over the timed steps (+ one RHS fill per step)
        "gpu_launches": int(launches_timed + args.steps),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N = 1 only (contract)
        # the same stencil family on the oracle port; 3D samples a 512^3 cube
        # (config 3 / the per-GPU point count of config 5)
        line["cpu_baseline"] = cpu_sample(family, 512 if family == "3d7" else shape[0],
                                          args.seed, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.problems import CONFIGS
    from paper_2011_06636_b200.solver import solve_fields

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        init_dist(dev)
    family, extent, _ = CONFIGS[args.config]
    n = args.size or extent
    prob = srj.baseline_problem(family, n, seed=args.seed, device=dev, rhs_on_device=True)
    A = prob.A
    if args.sweeps_per_pass:
        A.set_sweeps_per_pass(args.sweeps_per_pass)
    b = A.field(prob.b)
    x = A.new_field()
    x_alt = A.new_field()
    rule = srj.StoppingRule("relative_l2", args.tol, 10**9)
    ctrl = srj.Heuristic()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    launch_ms = []
    launch_bytes = []
    bpu = BYTES_PER_UPDATE[family]

    def one_solve():
        x.buf.zero_()
        return solve_fields(A, b, x, x_alt, ctrl, rule, record_history=False,
                            device_loop=not args.host_loop)

    # warm-up (also builds every scheme the solve visits)
    rep = None
    for _ in range(args.warmup):
        rep = one_solve()
    torch.cuda.synchronize()

    # per-launch timing of the cycle kernel: time each srj_run_cycle with events
    from paper_2011_06636_b200 import operators as ops_mod
    orig_run_cycle = ops_mod.StencilOperator.run_cycle

    def timed_run_cycle(self, *a, **kw):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = orig_run_cycle(self, *a, **kw)
        e1.record(stream)
        e1.synchronize()
        if out.executed > 0:
            launch_ms.append(e0.elapsed_time(e1))
            launch_bytes.append(bpu * A.n * out.executed + RESIDUAL_BYTES[family] * A.n)
        return out

    orig_solve_device = ops_mod.StencilOperator.solve_device
    solve_launches = [0]

    def timed_solve_device(self, *a, **kw):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out, recs = orig_solve_device(self, *a, **kw)
        e1.record(stream)
        e1.synchronize()
        launch_ms.append(e0.elapsed_time(e1))
        launch_bytes.append(sum(bpu * A.n * r.executed + RESIDUAL_BYTES[family] * A.n
                                for r in recs if r.executed > 0))
        solve_launches[0] += 1
        return out, recs

    ops_mod.StencilOperator.run_cycle = timed_run_cycle
    ops_mod.StencilOperator.solve_device = timed_solve_device

    step_ms = []
    sweeps = []
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.fill_(1.0)   # evict b/x from L2 between steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = one_solve()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            sweeps.append(rep.total_iterations)
            launches += 2  # baseline / first residual
        torch.cuda.synchronize()
    # cycle kernels: one per cycle (host loop) or per srj_solve call (device loop)
    launches += len(launch_ms)
    ops_mod.StencilOperator.run_cycle = orig_run_cycle
    ops_mod.StencilOperator.solve_device = orig_solve_device
    if world > 1:
        dist.barrier()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    updates = A.n * sum(sweeps) * world
    value = updates / (total_ms * 1e-3) / 1e9

    # e2e: public API with pinned host buffers, H2D + D2H inside the region
    b_host = torch.empty(A.n, dtype=torch.float64, pin_memory=True)
    b_host.copy_(torch.as_tensor(prob.b))
    x0_host = torch.zeros(A.n, dtype=torch.float64, pin_memory=True)
    p_host = srj.ProblemInstance(A=A, b=b_host, x0=x0_host, stopping_norm="relative_l2")
    e2e_ms = []
    e2e_sweeps = []
    # the solution lands in a pinned host buffer allocated once (outside the
    # timed region); its D2H copy is inside every timed step
    x_out = torch.empty(A.n, dtype=torch.float64, pin_memory=True)
    srj.solve(p_host, ctrl, rule, record_history=False, out=x_out)  # untimed warm-up
    if world > 1:
        dist.barrier()
    for _ in range(max(1, min(args.steps, 3))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r2 = srj.solve(p_host, ctrl, rule, record_history=False, out=x_out)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_sweeps.append(r2.total_iterations)
        assert r2.total_iterations == rep.total_iterations
    e2e_total = sum(e2e_ms)
    if world > 1:  # whole job: all replicas' updates over the slowest rank's time
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_val = A.n * sum(e2e_sweeps) * world / (e2e_total * 1e-3) / 1e9

    # north_star's host-side scheme selection: the same solve with the
    # controller loop on the host (one launch + one small D2H per cycle)
    host_loop_ms = None
    if not args.host_loop and A.solve_supported():
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        x.buf.zero_()
        r3 = solve_fields(A, b, x, x_alt, ctrl, rule, record_history=False, device_loop=False)
        e1.record(stream)
        e1.synchronize()
        host_loop_ms = e0.elapsed_time(e1)
        assert r3.total_iterations == rep.total_iterations

    info = A.describe()
    peak, peak_kind = measured_peak()
    achieved = sum(launch_bytes) / (sum(launch_ms) * 1e-3) / 1e9 if launch_ms else None
    traffic = traffic_from_profile(args.config)
    line = {
        "metric": METRIC["default"],
        "value": value, "unit": "GLUP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (f = 2u-1, u from SplitMix64(seed) in index order; x0 = 0)",
        "config": {"workload": CONFIG_DESC[args.config], "grid": n, "n": A.n,
                   "sweeps_per_solve": sweeps[-1], "cycles_per_solve": len(rep.cycles),
                   "levels": [c.level for c in rep.cycles],
                   "executed": [c.executed for c in rep.cycles],
                   "time_to_tolerance_ms": ms_per_step,
                   "time_to_tolerance_ms_host_loop": host_loop_ms,
                   "controller": "device-resident loop (srj_solve)" if (
                       A.solve_supported() and not args.host_loop) else "host loop",
                   "margins": margins(rep.cycles, args.tol),
                   "l2": "flushed between steps (512 MiB write)",
                   "sweeps_per_pass": info["sweeps_per_pass"] if info["tb_supported"] else 1,
                   "launch": info,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "e2e": {"value": e2e_val, "unit": "GLUP/s",
                "h2d_bytes_per_step": 2 * 8 * A.n, "d2h_bytes_per_step": 8 * A.n,
                "ms_per_step": e2e_total / len(e2e_ms)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None,
                     "traffic": traffic["traffic"] if traffic else None,
                     "traffic_launch_alg_bytes": traffic["alg_bytes"] if traffic else None,
                     "traffic_over_alg": traffic["ratio"] if traffic else None,
                     "traffic_launch": traffic["launch"] if traffic else None,
                     "peak_kind": peak_kind, "kernel": kernel_name(family, info),
                     "bytes_per_update": bpu,
                     "launches_timed": len(launch_ms),
                     **dram_view(achieved, peak, traffic)},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # N = 1 only (contract)
        line["cpu_baseline"] = cpu_sample(family, n, args.seed, args.cpu_seconds)
        line["cpu_baseline"]["reference_stock"] = reference_stock_sample(
            family, n, args.seed, min(args.cpu_seconds, 10.0))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def margins(cycles, tol):
    """How far this solve is from a different scheme sequence or sweep count:
    the smallest |ratio - 0.4| and |ratio - 0.2| over the cycles (Heuristic
    thresholds, solver.py:125-140) and the last residual's distance below tol."""
    r = [c.residual_after / c.residual_before for c in cycles
         if c.residual_before > 0 and c.residual_after > 0]
    if not r:
        return None
    return {"min_abs_ratio_minus_0.4": min(abs(v - 0.4) for v in r),
            "min_abs_ratio_minus_0.2": min(abs(v - 0.2) for v in r),
            "last_res_after_over_tol": cycles[-1].residual_after / tol}


def dram_view(achieved, peak, traffic):
    """The roofline block's `achieved` is ALGORITHMIC bytes / kernel time (the
    contract's definition).  With temporal blocking and L2 residency that is an
    effective bandwidth above the HBM peak; the DRAM bandwidth the kernel really
    drew is achieved x traffic_over_alg (ncu DRAM bytes of a captured launch /
    its algorithmic bytes), and the limiter comes from that capture's stall
    profile (profiles/traffic.json)."""
    if not achieved or not traffic:
        return {}
    dram = achieved * traffic["ratio"]
    out = {"achieved_is": "effective (algorithmic bytes / time)",
           "dram_achieved": dram, "dram_frac": dram / peak}
    if traffic.get("limiter"):
        out["limiter"] = traffic["limiter"]
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # c5 always, and c3 / c4 on several GPUs (BASELINE: slab-sharded configs)
    if args.config == "c5" or (args.config in ("c3", "c4") and (world > 1 or args.slabs)):
        run_slabs(args, rank, world, local)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
