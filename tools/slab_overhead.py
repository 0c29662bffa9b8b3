"""Host overhead per temporally blocked slab pass, eager vs CUDA-graph cycles.

Three virtual ranks on one GPU (LocalTbExchanger) so the middle slab has the
shape of a middle rank at 8 GPUs:
  c4: 4096 x (3 x 512) var-coef rows -> middle slab 512 owned + 2 x 6 ghost = 524 rows
  c3: 512 x 512 x (3 x 64) planes     -> middle slab 64 owned + 2 x 2 ghost planes
For each mode: the host time to issue one cycle's forward work (snapshot,
passes with their exchanges, residual) measured without synchronising, the
GPU time of the same work (CUDA events), and both per pass.

python tools/slab_overhead.py [c4 c3]  -> one JSON line per (config, mode)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(argv):
    import numpy as np
    import torch

    import paper_2011_06636_b200 as srj
    from paper_2011_06636_b200.distributed import LocalTbExchanger, TbSlabSolver, local_tb_slabs
    from paper_2011_06636_b200.problems import gaussian_field, harmonic_faces
    dev = torch.device("cuda", 0)
    level = 14
    sch = srj.scheme_for_level(level)
    for cfg in argv or ["c4", "c3"]:
        if cfg == "c4":
            nx, world, rows = 4096, 3, 512
            shape = (nx, world * rows)
            k = np.exp(gaussian_field(nx, 0))          # (nx+2)^2 node field
            kk = k[:world * rows + 2, :]               # rows for the 4096 x 1536 grid
            fx, fy = harmonic_faces(kk, (nx + 1.0) ** 2)
            fam, kw = "2d5var", {"face_x": fx, "face_y": fy}
        else:
            nx, world, planes = 512, 3, 64
            shape = (nx, nx, world * planes)
            fam, kw = "3d7", {}
        for graphs in (False, True):
            slabs = local_tb_slabs(fam, shape, world, range(world), dev, **kw)
            solver = TbSlabSolver(slabs, LocalTbExchanger(world), graphs=graphs)
            solver.load(seed=0)
            om = solver._omegas(sch.ordered_omegas())
            M = sch.M
            passes = -(-M // solver.ghost)
            host, gpu = [], []
            for rep in range(6):
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                t0 = time.perf_counter()
                solver._forward(om, M)
                t1 = time.perf_counter()
                e1.record()
                e1.synchronize()
                if rep >= 2:  # eager first sight, capture, then replays
                    host.append((t1 - t0) * 1e6)
                    gpu.append(e0.elapsed_time(e1) * 1e3)
            line = {"config": cfg, "graphs": graphs, "world_virtual": world,
                    "slab_rows_middle": slabs[1].A.planes, "M": M, "passes": passes,
                    "host_us_per_cycle": min(host), "host_us_per_pass": min(host) / passes,
                    "gpu_us_per_cycle": min(gpu), "gpu_us_per_pass": min(gpu) / passes,
                    "launches_per_cycle_counted": solver.launches}
            print(json.dumps(line), flush=True)
            del solver, slabs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:])
