"""Summarise an `ncu --set full` report into the CSVs kept under profiles/.

python tools/ncu_summary.py gpurun_out/c3_tb3.ncu-rep profiles/r01o_c3_k_tb3d \
    [--traffic c3 --alg-bytes B --launch "..."]

Writes <prefix>_details.csv (the report's details page) and <prefix>_raw_subset.csv
(DRAM bytes, duration, pipe utilisation, stall reasons, launch configuration of the
captured launch).  With --traffic, records the launch's DRAM read+write bytes
against its algorithmic bytes in profiles/traffic.json under that config key
(read by bench.py into roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ("dram__", "gpu__time_duration", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
        "launch__", "sm__pipe_fp64", "sm__inst_executed_pipe_", "smsp__pcsamp_warps_issue_stalled",
        "smsp__issue_active", "sm__throughput", "smsp__inst_executed.sum", "lts__t_bytes")


def ncu_page(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                          text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("prefix")
    ap.add_argument("--traffic", help="config key in profiles/traffic.json")
    ap.add_argument("--alg-bytes", type=float)
    ap.add_argument("--launch", default="")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    with open(a.prefix + "_details.csv", "w") as fh:
        fh.write(ncu_page(a.rep, "details"))
    rows = list(csv.reader(io.StringIO(ncu_page(a.rep, "raw"))))
    head, units, vals = rows[0], rows[1], rows[2]
    keep = [i for i, k in enumerate(head) if i == 0 or k.startswith(KEEP)]
    with open(a.prefix + "_raw_subset.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        for r in (head, units, vals):
            w.writerow([r[i] for i in keep])
    m = dict(zip(head, vals))
    u = dict(zip(head, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}
    rd = float(m["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
    wr = float(m["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    dur = float(m["gpu__time_duration.sum"]) * tscale[u["gpu__time_duration.sum"]]
    print(f"DRAM read {rd / 1e9:.2f} GB, write {wr / 1e9:.2f} GB, {dur * 1e3:.3f} ms, "
          f"{(rd + wr) / dur / 1e9:.1f} GB/s")
    if a.traffic:
        path = os.path.join(ROOT, "profiles", "traffic.json")
        with open(path) as fh:
            tr = json.load(fh)
        tr[a.traffic] = {
            "traffic": rd + wr,
            "alg_bytes": a.alg_bytes,
            "duration_s": dur,
            "traffic_over_alg": (rd + wr) / a.alg_bytes,
            "achieved_GBps": a.alg_bytes / dur / 1e9,
            "launch": a.launch,
            "source": a.source,
        }
        with open(path, "w") as fh:
            json.dump(tr, fh, indent=1)
            fh.write("\n")


if __name__ == "__main__":
    main()
