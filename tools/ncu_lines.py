"""Stall samples and executed instructions per CUDA source line of one kernel.

python tools/ncu_lines.py <sass.csv from `ncu -i rep --page source --csv --print-source sass`> \
    <object or .so with -lineinfo> <mangled-name substring> [top N]
Joins the per-instruction rows of the ncu SASS page with nvdisasm's line table
(by instruction order inside the function).
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_table(binary, fn_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(binary)], cwd=tmp, check=True,
                   capture_output=True)
    lines = []
    for cubin in sorted(os.listdir(tmp)):
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True,
                             text=True).stdout
        cur, active = None, False
        for ln in out.splitlines():
            if ln.startswith("//----") and ".text." in ln:
                active = fn_sub in ln
                continue
            if not active:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m:
                lines.append((cur, m.group(2).strip()))
        if lines:
            break
    return lines


def main():
    sass_csv, binary, fn_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    r = list(csv.reader(open(sass_csv)))
    hi = [i for i, x in enumerate(r) if x and x[0] == "Address"][0]
    hdr, rows = r[hi], r[hi + 1:]
    si, ei, st = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("# Samples")
    table = line_table(binary, fn_sub)
    rows = [x for x in rows if len(x) == len(hdr)]
    if len(table) != len(rows):
        print(f"warning: {len(table)} disassembled vs {len(rows)} profiled instructions", file=sys.stderr)
    agg = collections.defaultdict(lambda: [0, 0])
    for (loc, _), row in zip(table, rows):
        try:
            agg[loc][0] += int(row[st] or 0)
            agg[loc][1] += int(row[ei] or 0)
        except ValueError:
            pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    src = {}
    print(f"samples {ts}  instructions {ti}")
    for loc, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        text = ""
        if loc:
            for root in ("paper_2011_06636_b200/csrc",):
                p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), root, loc[0])
                if os.path.exists(p):
                    if p not in src:
                        src[p] = open(p).read().splitlines()
                    if loc[1] - 1 < len(src[p]):
                        text = src[p][loc[1] - 1].strip()[:90]
        print(f"{100 * s / ts:5.1f}% smp {100 * n / ti:5.1f}% ins  {loc[0] if loc else '?'}:{loc[1] if loc else 0}  {text}")


if __name__ == "__main__":
    main()
