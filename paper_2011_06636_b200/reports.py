"""schema=1 CSV writers for solve reports, traces and bench tables
(reference csvio.py:9-39, cli.py:26-27,91-104,202-211).

The layout is the reference's: a `# schema=1` line, optional `# key=value`
comments, a header, then rows whose reals carry 17 significant digits (exact
round trip).  Reports written from device solves therefore diff line-for-line
against the reference's `pkg/results/*.csv`; the residual columns differ only
where the norms' summation order shows in the 17th digit.
"""

from __future__ import annotations

SCHEMA_LINE = "# schema=1"
REPORT_HEADER = ["cycle", "level", "M", "res_before", "res_after", "avg_rate", "cum_iters"]
TRACE_HEADER = ["iteration", "residual"]
BENCH_HEADER = ["size", "controller", "rep", "iterations", "converged", "seconds"]


def fmt(value) -> str:
    """One CSV cell: booleans as 1/0, reals with 17 significant digits."""
    if isinstance(value, bool):
        return "1" if value else "0"
    if isinstance(value, float):
        return format(value, ".17g")
    return str(value)


def write_csv(fh, header, rows, comments=()) -> None:
    lines = [SCHEMA_LINE]
    lines.extend(f"# {c}" for c in comments)
    lines.append(",".join(header))
    lines.extend(",".join(fmt(v) for v in row) for row in rows)
    fh.write("\n".join(lines) + "\n")


def read_csv(path: str):
    """(header, rows of raw strings) of a schema=1 file."""
    with open(path, encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0].strip() != SCHEMA_LINE:
        raise ValueError(f"{path}: missing '{SCHEMA_LINE}' marker")
    body = [ln for ln in lines[1:] if ln and not ln.startswith("#")]
    if not body:
        raise ValueError(f"{path}: no header line")
    return body[0].split(","), [ln.split(",") for ln in body[1:]]


def report_rows(report):
    rows, cum = [], 0
    for c in report.cycles:
        cum += c.executed
        rows.append([c.cycle, c.level, c.M, c.residual_before, c.residual_after,
                     c.average_rate, cum])
    rows.append(["total", "", "", "", "", "", report.total_iterations])
    return rows


def write_report_csv(fh, report) -> None:
    """Per-cycle report of a SolveReport (reference cli.py:91-100)."""
    write_csv(fh, REPORT_HEADER, report_rows(report),
              comments=[f"converged={1 if report.converged else 0}"])


def write_trace_csv(fh, report) -> None:
    """Per-sweep residual trace (reference cli.py:103-104)."""
    write_csv(fh, TRACE_HEADER, report.residual_history)


def write_bench_csv(fh, rows) -> None:
    """Bench table rows (size, controller, rep, iterations, converged, seconds)."""
    write_csv(fh, BENCH_HEADER, rows)
