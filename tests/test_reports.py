"""schema=1 writers (§8 f4), pinned byte-for-byte against the reference's
pkg/results CSVs by feeding them the reference-run golden values (CPU)."""

from __future__ import annotations

import io
import os

import pytest

import _parity as P
from paper_2011_06636_b200 import reports
from paper_2011_06636_b200.solver import CycleStats, SolveReport

RESULTS = "/root/reference/pkg/results"


def _report_from_golden(name):
    c = P.case(name)
    cycles = [CycleStats(cycle=r[0], level=r[1], M=r[2], executed=r[3], residual_before=r[4],
                         residual_after=r[5], average_rate=r[6]) for r in c["cycles"]]
    hist = [tuple(h) for h in c.get("history", [])]
    return SolveReport(converged=c["converged"], total_iterations=c["total_iterations"],
                       cycles=cycles, wall_time=0.0, x=None, residual_history=hist)


def _body(path):
    with open(path) as fh:
        lines = fh.read().splitlines()
    return [ln for ln in lines if not ln.startswith("  $")]  # drop the command echo


@pytest.mark.skipif(not os.path.isdir(RESULTS), reason="reference not mounted")
@pytest.mark.parametrize("fname,name", [
    ("report_poisson1d_100_heuristic.csv", "poisson1d_100_heuristic"),
    ("report_poisson1d_100_increasing.csv", "poisson1d_100_increasing"),
    ("report_poisson1d_100_cjm63.csv", "poisson1d_100_cjm63"),
    ("report_laplace2d_64_heuristic.csv", "laplace2d_64_seed1"),
])
def test_report_writer_is_byte_identical(fname, name):
    buf = io.StringIO()
    reports.write_report_csv(buf, _report_from_golden(name))
    assert buf.getvalue().splitlines() == _body(os.path.join(RESULTS, fname))


@pytest.mark.skipif(not os.path.isdir(RESULTS), reason="reference not mounted")
@pytest.mark.parametrize("fname,name", [
    ("convergence_poisson1d_100_heuristic.csv", "poisson1d_100_heuristic"),
    ("convergence_laplace2d_64_heuristic.csv", "laplace2d_64_seed1"),
])
def test_trace_writer_is_byte_identical(fname, name):
    buf = io.StringIO()
    reports.write_trace_csv(buf, _report_from_golden(name))
    assert buf.getvalue().splitlines() == _body(os.path.join(RESULTS, fname))


def test_fmt_and_roundtrip(tmp_path):
    assert reports.fmt(True) == "1" and reports.fmt(False) == "0"
    assert reports.fmt(0.1) == "0.10000000000000001"
    assert reports.fmt(10.0) == "10" and reports.fmt(7) == "7"
    path = tmp_path / "t.csv"
    with open(path, "w") as fh:
        reports.write_bench_csv(fh, [[100, "heuristic", 0, 1003, True, 0.5]])
    header, rows = reports.read_csv(str(path))
    assert header == reports.BENCH_HEADER and rows == [["100", "heuristic", "0", "1003", "1", "0.5"]]
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n")
    with pytest.raises(ValueError):
        reports.read_csv(str(bad))
