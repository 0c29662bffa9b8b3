"""Data collection (§8 f1): host-side aggregation / threshold fit / file
formats on CPU, the batched device trials against the reference's own
collections on the GPU."""

from __future__ import annotations

import math

import numpy as np
import pytest

import _parity as P
from paper_2011_06636_b200 import datacollect as dc


def _pt(action, rate, level=3, ratio=0.3, trial=1, step=1):
    return dc.DataPoint(action=action, avg_rate=rate, level=level, prev_ratio=ratio, trial=trial,
                        step=step)


def test_admissible_actions():
    assert dc.admissible(0) == ("increase", "keep")
    assert dc.admissible(5) == ("increase", "keep", "decrease")
    assert dc.admissible(dc.MAX_LEVEL) == ("keep", "decrease")


def test_aggregate_labels_separated_and_overlapping_clusters():
    rng = np.random.default_rng(0)
    sep = [_pt(a, base + 0.001 * rng.standard_normal(), step=i)
           for i in range(400) for a, base in (("increase", 0.5), ("keep", 0.3), ("decrease", 0.1))]
    (c,) = dc.aggregate(sep, n_set=2000)
    assert c.best_action == "increase" and c.actions["keep"].count == 400
    noisy = [_pt(a, 0.3 + rng.standard_normal(), step=i)
             for i in range(50) for a in ("increase", "keep")]
    assert dc.aggregate(noisy, n_set=1000)[0].best_action == dc.INCONCLUSIVE
    fwd = dc.aggregate(sep, n_set=90)
    rev = dc.aggregate(list(reversed(sep)), n_set=90)
    assert fwd == rev
    with pytest.raises(ValueError):
        dc.aggregate([])


def test_aggregate_partial_chunks():
    pts = [_pt("keep", 0.1, step=i) for i in range(105)]
    assert len(dc.aggregate(pts, n_set=100)) == 1     # tail of 5 < 10 dropped
    pts = [_pt("keep", 0.1, step=i) for i in range(115)]
    assert len(dc.aggregate(pts, n_set=100)) == 2     # tail of 15 kept


def _cluster(ratio, best, level=0):
    return dc.ClusterSummary(level_bucket=level, mean_ratio=ratio, best_action=best, actions={})


def test_fit_thresholds_midpoints_and_errors():
    cl = [_cluster(r, "keep") for r in (0.05, 0.1, 0.15)] + \
         [_cluster(r, "decrease") for r in (0.25, 0.3, 0.35)] + \
         [_cluster(r, "increase") for r in (0.45, 0.5, 0.6)]
    assert dc.fit_thresholds(cl) == pytest.approx((0.4, 0.2))
    cl2 = cl + [_cluster(0.32, dc.INCONCLUSIVE)]
    assert dc.fit_thresholds(cl2) == pytest.approx((0.4, 0.2))
    cl3 = cl + [_cluster(0.12, "increase")]      # one outlier of ten: tolerated
    t_hi, t_lo = dc.fit_thresholds(cl3)
    assert 0.35 < t_hi < 0.45 and 0.15 < t_lo < 0.25
    scrambled = [_cluster(0.1 * i, a) for i, a in enumerate(
        ["increase", "keep", "decrease", "increase", "keep", "decrease"])]
    with pytest.raises(dc.ThresholdFitError):
        dc.fit_thresholds(scrambled)
    with pytest.raises(ValueError):
        dc.fit_thresholds([_cluster(0.1, "keep"), _cluster(0.3, "decrease")])


def test_points_and_thresholds_files(tmp_path):
    pts = [_pt("keep", 0.25, ratio=0.125, trial=2, step=3), _pt("increase", 1.0 / 3.0)]
    path = tmp_path / "p.csv"
    with open(path, "w") as fh:
        dc.write_points_csv(fh, pts)
    back = dc.read_points_csv(str(path))
    assert [(p.trial, p.step, p.action, p.avg_rate, p.level, p.prev_ratio) for p in back] == \
        [(p.trial, p.step, p.action, p.avg_rate, p.level, p.prev_ratio) for p in pts]
    tpath = tmp_path / "t.txt"
    dc.write_thresholds(str(tpath), 0.4, 0.2)
    assert dc.read_thresholds(str(tpath)) == (0.4, 0.2)
    (tmp_path / "bad.txt").write_text("t_hi=0.4\n")
    with pytest.raises(ValueError):
        dc.read_thresholds(str(tmp_path / "bad.txt"))


def _check_points(points, packed):
    ints, reals = packed["ints"], packed["reals"]
    assert len(points) == len(ints)
    for p, i, r in zip(points, ints, reals):
        assert (p.trial, p.step, dc.ACTIONS.index(p.action), p.level) == tuple(i)
        for got, want in zip((p.avg_rate, p.prev_ratio, p.res_before, p.res_after), r):
            assert math.isclose(got, want, rel_tol=1e-9, abs_tol=1e-300), (p, r)


@pytest.mark.gpu
def test_batched_collect_matches_reference():
    g = P.traces()["datacollect"]
    _check_points(dc.collect([10], 2, target_tol=1e-8, seed=5), g["collect_10_t2_s5"])
    _check_points(dc.collect([5, 30], 2, target_tol=1e-8, seed=7), g["collect_5_30_t2_s7"])
    _check_points(dc.collect_until([5, 10], 200, target_tol=1e-6, seed=2), g["until_5_10_200_s2"])
    with pytest.raises(ValueError):
        dc.collect([], 1)


@pytest.mark.gpu
def test_batched_collection_recovers_reference_thresholds():
    g = P.traces()["datacollect"]["fit_10_50_40000_s3"]
    pts = dc.collect_until([10, 50], 40000, seed=3)
    assert len(pts) == g["count"]
    clusters = dc.aggregate(pts, n_set=1000)
    assert [(c.level_bucket, c.best_action) for c in clusters] == \
        [(c[0], c[2]) for c in g["clusters"]]
    t_hi, t_lo = dc.fit_thresholds(clusters)
    assert t_hi == pytest.approx(g["t_hi"], rel=1e-9) and t_lo == pytest.approx(g["t_lo"], rel=1e-9)
