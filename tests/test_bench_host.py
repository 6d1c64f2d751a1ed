"""Host logic of bench.py's roofline arithmetic (CPU only): the algorithmic bytes of a grid-path
attempt and the measured gather-bound floor."""
import json
import os

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM = 6546.6


def test_attempt_bytes_match_survey_table():
    # C4 70.0 / 78.0 MB, C5 3.50 / 3.90 GB per accepted attempt, B_pair 2.58 GB
    for (m, nnz), (ra, r2) in {(100_000, 2_000_000): (70.0e6, 78.0e6),
                               (5_000_000, 100_000_000): (3.50e9, 3.90e9)}.items():
        n = 2 * m
        pair, a = bench.attempt_bytes(n, m, nnz, "ra")
        _, b = bench.attempt_bytes(n, m, nnz, "r2")
        assert a == pytest.approx(ra, rel=2e-3) and b == pytest.approx(r2, rel=2e-3)
        assert pair == 24 * nnz + 4 * (m + 1) + 4 * (n + 1) + 8 * n + 8 * m
    assert bench.attempt_bytes(10_000_000, 5_000_000, 100_000_000, "ra")[0] == pytest.approx(2.58e9, rel=1e-3)


def _sweep():
    with open(os.path.join(ROOT, "profiles", "gather_rates.json")) as f:
        return sorted((d["array_mb"], d["ms_per_1e8"]) for d in json.load(f)["spmv_like_sweep"])


def test_gather_floor_at_table_points():
    pts = _sweep()
    # a square LP whose two targets have the same size S: each SpMV floor = nnz/1e8 x table(S)
    for mb, ms in pts:
        if mb > 64:      # past the knee a column split may beat the table value
            continue
        n = int(mb * 1e6 / 8)
        _, pair = bench.gather_floor_us(n, n, 100_000_000, "ra", HBM)
        assert pair == pytest.approx(2 * ms * 1e3, rel=1e-9)


def test_gather_floor_split_and_monotone():
    pts = dict(_sweep())
    t40 = pts[32.0] + (pts[48.0] - pts[32.0]) * (40 - 32) / 16     # ms per 1e8 gathers, 40 MB target
    full, pair = bench.gather_floor_us(10_000_000, 5_000_000, 100_000_000, "ra", HBM)
    unsplit = (pts[80.0] + t40) * 1e3                               # x' (80 MB) in one pass + y' (40 MB)
    two_pass = (t40 + 16 * 5_000_000 / (HBM * 1e9) * 1e3 + t40) * 1e3   # x' as two 40 MB halves + y'
    assert pair < unsplit                     # the split is the cheaper layout at C5
    assert pair == pytest.approx(two_pass, rel=1e-9)
    assert pair >= 2 * min(pts.values()) * 1e3
    # the r2HPDHG update moves more bytes than raPDHG's: its floor is higher by exactly that
    full2, pair2 = bench.gather_floor_us(10_000_000, 5_000_000, 100_000_000, "r2", HBM)
    assert pair2 == pair
    assert full2 - full == pytest.approx(((88e7 + 88 * 5e6) - (64e7 + 56 * 5e6)) / (HBM * 1e9) * 1e6, rel=1e-9)
    # more nonzeros, larger floor
    assert bench.gather_floor_us(10_000_000, 5_000_000, 200_000_000, "ra", HBM)[1] > pair


def test_infeasibility_leg_statuses_are_as_planted():
    """The bench's mixed-status batch: the oracle classifies a sample exactly as planted
    (OPTIMAL for c_j > 0, DUAL_INFEASIBLE for c_j < 0 along the unbounded column)."""
    import numpy as np
    import oracle
    lp, C, unbounded = bench.infeasibility_workload(1024)
    assert C.shape == (1024, lp.n) and unbounded.sum() == 512
    assert np.diff(lp.row_ptr).max() <= 8 and np.bincount(lp.col_idx, minlength=lp.n).max() <= 8
    idx = np.arange(0, 1024, 37)
    _, _, res = oracle.solve_batch(lp, C[idx], None, "ra", iteration_limit=200_000)
    got = np.array([r["status"] for r in res])
    assert (got == np.where(unbounded[idx], oracle.DUAL_INFEASIBLE, oracle.OPTIMAL)).all()
