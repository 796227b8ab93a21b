"""Pins for oracle/metrics.py (definitions of tab:exp11)."""
import json
import os

from oracle import metrics as M
from oracle import scheduler as S
from workloads import c1_trace


def test_nearest_rank():
    assert M.nearest_rank(range(1, 101), 95) == 95       # S:433 worked by hand
    assert M.nearest_rank([5], 95) == 5
    assert M.nearest_rank([1, 2, 3, 4], 50) == 2


def test_cdf():
    assert M.jct_cdf([2, 2, 4]) == [(2, 2 / 3), (4, 1.0)]
    assert M.jct_cdf([7]) == [(7, 1.0)]


def test_tab_exp11_ratio_fixture():
    with open(os.path.join(os.path.dirname(__file__), "golden", "tab_exp11.json")) as f:
        g = json.load(f)
    assert round(g["FIFO"]["avg_jct"] / g["SRTF"]["avg_jct"], 2) == g["fifo_over_srtf_avg_jct"]


def test_summarize_hw_c1():
    jobs, C = c1_trace()
    f = M.summarize(jobs, S.simulate(jobs, C, S.FIFO).stats)
    s = M.summarize(jobs, S.simulate(jobs, C, S.SRTF).stats)
    assert f == {"makespan": 90000, "avg_queuing": (0 + 75000) / 2, "avg_jct": 82500,
                 "p95_jct": 85000, "n_jobs": 2}
    assert s["avg_jct"] == 51500 and s["makespan"] == 90000
