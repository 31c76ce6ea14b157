"""scaling.py against hand-worked values of the reference's definitions
(src/workbench.cpp:416-460)."""
import json
import math

import pytest

from paper_2506_19370_b200 import scaling as S


def test_scaling_metrics_weak_and_strong():
    recs = [S.ScalingRecord(1000, 1, 10.0, 100),   # base
            S.ScalingRecord(2000, 2, 11.0, 100),   # weak vs 0 (same load)
            S.ScalingRecord(1000, 2, 5.5, 100)]    # strong vs 0 (same N)
    rows = S.scaling_metrics(recs)
    assert rows[0].S == pytest.approx(1 * 10.0 * 1e6 / (4 * 1000 * 100))
    assert math.isnan(rows[0].Ew_T) and math.isnan(rows[0].Es_T)
    assert rows[1].Ew_T == pytest.approx(0.1 / 0.11)
    assert rows[1].Ew_S == pytest.approx(rows[0].S / rows[1].S)
    assert math.isnan(rows[1].Es_T)
    assert rows[2].Es_T == pytest.approx(0.1 * 1 / (0.055 * 2))
    assert rows[2].Es_S == pytest.approx(rows[0].S / rows[2].S)
    assert rows[2].Ew_T == pytest.approx(0.1 / 0.055) or math.isnan(rows[2].Ew_T)
    csv = S.scaling_csv(rows)
    assert csv.splitlines()[0] == "N,N_C,seconds,steps,S,Ew_T,Ew_S,Es_T,Es_S"
    with pytest.raises(ValueError):
        S.scaling_metrics(recs[:1])


def test_records_from_bench_lines():
    a = {"n_gpus": 1, "steps": 10, "ms_per_step": 3.5, "config": {"points_per_gpu": 4194304, "points_total": 4194304}}
    b = {"n_gpus": 2, "steps": 10, "ms_per_step": 3.6, "config": {"points_per_gpu": 4194304, "points_total": 8388608}}
    ref = {"impl": "reference", "n_gpus": 1, "steps": 10, "ms_per_step": 200.0, "config": {}}
    recs = S.records_from_bench([json.dumps(a), b, ref])
    assert [(r.n_points, r.n_workers) for r in recs] == [(4194304, 1), (8388608, 2)]
    rows = S.scaling_metrics(recs)
    assert rows[1].Ew_T == pytest.approx(3.5 / 3.6)
