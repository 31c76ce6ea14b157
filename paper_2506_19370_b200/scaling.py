"""Scaling metrics of a set of runs, as the reference's workbench reports them
(wb::scaling_metrics / scaling_csv, src/workbench.cpp:416-460):

* S = N_C * seconds * 1e6 / (4 N steps) -- core-microseconds per point per
  RK stage (the paper's normalised cost, with N_C the number of workers:
  GPUs here);
* E^s (strong) for a record with the same point count N as an earlier record
  with a different worker count: from the time per step, T_b N_C,b / (T_i
  N_C,i), and from S, S_b / S_i;
* E^w (weak) for a record whose load N / N_C is within 2% of an earlier
  record's with a different worker count: T_b / T_i and S_b / S_i.

The first matching earlier record is the base, as in the reference. Records
come from bench.py JSON lines (`records_from_bench`): N = points_total,
N_C = n_gpus, seconds = ms_per_step x steps / 1000.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass


@dataclass
class ScalingRecord:
    n_points: int
    n_workers: int
    seconds: float
    steps: int


@dataclass
class ScalingRow:
    rec: ScalingRecord
    S: float = math.nan
    Ew_T: float = math.nan
    Ew_S: float = math.nan
    Es_T: float = math.nan
    Es_S: float = math.nan


def scaling_metrics(recs):
    if len(recs) < 2:
        raise ValueError("scaling_metrics: need at least 2 records")
    rows = [ScalingRow(r, S=r.n_workers * r.seconds * 1e6 / (4.0 * r.n_points * r.steps)) for r in recs]

    def per_step(r):
        return r.seconds / r.steps

    for i, row in enumerate(rows):
        ri = row.rec
        for b in range(i):
            rb = rows[b].rec
            if rb.n_points == ri.n_points and rb.n_workers != ri.n_workers:
                row.Es_T = per_step(rb) * rb.n_workers / (per_step(ri) * ri.n_workers)
                row.Es_S = rows[b].S / row.S
                break
        for b in range(i):
            rb = rows[b].rec
            load_b, load_i = rb.n_points / rb.n_workers, ri.n_points / ri.n_workers
            if abs(load_b - load_i) <= 0.02 * load_b and rb.n_workers != ri.n_workers:
                row.Ew_T = per_step(rb) / per_step(ri)
                row.Ew_S = rows[b].S / row.S
                break
    return rows


def scaling_csv(rows) -> str:
    out = ["N,N_C,seconds,steps,S,Ew_T,Ew_S,Es_T,Es_S"]
    for r in rows:
        v = [r.rec.n_points, r.rec.n_workers, r.rec.seconds, r.rec.steps, r.S, r.Ew_T, r.Ew_S, r.Es_T, r.Es_S]
        out.append(",".join(f"{x:.12g}" if isinstance(x, float) else str(x) for x in v))
    return "\n".join(out) + "\n"


def records_from_bench(lines):
    """ScalingRecords of bench.py JSON lines (dicts or strings); the reference
    arm's lines and lines without a timing are skipped."""
    recs = []
    for ln in lines:
        d = json.loads(ln) if isinstance(ln, str) else ln
        if d.get("impl") == "reference" or "ms_per_step" not in d:
            continue
        n = d.get("config", {}).get("points_total") or d["config"].get("points_per_gpu", 0) * d["n_gpus"]
        recs.append(ScalingRecord(int(n), int(d["n_gpus"]), d["ms_per_step"] * d["steps"] * 1e-3, int(d["steps"])))
    return recs
