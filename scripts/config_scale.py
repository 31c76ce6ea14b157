"""BASELINE configs 3 and 4 at their stated scale and step counts on one
B200: config 3 (cylinder, ~4M points: problems.cylinder_flow(fine=True))
for 1000 supersteps, config 4 (forward-facing step, problems.step_flow(4):
12.9M points, CFL 0.25) for 2000 supersteps. Reports device time per
superstep (CUDA events over a steady window, graph replays), the rate, the
simulated time reached and the minimum density / pressure over all points at
the end (no InvalidStateError = positivity held at every stage).
    python scripts/config_scale.py [out.json] [c3,c3_025,c3_coarse,c4]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402


def run(name, build, steps, cfl):
    t0 = time.perf_counter()
    dec, ic, meta = build()
    tb = time.perf_counter() - t0
    ctx = N.Context(0)
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=cfl))
    npts = E.total_points()
    E.run(3)  # t = 0 step + graph capture
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(E.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timed = min(100, steps - 3)
    a.record(st)
    E.enqueue(timed)
    b.record(st)
    torch.cuda.synchronize()
    E.check_error()
    ms = a.elapsed_time(b) / timed
    t1 = time.perf_counter()
    failure = None
    try:
        E.run(steps - 3 - timed)
    except N.InvalidStateError as ex:  # where and when positivity was lost
        failure = {"error": str(ex), "patch": ex.patch, "subpatch": ex.subpatch, "i": ex.i, "j": ex.j, "t": ex.t}
    wall = time.perf_counter() - t1
    t, n = E.time()
    rmin = pmin = np.inf
    for k in range(len(dec.subs)):
        e = E.get_state(k)
        m = dec.subs[k].mask != 0
        rho = e[0][m]
        p = 0.4 * (e[3][m] - 0.5 * (e[1][m] ** 2 + e[2][m] ** 2) / rho)
        rmin, pmin = min(rmin, rho.min()), min(pmin, p.min())
    out = {"config": name, "points": npts, "subpatches": len(dec.subs), "build_s": tb, "cfl": cfl,
           "steps": n, "t_final": t, "ms_per_step": ms, "pt_stage_per_s": 5 * npts / (ms * 1e-3),
           "rest_wall_s": wall, "min_rho": float(rmin), "min_p": float(pmin), "failure": failure}
    print(json.dumps(out), flush=True)
    E.close()
    return out


which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c3", "c3_025", "c3_coarse", "c4"]
cases = {
    "c3": ("config3: Mach 3 cylinder, ring 3072x147 + 50 Cartesian 256^2 subpatches, CFL 0.5",
           lambda: P.cylinder_flow(True, fine=True), 1000, 0.5),
    "c3_025": ("config3: the same at CFL 0.25", lambda: P.cylinder_flow(True, fine=True), 1000, 0.25),
    "c3_coarse": ("config3 (2.57M layout), CFL 0.5", lambda: P.cylinder_flow(True), 1000, 0.5),
    "c4": ("config4: Mach 3 forward-facing step, step_flow(4), CFL 0.25", lambda: P.step_flow(4), 2000, 0.25),
}
res = [run(*cases[k]) for k in which]
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        json.dump(res, fh, indent=1)
