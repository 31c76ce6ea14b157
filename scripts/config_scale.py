"""BASELINE configs 3 and 4 at their stated scale on one B200: config 3
(cylinder, ~4M points: problems.cylinder_flow(fine=True)) for up to 1000
supersteps, config 4 (forward-facing step, problems.step_flow(4): 12.9M
points, CFL 0.25) for up to 2000. From the impulsive Mach 3 start these
layouts lose positivity at a wall after some hundreds of steps -- and so does
the reference's own Engine::run on the same patches, at the same step and
point (scripts/long_run_check.py, tests/test_horizon.py) -- so the run
proceeds in windows of 10 supersteps with the error word checked after each
and stops at the first InvalidStateError. Reports device time per superstep
(CUDA events over a steady window inside the run's stable part, graph
replays), the rate, the steps completed and where positivity was lost.
    python scripts/config_scale.py [out.json] [c3,c3_noslip,c4]"""
import json
import os
import sys
import time

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
    timed = 20
    a.record(st)
    E.enqueue(timed)
    b.record(st)
    torch.cuda.synchronize()
    E.check_error()
    ms = a.elapsed_time(b) / timed
    failure = None
    done = 3 + timed
    t1 = time.perf_counter()
    while done < steps:
        k = min(10, steps - done)
        try:
            E.run(k)
        except N.InvalidStateError as ex:
            failure = {"within_steps": [done + 1, done + k], "patch": ex.patch, "subpatch": ex.subpatch,
                       "i": ex.i, "j": ex.j, "t": ex.t}
            break
        done += k
    wall = time.perf_counter() - t1
    t, n = E.time()
    out = {"config": name, "points": npts, "subpatches": len(dec.subs), "build_s": tb, "cfl": cfl,
           "steps_requested": steps, "steps_completed": done, "t_reached": t, "ms_per_step": ms,
           "pt_stage_per_s": 5 * npts / (ms * 1e-3), "run_wall_s": wall, "positivity_lost": failure}
    print(json.dumps(out), flush=True)
    E.close()
    return out


which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c3", "c3_noslip", "c4"]
cases = {
    "c3": ("config3: Mach 3 cylinder (slip body), ring 3072x147 + 50 Cartesian 256^2 subpatches, CFL 0.5",
           lambda: P.cylinder_flow(True, fine=True), 1000, 0.5),
    "c3_noslip": ("config3 with the body noslip_adiabatic (the reference's flow-cylinder), CFL 0.5",
                  lambda: P.cylinder_flow(True, fine=True, body="noslip"), 1000, 0.5),
    "c4": ("config4: Mach 3 forward-facing step, step_flow(4), CFL 0.25", lambda: P.step_flow(4), 2000, 0.25),
}
res = [run(*cases[k]) for k in which]
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        json.dump(res, fh, indent=1)
