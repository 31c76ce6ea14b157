"""BASELINE config 3 (cylinder) or 4 (forward-facing step) on one GPU:
build, run, time. Usage: python scripts/config3_run.py [steps] [full|medium|step1|step2|step3]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
which = sys.argv[2] if len(sys.argv) > 2 else "full"
full = which == "full"
t0 = time.time()
if which.startswith("step"):
    dec, ic, meta = P.step_flow(int(which[4:]))
else:
    dec, ic, meta = P.cylinder_flow(full=full)
t1 = time.time()
ctx = N.Context(0)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=meta["cfl"]))
t2 = time.time()
npts = E.total_points()
E.run(3)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(E.stream())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
E.enqueue(steps)
b.record(st)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
E.ctx.check(0)
t, nst = E.time()
rho = np.concatenate([E.get(k, "e", 0)[dec.subs[k].mask != 0] for k in range(len(dec.subs))])
print(f"{which}: {len(dec.subs)} subpatches, {npts} points; build {t1 - t0:.1f}s, "
      f"engine setup {t2 - t1:.1f}s; {ms:.3f} ms/step = {5 * npts / (ms * 1e-3):.3e} pt-stage/s; t = {t:.4g} after "
      f"{nst} steps; rho in [{rho.min():.4f}, {rho.max():.4f}]; groups "
      + str({g: round(E.time_group(g, reps=3), 4) for g in ("viscosity", "pass_a", "pass_b", "pass_c", "filter")}))
