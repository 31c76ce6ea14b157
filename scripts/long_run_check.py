"""Long-horizon stability of the non-smooth configurations, product against
the compiled reference on the SAME patches (oracle/_ref ref_engine_testgeom):
3 = the config-3 cylinder layout at 0.70M points, 5 = the config-4 step
layout (step_flow(1)). Our engine steps one superstep at a time (the error
word is checked every step) until InvalidStateError or N steps; the
reference then runs to the same step count (all host threads): both report
where and when positivity was lost, and the states are compared at a common
step before that.
    python scripts/long_run_check.py 3|5 [N]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref  # noqa: E402
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402
from tests.helpers import engine_from_reference  # noqa: E402

which = int(sys.argv[1])
nmax = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cfl = 0.5 if which == 3 else 0.25
threads = os.cpu_count() or 1
R = ref.RefEngine.testgeom(which, 0, cfl=cfl, workers=threads, weight_path=EN.DEFAULT_WEIGHTS)
ctx = N.Context(0)
E, dec = engine_from_reference(ctx, R, EN.EngineConfig(cfl=cfl))
fail = None
snap = {}
for k in range(1, nmax + 1):
    try:
        E.run(1)
    except N.InvalidStateError as ex:
        fail = {"step": k, "patch": ex.patch, "subpatch": ex.subpatch, "i": ex.i, "j": ex.j, "t": ex.t}
        break
    if k % 50 == 0:
        snap[k] = [E.get_state(s) for s in range(R.nsubs)]
print("product:", json.dumps({"steps_ok": k - 1 if fail else nmax, "failure": fail}), flush=True)
target = (fail["step"] if fail else nmax)
cmp_step = max([s for s in snap if s < target], default=None)
rfail = None
out = {}
try:
    if cmp_step:
        R.run(cmp_step)
        dn = wn = 0.0
        for s in range(R.nsubs):
            a, b = snap[cmp_step][s], R.get_state(s)
            dn += float(((a - b) ** 2).sum())
            wn += float((b ** 2).sum())
        out["rel_l2_at_step"] = [cmp_step, (dn / wn) ** 0.5]
        print("compare:", json.dumps(out), flush=True)
    R.run(target + 20)
except Exception as ex:  # the reference's InvalidStateError
    rfail = {"error": str(ex), "time": R.time()}
print("reference:", json.dumps({"ran_to": R.time(), "failure": rfail}), flush=True)
