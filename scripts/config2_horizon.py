"""BASELINE config 2 (one 512 x 512 subpatch, seeded Riemann quadrants, ANN
classifier, CFL 0.5) for its stated 200 supersteps: the product on the B200
against the compiled reference's own Engine::run (oracle/_ref; a single
subpatch is one reference worker, so this takes minutes of CPU time and is a
script, not a test). Prints, at steps 50 / 100 / 200, the per-field relative
L2 difference and the tau agreement (all points, and the points whose
reference logit margin exceeds 1e-9).
    python scripts/config2_horizon.py [n] [steps...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fcs_oracle as O, ref  # noqa: E402  (checker only)
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
marks = [int(a) for a in sys.argv[2:]] or [50, 100, 200]
ctx = N.Context(0)
dec, ic, meta = P.riemann_quadrants(n=n, seed=2)
p = dec.patches[0]
R = ref.RefEngine(p.origin[0], p.origin[1], p.e1[0], p.e2[1], 1, 1, n - 2 * p.nv, p.nv, [5, 5, 5, 5], cfl=meta["cfl"],
                  workers=os.cpu_count() or 1, weight_path=EN.DEFAULT_WEIGHTS)
e0 = P.initial_state(dec, ic, 0)
R.set_state(0, e0)
R.finish_ic()
E = EN.Engine(ctx, dec, cfg=EN.EngineConfig(cfl=meta["cfl"]), initial_states=[e0])
mlp = O.Mlp.load(EN.DEFAULT_WEIGHTS)
done = 0
for m in marks:
    t0 = time.time()
    R.run(m - 1)
    E.run(m - 1 - done)
    margin = O.classify_field(mlp, O.proxy_mwsb(R.get_state(0))[0])[1]
    R.run(m)
    E.run(1)
    done = m
    g, w = E.get_state(0), R.get_state(0)
    l2 = [float(np.linalg.norm(g[c] - w[c]) / max(np.linalg.norm(w[c]), 1e-300)) for c in range(4)]
    tau, tau_ref = E.get(0, "tau"), R.get(0, "tau")
    sure = margin > 1e-9
    print(f"step {m}: t = {E.time()[0]:.6f} (reference {R.time()[0]:.6f}); rel L2 per field "
          f"{' '.join(f'{v:.2e}' for v in l2)}; tau differs at {int((tau != tau_ref).sum())} of {tau.size} points, at "
          f"{int((tau[sure] != tau_ref[sure]).sum())} of the {int(sure.sum())} with margin > 1e-9; tau < 4 at "
          f"{int((tau_ref < 4).sum())} points ({time.time() - t0:.0f} s)", flush=True)
