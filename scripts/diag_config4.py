"""Per-step divergence of the product from the reference on config 4
(step_flow(k), reference geometry/plan), for several pass families."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import fcs_oracle as O, ref  # noqa: E402
from paper_2506_19370_b200 import _native as N, engine as EN, problems as PR  # noqa: E402
from helpers import engine_from_reference  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["default", "refo", "general"]
ctx = N.Context(0)
mlp = O.Mlp.load(EN.DEFAULT_WEIGHTS)
for var in variants:
    R = ref.RefEngine.testgeom(5 if scale == 1 else 6, 0, cfl=0.25, workers=os.cpu_count(), weight_path=EN.DEFAULT_WEIGHTS)
    cfg = EN.EngineConfig(cfl=0.25, reference_order=(var == "refo"), force_general=(var == "general"))
    E, _ = engine_from_reference(ctx, R, cfg)
    for s in range(1, steps + 1):
        # tau margins of the state entering this step (reference)
        pre = [R.get_state(k) for k in range(R.nsubs)]
        R.run(s)
        E.run(1)
        worst = (0.0, -1, -1)
        ntau = nlow = 0
        dn = np.zeros(4)
        wn = np.zeros(4)
        for k in range(R.nsubs):
            g, w = E.get_state(k), R.get_state(k)
            for c in range(4):
                dn[c] += float(np.sum((g[c] - w[c]) ** 2))
                wn[c] += float(np.sum(w[c] ** 2))
                err = float(np.linalg.norm(g[c] - w[c]) / max(np.linalg.norm(w[c]), 1e-300))
                if err > worst[0]:
                    worst = (err, k, c)
            t, tr = E.get(k, "tau"), R.get(k, "tau")
            bad = t != tr
            ntau += int(bad.sum())
            if bad.any():
                mk = R.get(k, "mask")
                e = np.where(mk[None] > 0, pre[k], np.array([1.4, 4.2, 0, 8.8])[:, None, None])
                try:
                    m = O.classify_field(mlp, O.proxy_mwsb(e)[0])[1]
                    nlow += int((bad & (m <= 1e-9)).sum())
                    print(f"   sub {k}: {int(bad.sum())} tau mismatches, margins there {np.sort(m[bad])[:6]}")
                except Exception as ex:
                    print("   margin failed", ex)
        dom = np.sqrt(dn / np.maximum(wn, 1e-300))
        print(f"{var} step {s}: domain rel L2 per field {dom}; worst per-sub rel L2 {worst[0]:.3e} (sub {worst[1]} comp {worst[2]}), tau mismatches {ntau}, "
              f"low-margin points {nlow}", flush=True)
    E.close()
