"""How localized is the artificial viscosity on the bench workload (config 5:
8 x 8 vortex tiles + 1e-3 noise)? Counts, after a few supersteps, the points
with tau < 4, the points with mu != 0 and the rows / columns on which mu is
not identically zero.    python scripts/mu_sparsity.py [steps...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402

ctx = N.Context(0)
dec, ic, _ = P.vortex_tiles(r=8, s=8)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
done = 0
for target in [int(a) for a in sys.argv[1:]] or [1, 3, 13, 50, 100]:
    E.run(target - done)
    done = target
    npts = low = nz = rows = cols = nrows = ncols = 0
    for k in range(len(dec.subs)):
        tau, mu = E.get(k, "tau"), E.get(k, "mu")
        npts += tau.size
        low += int((tau < 4).sum())
        nz += int((mu != 0).sum())
        rows += int((mu != 0).any(axis=1).sum())
        cols += int((mu != 0).any(axis=0).sum())
        nrows += mu.shape[0]
        ncols += mu.shape[1]
    print(f"step {done}: tau<4 at {low} of {npts} points ({100 * low / npts:.3f}%), mu != 0 at {nz} ({100 * nz / npts:.3f}%), "
          f"rows with mu != 0: {rows} of {nrows} ({100 * rows / nrows:.1f}%), columns: {cols} of {ncols} ({100 * cols / ncols:.1f}%)",
          flush=True)
