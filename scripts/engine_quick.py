"""Quick GPU check of the full FC-SDNN step against the numpy oracle (dev script)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import fcs_oracle as O  # noqa: E402  (checker only)
from paper_2506_19370_b200 import _native as N, engine as EN, problems as P  # noqa: E402


def oracle_engine(dec, ic, cfl):
    mlp = O.Mlp.load(EN.DEFAULT_WEIGHTS)

    def osub(d, e):
        bc = lambda L: [None if b is None else (b[0], np.array(b[1]), b[2]) for b in L]
        return O.Sub(d.ni, d.nj, d.mask, d.iq1x, d.iq2x, d.iq1y, d.iq2y, d.h_min, d.h_max, d.w_norm,
                     1 / ((d.ni - 1) * d.h1), 1 / ((d.nj - 1) * d.h2), bc(d.bc_row_lo), bc(d.bc_row_hi),
                     bc(d.bc_col_lo), bc(d.bc_col_hi), e=e.copy())

    sol, vis = dec.plan.per_sub(len(dec.subs))
    OE = O.Engine([osub(d, P.initial_state(dec, ic, k)) for k, d in enumerate(dec.subs)], O.Plan(sol, vis), mlp,
                  cfl=cfl)
    OE.finish_ic()
    return OE


ctx = N.Context(0)
for name, (dec, ic, meta) in [("riemann64", P.riemann_quadrants(n=64, seed=2)),
                              ("vortex2x2", P.vortex_tiles(r=2, s=2, n0=46))]:
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5, debug_rhs=True))
    OE = oracle_engine(dec, ic, 0.5)
    for step in range(3):
        E.step_by_phases()
        OE.step()
        err = max(np.abs(E.get_state(k) - OE.subs[k].e).max() / np.abs(OE.subs[k].e).max() for k in range(len(dec.subs)))
        tm = sum(int((E.get(k, "tau") != OE.subs[k].tau).sum()) for k in range(len(dec.subs)))
        print(f"{name} step {step}: state rel err {err:.3e} tau mismatches {tm}", flush=True)
    # whole-step path (graph) must match the phase path
    E2 = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    E2.run(3)
    err = max(np.abs(E2.get_state(k) - E.get_state(k)).max() for k in range(len(dec.subs)))
    print(f"{name} graph run vs phase run: max abs diff {err:.3e}", flush=True)

# timing: config 2
dec, ic, meta = P.riemann_quadrants(n=512, seed=2)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(2)
torch.cuda.synchronize()
s = torch.cuda.ExternalStream(E.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 20
e0.record(s)
E.enqueue(steps)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
npts = E.total_points()
print(f"config2 512^2: {ms:.3f} ms/step  {5 * npts / (ms * 1e-3):.3e} pt-stage/s", flush=True)
dec, ic, meta = P.vortex_tiles(r=8, s=8)
E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
E.run(2)
torch.cuda.synchronize()
s = torch.cuda.ExternalStream(E.stream())
e0.record(s)
E.enqueue(steps)
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
npts = E.total_points()
print(f"config5 8x8x256^2: {ms:.3f} ms/step  {5 * npts / (ms * 1e-3):.3e} pt-stage/s", flush=True)
