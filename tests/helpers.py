"""Shared test helpers: wire a product Decomposition into the numpy oracle."""
import numpy as np

from oracle import fcs_oracle as O
from paper_2506_19370_b200 import engine as EN, problems as P


def oracle_engine(dec, ic=None, cfl=0.5, states=None):
    mlp = O.Mlp.load(EN.DEFAULT_WEIGHTS)

    def osub(d, e):
        bc = lambda L: [None if b is None else (b[0], np.array(b[1]), b[2]) for b in L]
        return O.Sub(d.ni, d.nj, d.mask, d.iq1x, d.iq2x, d.iq1y, d.iq2y, d.h_min, d.h_max, d.w_norm,
                     1 / ((d.ni - 1) * d.h1), 1 / ((d.nj - 1) * d.h2), bc(d.bc_row_lo), bc(d.bc_row_hi),
                     bc(d.bc_col_lo), bc(d.bc_col_hi), e=np.array(e, dtype=np.float64))

    if states is None:
        states = [P.initial_state(dec, ic, k) for k in range(len(dec.subs))]
    sol, vis = dec.plan.per_sub(len(dec.subs))
    OE = O.Engine([osub(d, states[k]) for k, d in enumerate(dec.subs)], O.Plan(sol, vis), mlp, cfl=cfl)
    OE.finish_ic()
    return OE


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def line_rel_l2(got, ref):
    return np.linalg.norm(got - ref, axis=-1) / np.maximum(np.linalg.norm(ref, axis=-1), 1e-300)
