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


# ---------------------------------------------------------------------------
# geometry and plan exported from the compiled reference (oracle/_ref): the
# SubpatchData + CommPlan the reference built, fed to the product through its
# public API -- the product never builds these geometries itself.


class _Sp:
    def __init__(self, i0, j0):
        self.i0, self.j0 = i0, j0


class _RefSub:
    pass


class RefDecomposition:
    """Duck-typed Decomposition (subs, plan) from a reference engine R."""

    def __init__(self, R):
        from paper_2506_19370_b200 import geometry as G
        self.subs = []
        sol = {k: [] for k in ("dst_sub", "dst", "src_sub", "src")}
        vis = {k: [] for k in ("dst_sub", "dst", "src_sub", "src", "w")}
        sint = {k: [] for k in ("dst_sub", "dst", "src_sub", "si0", "sj0", "wx", "wy")}
        vint = {k: [] for k in ("dst_sub", "dst", "src_sub", "si0", "sj0", "wx", "wy", "w")}
        for k in range(R.nsubs):
            info = R.sub_info(k)
            ni, nj = R.dims[k]
            d = _RefSub()
            d.sp = _Sp(info["i0"], info["j0"])
            d.patch, d.ni, d.nj, d.h1, d.h2 = info["patch"], ni, nj, info["h1"], info["h2"]
            d.cut_i, d.cut_j = info["cut_i"], info["cut_j"]
            d.mask = R.get(k, "mask").astype(np.uint8)
            for f in ("iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm", "x", "y"):
                setattr(d, f, R.get(k, f))
            L = R.lines(k)

            def ends(kind, bc, sl):
                return [None if kind[q] < 0 else (int(kind[q]), tuple(bc[q, :4]), float(bc[q, 4]))
                        for q in range(sl.start, sl.stop)]
            d.bc_row_lo = ends(L["kind_lo"], L["bc_lo"], slice(0, nj))
            d.bc_row_hi = ends(L["kind_hi"], L["bc_hi"], slice(0, nj))
            d.bc_col_lo = ends(L["kind_lo"], L["bc_lo"], slice(nj, nj + ni))
            d.bc_col_hi = ends(L["kind_hi"], L["bc_hi"], slice(nj, nj + ni))
            d.lines = L
            self.subs.append(d)
            for which, cp_d, it_d in ((0, sol, sint), (1, vis, vint)):
                cp, cw, it, iw = R.plan(k, which)
                cp_d["dst_sub"] += [k] * len(cp)
                cp_d["dst"] += list(cp[:, 0])
                cp_d["src_sub"] += list(cp[:, 1])
                cp_d["src"] += list(cp[:, 2])
                if which == 1:
                    cp_d["w"] += list(cw)
                it_d["dst_sub"] += [k] * len(it)
                it_d["dst"] += list(it[:, 0])
                it_d["src_sub"] += list(it[:, 1])
                it_d["si0"] += list(it[:, 2])
                it_d["sj0"] += list(it[:, 3])
                it_d["wx"] += list(iw[:, 0:6])
                it_d["wy"] += list(iw[:, 6:12])
                if which == 1:
                    it_d["w"] += list(iw[:, 12])
        arr = lambda v, t: np.asarray(v, dtype=t)  # noqa: E731
        fin = lambda dct: {k: (arr(v, np.float64).reshape(-1, 6) if k in ("wx", "wy") else  # noqa: E731
                               arr(v, np.float64) if k == "w" else arr(v, np.int32)) for k, v in dct.items()}
        self.plan = G.Plan(arr(sol["dst_sub"], np.int32), arr(sol["dst"], np.int32), arr(sol["src_sub"], np.int32),
                           arr(sol["src"], np.int32), arr(vis["dst_sub"], np.int32), arr(vis["dst"], np.int32),
                           arr(vis["src_sub"], np.int32), arr(vis["src"], np.int32), arr(vis["w"], np.float64),
                           sol_interps=fin(sint), visc_interps=fin(vint))

    def total_points(self):
        return sum(d.ni * d.nj for d in self.subs)


def engine_from_reference(ctx, R, cfg=None):
    """Product engine on the reference's geometry and plan, starting from the
    reference's state after Engine::init (IC, enforce_bc, exchange)."""
    dec = RefDecomposition(R)
    cfg = cfg or EN.EngineConfig(cfl=0.5)
    states = [R.get_state(k) for k in range(R.nsubs)]
    E = EN.Engine(ctx, dec, cfg=cfg, initial_states=None)
    for k, e in enumerate(states):
        E.set_state(k, e)
    return E, dec
