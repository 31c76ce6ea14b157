"""Init-time host geometry for rectangular (affine) patches.

The step engine consumes what the reference's init phase produces --
SubpatchData geometry/masks/metrics/line BCs (``init_subpatch_data``,
src/subpatch_data.cpp:69-154) and the CommPlan (``Engine::build_plan``,
src/runtime.cpp:89-274). This module builds those arrays from scratch for
affine I patches split by ``subdivide_Q`` (src/geometry.cpp:213-255), which is
every configuration the benchmark runs (BASELINE configs 2 and 5), using the
reference's own definitions:

* ``classify_end`` / ``fringe_mask``        src/geometry.cpp:444-495
* mapping, Jacobian inverse, local spacing  src/subpatch_data.cpp:96-118, include/fcs/linalg.hpp:17-27
* ``raw_window``                            src/viscosity.cpp:253-293
* intra-patch copy plan + w_norm            src/runtime.cpp:161-247 (copies only)

Curvilinear, periodic and corner (C1/C2) patches with inter-patch 6x6
interpolation are the next row; they are rejected
here rather than approximated.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# BcKind (include/fcs/bc.hpp:10-17)
INFLOW, OUTFLOW_PRESSURE, SLIP_WALL, NOSLIP_ADIABATIC, SUPERSONIC_OUTFLOW, ZERO_NORMAL_ALL = range(6)


class DecompositionError(RuntimeError):
    """include/fcs/errors.hpp:26-29"""


@dataclass
class BcSpec:
    """include/fcs/bc.hpp:19-23"""

    kind: int = SLIP_WALL
    state: tuple = (0.0, 0.0, 0.0, 0.0)
    pressure: float = 1.0


@dataclass
class SideInfo:
    on_gamma: bool = False
    tag: str = ""


@dataclass
class Subpatch:
    """include/fcs/geometry.hpp:150-169 (rectangles only)."""

    local_index: int
    i0: int
    i1: int
    j0: int
    j1: int
    global_id: int = -1

    @property
    def ni(self):
        return self.i1 - self.i0 + 1

    @property
    def nj(self):
        return self.j1 - self.j0 + 1

    def n_points(self):
        return self.ni * self.nj


@dataclass
class AffinePatch:
    """Patch with an AffineMap origin + q1 e1 + q2 e2 (include/fcs/geometry.hpp:70-83)."""

    origin: tuple
    e1: tuple
    e2: tuple
    sides: list  # 4 SideInfo: W, E, S, N
    index: int = 0
    nv: int = 9
    np1: int = 0
    np2: int = 0
    h1: float = 0.0
    h2: float = 0.0
    subpatches: list = field(default_factory=list)

    def map(self, q1, q2):
        o, a, b = self.origin, self.e1, self.e2
        return (o[0] + q1 * a[0]) + q2 * b[0], (o[1] + q1 * a[1]) + q2 * b[1]

    def jacobian(self):
        return (self.e1[0], self.e2[0], self.e1[1], self.e2[1])


def subdivide_Q(p: AffinePatch, r: int, s: int, n0: int, nv: int):
    """src/geometry.cpp:213-255 (non-periodic q1)."""
    if r < 1 or s < 1:
        raise ValueError("subdivide_Q: r, s must be >= 1")
    p.nv = nv
    p.np1 = r * (n0 - 1) + 2 * nv + 1
    p.h1 = 1.0 / (p.np1 - 1)
    p.np2 = s * (n0 - 1) + 2 * nv + 1
    p.h2 = 1.0 / (p.np2 - 1)
    p.subpatches = []
    for b in range(s):
        for a in range(r):
            p.subpatches.append(Subpatch(b * r + a, a * (n0 - 1), (a + 1) * (n0 - 1) + 2 * nv,
                                         b * (n0 - 1), (b + 1) * (n0 - 1) + 2 * nv))


def _end_side(p: AffinePatch, sp: Subpatch, axis: int, high: bool):
    """classify_end (src/geometry.cpp:444-469) for a rectangle: the patch side
    under the line end, or None."""
    if axis == 0:
        e = sp.i1 if high else sp.i0
        if e == 0:
            return p.sides[0]
        if e == p.np1 - 1:
            return p.sides[1]
        return None
    e = sp.j1 if high else sp.j0
    if e == 0:
        return p.sides[2]
    if e == p.np2 - 1:
        return p.sides[3]
    return None


def end_internal(p, sp, axis, high):
    side = _end_side(p, sp, axis, high)
    return not (side is not None and side.on_gamma)


def fringe_mask(p: AffinePatch, sp: Subpatch, nf: int) -> np.ndarray:
    """src/geometry.cpp:471-495: 1 interior, 2 within nf points of an internal side."""
    m = np.ones((sp.nj, sp.ni), dtype=np.uint8)
    if end_internal(p, sp, 0, False):
        m[:, :nf] = 2
    if end_internal(p, sp, 0, True):
        m[:, -nf:] = 2
    if end_internal(p, sp, 1, False):
        m[:nf, :] = 2
    if end_internal(p, sp, 1, True):
        m[-nf:, :] = 2
    return m


def raw_window(p: AffinePatch, sp: Subpatch, u, v, nf: int):
    """src/viscosity.cpp:253-293 for a rectangle of a non-corner patch."""
    band = 2.0 * p.nv

    def ramp(dist):
        t = np.clip((dist - nf) / (band - nf), 0.0, 1.0)
        s = np.sin(0.5 * math.pi * t)
        return s * s

    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    w = np.ones(np.broadcast(u, v).shape)
    if not (sp.i0 == 0 and p.sides[0].on_gamma):
        w = w * ramp(u - sp.i0)
    if not (sp.i1 == p.np1 - 1 and p.sides[1].on_gamma):
        w = w * ramp(sp.i1 - u)
    if not (sp.j0 == 0 and p.sides[2].on_gamma):
        w = w * ramp(v - sp.j0)
    if not (sp.j1 == p.np2 - 1 and p.sides[3].on_gamma):
        w = w * ramp(sp.j1 - v)
    return w


@dataclass
class SubData:
    """What one SubpatchData carries into the step (rectangular subpatch)."""

    sp: Subpatch
    patch: int
    ni: int
    nj: int
    h1: float
    h2: float
    mask: np.ndarray
    x: np.ndarray
    y: np.ndarray
    iq1x: np.ndarray
    iq2x: np.ndarray
    iq1y: np.ndarray
    iq2y: np.ndarray
    h_min: np.ndarray
    h_max: np.ndarray
    w_norm: np.ndarray = None
    # per line end: (kind, state4, pressure) or None -- rows lo/hi (nj), cols lo/hi (ni)
    bc_row_lo: list = None
    bc_row_hi: list = None
    bc_col_lo: list = None
    bc_col_hi: list = None
    # L-shaped subpatch (geom::Subpatch::i_cut/j_cut, local): points
    # (i < cut_i and j < cut_j) are not in the set
    cut_i: int = 0
    cut_j: int = 0
    det: np.ndarray = None  # |det J| (SubpatchData::det): window quadrature


@dataclass
class Plan:
    """CommPlan (include/fcs/runtime.hpp:16-49): copies, and optionally the
    6x6 interpolations as dicts of arrays (dst_sub, dst, src_sub, si0, sj0,
    wx (n, 6), wy (n, 6); plus w for the viscosity blend)."""

    sol_dst_sub: np.ndarray
    sol_dst: np.ndarray
    sol_src_sub: np.ndarray
    sol_src: np.ndarray
    v_dst_sub: np.ndarray
    v_dst: np.ndarray
    v_src_sub: np.ndarray
    v_src: np.ndarray
    v_w: np.ndarray
    sol_interps: dict = None
    visc_interps: dict = None

    def per_sub(self, nsub):
        """oracle-friendly view: per recipient (dst, src_sub, src) and (..., w)."""
        sol, vis = [], []
        for k in range(nsub):
            m = self.sol_dst_sub == k
            sol.append((self.sol_dst[m], self.sol_src_sub[m], self.sol_src[m]))
            mv = self.v_dst_sub == k
            vis.append((self.v_dst[mv], self.v_src_sub[mv], self.v_src[mv], self.v_w[mv]))
        return sol, vis


def init_subpatch_data(p: AffinePatch, sp: Subpatch, nf: int, bcs: dict) -> SubData:
    """src/subpatch_data.cpp:69-154 for a rectangular subpatch of an affine patch."""
    ii = np.arange(sp.i0, sp.i1 + 1, dtype=np.float64)
    jj = np.arange(sp.j0, sp.j1 + 1, dtype=np.float64)
    q1 = (ii * p.h1)[None, :] * np.ones((sp.nj, 1))
    q2 = (jj * p.h2)[:, None] * np.ones((1, sp.ni))
    x, y = p.map(q1, q2)
    a, b, c, d = p.jacobian()
    det = a * d - b * c
    sh = (sp.nj, sp.ni)
    iq1x = np.full(sh, d / det)
    iq1y = np.full(sh, -b / det)
    iq2x = np.full(sh, -c / det)
    iq2y = np.full(sh, a / det)

    def dist(xa, ya, xb, yb):
        return np.hypot(xa - xb, ya - yb)

    x1a, y1a = p.map(q1 + p.h1, q2)
    x1b, y1b = p.map(q1 - p.h1, q2)
    x2a, y2a = p.map(q1, q2 + p.h2)
    x2b, y2b = p.map(q1, q2 - p.h2)
    h1p = np.maximum(dist(x1a, y1a, x, y), dist(x, y, x1b, y1b))
    h2p = np.maximum(dist(x2a, y2a, x, y), dist(x, y, x2b, y2b))

    def resolve(axis, high):
        side = _end_side(p, sp, axis, high)
        if side is None or not side.on_gamma:
            return None
        if side.tag not in bcs:
            raise KeyError(f"no boundary condition for side tag '{side.tag}'")
        bc = bcs[side.tag]
        return (bc.kind, tuple(bc.state), bc.pressure)

    return SubData(sp=sp, patch=p.index, ni=sp.ni, nj=sp.nj, h1=p.h1, h2=p.h2,
                   mask=fringe_mask(p, sp, nf), x=x, y=y, iq1x=iq1x, iq2x=iq2x, iq1y=iq1y, iq2y=iq2y,
                   h_min=np.minimum(h1p, h2p), h_max=np.maximum(h1p, h2p),
                   bc_row_lo=[resolve(0, False)] * sp.nj, bc_row_hi=[resolve(0, True)] * sp.nj,
                   bc_col_lo=[resolve(1, False)] * sp.ni, bc_col_hi=[resolve(1, True)] * sp.ni,
                   det=np.full(sh, abs(det)))


def build_plan(p: AffinePatch, subs: list, nf: int) -> Plan:
    """Engine::build_plan (src/runtime.cpp:161-247) for one patch whose
    subpatches meet on coincident lattices: w_norm, the weighted viscosity
    copies and the fringe solution copies from the deepest-window interior
    donor. Fills ``SubData.w_norm``."""
    sol = {k: [] for k in ("dst_sub", "dst", "src_sub", "src")}
    vis = {k: [] for k in ("dst_sub", "dst", "src_sub", "src", "w")}
    S = len(subs)
    boxes = [(d.sp.i0, d.sp.i1, d.sp.j0, d.sp.j1) for d in subs]
    for k, d in enumerate(subs):
        sp = d.sp
        I, J = np.meshgrid(np.arange(sp.i0, sp.i1 + 1), np.arange(sp.j0, sp.j1 + 1))
        w_own = raw_window(p, sp, I.astype(np.float64), J.astype(np.float64), nf)
        denom = w_own.copy()
        contribs = []  # (donor k2, jl-slice, il-slice, w_raw, donor local idx, donor mask)
        for k2 in range(S):
            if k2 == k:
                continue
            a0, a1, b0, b1 = boxes[k2]
            ilo, ihi = max(sp.i0, a0), min(sp.i1, a1)
            jlo, jhi = max(sp.j0, b0), min(sp.j1, b1)
            if ilo > ihi or jlo > jhi:
                continue
            sl = (slice(jlo - sp.j0, jhi - sp.j0 + 1), slice(ilo - sp.i0, ihi - sp.i0 + 1))
            Iu, Jv = I[sl].astype(np.float64), J[sl].astype(np.float64)
            w2 = raw_window(p, subs[k2].sp, Iu, Jv, nf)
            d2 = subs[k2]
            src = (J[sl] - b0) * d2.ni + (I[sl] - a0)
            denom[sl] += w2
            contribs.append((k2, sl, w2, src, d2.mask.ravel()[src]))
        if not np.all(denom > 1e-14):
            raise DecompositionError(f"window partition vanishes in subpatch {k}")
        d.w_norm = w_own / denom
        dst_all = (J - sp.j0) * sp.ni + (I - sp.i0)
        best_w = np.full(denom.shape, -1.0)
        best_sub = np.full(denom.shape, -1)
        best_src = np.zeros(denom.shape, dtype=np.int64)
        for k2, sl, w2, src, dmask in contribs:
            w = w2 / denom[sl]
            keep = w > 1e-15
            vis["dst_sub"].append(np.full(keep.sum(), k))
            vis["dst"].append(dst_all[sl][keep])
            vis["src_sub"].append(np.full(keep.sum(), k2))
            vis["src"].append(src[keep])
            vis["w"].append(w[keep])
            # deepest-window interior copy donor (strictly greater wins: first max kept)
            cand = (dmask == 1) & (w2 > best_w[sl])
            bw, bs, bsrc = best_w[sl], best_sub[sl], best_src[sl]
            bw[cand] = w2[cand]
            bs[cand] = k2
            bsrc[cand] = src[cand]
            best_w[sl], best_sub[sl], best_src[sl] = bw, bs, bsrc
        fr = d.mask == 2
        if np.any(fr & (best_sub < 0)):
            raise DecompositionError(f"orphan fringe point in subpatch {k}")
        sol["dst_sub"].append(np.full(fr.sum(), k))
        sol["dst"].append(dst_all[fr])
        sol["src_sub"].append(best_sub[fr])
        sol["src"].append(best_src[fr])

    def cat(lst, dt):
        return np.concatenate(lst).astype(dt) if lst else np.zeros(0, dtype=dt)

    return Plan(cat(sol["dst_sub"], np.int32), cat(sol["dst"], np.int32), cat(sol["src_sub"], np.int32),
                cat(sol["src"], np.int32), cat(vis["dst_sub"], np.int32), cat(vis["dst"], np.int32),
                cat(vis["src_sub"], np.int32), cat(vis["src"], np.int32), cat(vis["w"], np.float64))


@dataclass
class Decomposition:
    patches: list
    subs: list  # SubData, global id order
    plan: Plan
    bcs: dict
    nf: int = 5

    def total_points(self):
        return sum(d.ni * d.nj for d in self.subs)


def rect_decomposition(origin, lx, ly, r, s, n0, nv, side_bcs, nf=5) -> Decomposition:
    """One affine I patch [x0, x0+lx] x [y0, y0+ly], subdivide_Q(r, s, n0, nv).
    side_bcs: 4 entries (W, E, S, N), a BcSpec (physical side) or None (interior side)."""
    return affine_decomposition(origin, (lx, 0.0), (0.0, ly), r, s, n0, nv, side_bcs, nf)


def affine_decomposition(origin, e1, e2, r, s, n0, nv, side_bcs, nf=5) -> Decomposition:
    """One affine I patch origin + q1 e1 + q2 e2 (a rotated / sheared
    parallelogram exercises every metric term), subdivide_Q(r, s, n0, nv)."""
    if nv <= nf:
        raise ValueError(f"window construction requires nv > nf (got nv={nv}, nf={nf})")
    names = ("w", "e", "s", "n")
    sides, bcs = [], {}
    for k, bc in enumerate(side_bcs):
        if bc is None:
            sides.append(SideInfo(False, ""))
        else:
            sides.append(SideInfo(True, names[k]))
            bcs[names[k]] = bc
    p = AffinePatch(origin=tuple(origin), e1=tuple(e1), e2=tuple(e2), sides=sides)
    subdivide_Q(p, r, s, n0, nv)
    for g, sp in enumerate(p.subpatches):
        sp.global_id = g
    subs = [init_subpatch_data(p, sp, nf, bcs) for sp in p.subpatches]
    plan = build_plan(p, subs, nf)
    return Decomposition([p], subs, plan, bcs, nf)
