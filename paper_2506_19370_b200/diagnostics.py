"""Measurements and writers after the step (
src/workbench.cpp:187-412).

The per-point work runs on the device through the C ABI:

* ``energy_integral`` / ``area_integral`` (window_quadrature, :187-220): the
  per-point weights w_norm |det J| x trapezoid factors are built here once
  (``quadrature_weights``) and uploaded; ``fcsg_engine_integrals`` reduces
  h1 h2 sum wq v per subpatch on the device; the subpatch sums are added in id
  order as the reference does.
* ``density_gradient_raster`` (:222-305): ``fcsg_engine_gradient`` computes
  |grad rho| with the FC line derivatives; the raster's point location --
  the containing patch and the subpatch with the deepest window per pixel --
  is static geometry, built once on the host (``raster_plan``, the same
  search as the reference), and ``fcsg_engine_sample`` evaluates the bilinear
  samples on the device.

The rest is host-side post-processing of small arrays or file output, as in
the reference: ``schlieren`` (:307-320), ``write_pgm`` (:322-333),
``fit_shock_angle`` (:335-366), ``write_subpatch_csv`` (:368-386),
``write_manifest`` (:388-412).
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

from .problems import GAMMA

__all__ = ["Raster", "quadrature_weights", "set_quadrature", "energy_integral", "area_integral", "raster_plan",
           "density_gradient_raster", "schlieren", "write_pgm", "fit_shock_angle", "write_subpatch_csv",
           "write_manifest"]


@dataclass
class Raster:
    """include/fcs/workbench.hpp:90-95: v[j][i], row 0 at the bottom (y0)."""

    nx: int = 0
    ny: int = 0
    x0: float = 0.0
    y0: float = 0.0
    dx: float = 0.0
    dy: float = 0.0
    v: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))

    def at(self, i, j):
        return self.v[j, i]


# ---------------------------------------------------------------------------
# window quadrature


def _segments(d):
    """row_begin / col_begin of every local line (L-shaped subpatches)"""
    ci, cj = getattr(d, "cut_i", 0), getattr(d, "cut_j", 0)
    rb = np.where(np.arange(d.nj) < cj, ci, 0)
    cb = np.where(np.arange(d.ni) < ci, cj, 0)
    return rb, cb


def quadrature_weights(d) -> np.ndarray:
    """window_quadrature's per-point weight (src/workbench.cpp:195-201):
    w = w_norm det; halved at the first and last point of the row segment
    and of the column segment; 0 outside the point set. d.det = |det J|."""
    if getattr(d, "det", None) is None:
        raise ValueError("quadrature needs SubData.det (|det J|)")
    rb, cb = _segments(d)
    w = d.w_norm * d.det
    I = np.arange(d.ni)[None, :]
    J = np.arange(d.nj)[:, None]
    row_end = (I == rb[:, None]) | (I == d.ni - 1)
    col_end = (J == cb[None, :]) | (J == d.nj - 1)
    w = np.where(row_end, w * 0.5, w)
    w = np.where(col_end, w * 0.5, w)
    inset = ~((I < getattr(d, "cut_i", 0)) & (J < getattr(d, "cut_j", 0)))
    return np.ascontiguousarray(np.where(inset, w, 0.0))


def set_quadrature(E, dec):
    """upload every subpatch's weights (once per engine)"""
    for k, d in enumerate(dec.subs):
        E.set_quadrature(k, quadrature_weights(d))


def energy_integral(E) -> float:
    """window-weighted integral of E over the domain (energy_integral)"""
    return float(sum(E.integrals(3).tolist()))


def area_integral(E) -> float:
    """the same quadrature of the constant 1 (area_integral)"""
    return float(sum(E.integrals(-1).tolist()))


# ---------------------------------------------------------------------------
# |grad rho| raster


@dataclass
class RasterPlan:
    raster: Raster
    sub: np.ndarray
    il: np.ndarray
    jl: np.ndarray
    fu: np.ndarray
    fv: np.ndarray


def raster_plan(patches, subs, nf: int, nx: int, ny: int) -> RasterPlan:
    """density_gradient_raster's pixel search (src/workbench.cpp:240-299):
    domain bounding box of the valid points, then per pixel the first patch
    that contains it (margin 1e-9) and, in it, the subpatch with the deepest
    raw window (+1e-12, first maximum wins); cell origin and fractions
    clamped as the reference clamps them. Patches: multipatch.Patch (mapping,
    subdivision), subs: their SubData in global id order."""
    from . import multipatch as M

    x0 = min(float(d.x[d.mask != 0].min()) for d in subs)
    x1 = max(float(d.x[d.mask != 0].max()) for d in subs)
    y0 = min(float(d.y[d.mask != 0].min()) for d in subs)
    y1 = max(float(d.y[d.mask != 0].max()) for d in subs)
    r = Raster(nx, ny, x0, y0, (x1 - x0) / (nx - 1), (y1 - y0) / (ny - 1), np.zeros((ny, nx)))
    I, J = np.meshgrid(np.arange(nx), np.arange(ny))
    X = (x0 + I * r.dx).ravel()
    Y = (y0 + J * r.dy).ravel()
    n = X.size
    sub = np.full(n, -1, dtype=np.int32)
    il = np.zeros(n, dtype=np.int32)
    jl = np.zeros(n, dtype=np.int32)
    fu = np.zeros(n)
    fv = np.zeros(n)
    todo = np.ones(n, bool)
    sub_i0 = np.array([d.sp.i0 for d in subs], dtype=np.int64)
    sub_j0 = np.array([d.sp.j0 for d in subs], dtype=np.int64)
    sub_ni = np.array([d.ni for d in subs], dtype=np.int64)
    sub_nj = np.array([d.nj for d in subs], dtype=np.int64)
    for p in patches:
        idx = np.nonzero(todo)[0]
        if idx.size == 0:
            break
        ok, q1, q2 = M._contains_arr(p, X[idx], Y[idx], 1e-9)
        idx, q1, q2 = idx[ok], q1[ok], q2[ok]
        uu, vv = q1 / p.h1, q2 / p.h2
        bw = np.full(idx.size, -1.0)
        best = np.full(idx.size, -1, dtype=np.int64)
        bu = np.zeros(idx.size)
        bv = np.zeros(idx.size)
        for sp in p.subpatches:
            u, v = uu.copy(), vv.copy()
            if p.periodic1:
                while True:
                    m = u < sp.i0 - 1e-9
                    if not m.any():
                        break
                    u = np.where(m, u + p.np1, u)
                while True:
                    m = u > sp.i1 + 1e-9
                    if not m.any():
                        break
                    u = np.where(m, u - p.np1, u)
            inside = ~((u < sp.i0 - 1e-9) | (u > sp.i1 + 1e-9) | (v < sp.j0 - 1e-9) | (v > sp.j1 + 1e-9))
            inside &= ~((u < sp.i_cut - 1e-9) & (v < sp.j_cut - 1e-9))
            w = M._raw_window_arr(p, sp, u, v, nf) + 1e-12
            better = inside & (w > bw)
            bw = np.where(better, w, bw)
            best = np.where(better, sp.global_id, best)
            bu = np.where(better, u, bu)
            bv = np.where(better, v, bv)
        hit = best >= 0
        g = best[hit]
        i0, j0 = sub_i0[g], sub_j0[g]
        i0l = np.minimum(np.maximum(np.floor(bu[hit]).astype(np.int64) - i0, 0), sub_ni[g] - 2)
        j0l = np.minimum(np.maximum(np.floor(bv[hit]).astype(np.int64) - j0, 0), sub_nj[g] - 2)
        q = idx[hit]
        sub[q], il[q], jl[q] = g, i0l, j0l
        fu[q] = np.minimum(np.maximum(bu[hit] - i0 - i0l, 0.0), 1.0)
        fv[q] = np.minimum(np.maximum(bv[hit] - j0 - j0l, 0.0), 1.0)
        todo[q] = False
    return RasterPlan(r, sub, il, jl, fu, fv)


def density_gradient_raster(E, dec=None, nx: int = 0, ny: int = 0, plan: RasterPlan = None) -> Raster:
    """|grad rho| on a uniform nx x ny raster (density_gradient_raster):
    gradient and sampling on the device; pass a prebuilt plan to reuse the
    point location across outputs."""
    if plan is None:
        plan = raster_plan(dec.patches, dec.subs, getattr(dec, "nf", 5), nx, ny)
    E.gradient(0)
    vals = E.sample(plan.sub, plan.il, plan.jl, plan.fu, plan.fv)
    r = plan.raster
    return Raster(r.nx, r.ny, r.x0, r.y0, r.dx, r.dy, vals.reshape(r.ny, r.nx))


def schlieren(grad: Raster, beta: float = 10.0) -> Raster:
    """sigma = exp(-beta (g - min) / (max - min)); 1 on a uniform field"""
    lo, hi = float(grad.v.min()), float(grad.v.max())
    if hi - lo <= 0.0:
        v = np.ones_like(grad.v)
    else:
        v = np.exp(-beta * (grad.v - lo) / (hi - lo))
    return Raster(grad.nx, grad.ny, grad.x0, grad.y0, grad.dx, grad.dy, v)


def write_pgm(r: Raster, path: str):
    """binary PGM, rows top-down (row 0 of the raster is the bottom)"""
    v = np.clip(r.v, 0.0, 1.0)
    # std::lround: halves away from zero (values are >= 0)
    b = np.floor(255.0 * v[::-1] + 0.5).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(f"P5\n{r.nx} {r.ny}\n255\n".encode())
        f.write(b.tobytes())


def fit_shock_angle(grad: Raster, x_lo, x_hi, y_lo, y_hi) -> float:
    """straight-line fit to the per-column argmax of |grad rho| (degrees)"""
    i_lo = max(0, int(math.ceil((x_lo - grad.x0) / grad.dx)))
    i_hi = min(grad.nx - 1, int(math.floor((x_hi - grad.x0) / grad.dx)))
    j_lo = max(0, int(math.ceil((y_lo - grad.y0) / grad.dy)))
    j_hi = min(grad.ny - 1, int(math.floor((y_hi - grad.y0) / grad.dy)))
    gmax = 0.0
    for i in range(i_lo, i_hi + 1):
        for j in range(j_lo, j_hi + 1):
            gmax = max(gmax, grad.at(i, j))
    pts = []
    for i in range(i_lo, i_hi + 1):
        best, bj = 0.0, -1
        for j in range(j_lo, j_hi + 1):
            if grad.at(i, j) > best:
                best, bj = grad.at(i, j), j
        if bj < 0 or best < 0.2 * gmax:
            continue
        pts.append((grad.x0 + i * grad.dx, grad.y0 + bj * grad.dy))
    if len(pts) < 5:
        raise ValueError("fit_shock_angle: fewer than 5 usable columns")
    sx = sy = sxx = sxy = 0.0
    for x, y in pts:
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
    n = float(len(pts))
    slope = (n * sxy - sx * sy) / (n * sxx - sx * sx)
    return math.atan(slope) * 180.0 / math.pi


def _g17(v) -> str:
    return format(float(v), ".17g")


def write_subpatch_csv(E, dec, out_dir: str):
    """sub_<id>.csv: x,y,rho,u,v,p,mu,tau at the points of the set, the state
    read back from the device once per subpatch"""
    os.makedirs(out_dir, exist_ok=True)
    for k, d in enumerate(dec.subs):
        e = E.get_state(k)
        mu = E.get(k, "mu")
        tau = E.get(k, "tau")
        ci, cj = getattr(d, "cut_i", 0), getattr(d, "cut_j", 0)
        with open(os.path.join(out_dir, f"sub_{k}.csv"), "w") as f:
            f.write("x,y,rho,u,v,p,mu,tau\n")
            for jl in range(d.nj):
                for il in range(d.ni):
                    if d.mask[jl, il] == 0 or (il < ci and jl < cj):
                        continue
                    rho = e[0, jl, il]
                    u = e[1, jl, il] / rho
                    v = e[2, jl, il] / rho
                    p = (GAMMA - 1.0) * (e[3, jl, il] - 0.5 * rho * (u * u + v * v))
                    f.write(",".join(_g17(a) for a in (d.x[jl, il], d.y[jl, il], rho, u, v, p, mu[jl, il]))
                            + f",{int(tau[jl, il])}\n")


def write_manifest(out_dir: str, problem: str, steps: int, t_final: float, wall_seconds: float,
                   seconds_per_step: float, n_points: int, n_subpatches: int, n_workers: int = 1,
                   energy_series=None):
    """manifest.json (format fcs-manifest v1) and energy.csv"""
    os.makedirs(out_dir, exist_ok=True)
    j = {"format": "fcs-manifest", "version": 1, "problem": problem, "steps": steps, "t_final": t_final,
         "wall_seconds": wall_seconds, "seconds_per_step": seconds_per_step, "n_points": n_points,
         "n_subpatches": n_subpatches, "n_workers": n_workers}
    if energy_series:
        with open(os.path.join(out_dir, "energy.csv"), "w") as f:
            f.write("t,E\n")
            for t, en in energy_series:
                f.write(f"{_g17(t)},{_g17(en)}\n")
        j["energy_series"] = "energy.csv"
    with open(os.path.join(out_dir, "manifest.json"), "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")

