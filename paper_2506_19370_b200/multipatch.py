"""Init-time host geometry for general multi-patch decompositions (SURVEY.md
section 8(f) item 1): curvilinear mappings, periodic patches, C1 corner
patches with L-shaped subpatches, and the CommPlan with inter-patch 6x6
Lagrange interpolation.

Everything here runs once at engine construction and produces what the
reference's init phase produces -- per-subpatch geometry, masks, metrics and
line BCs (``init_subpatch_data``, src/subpatch_data.cpp:69-154) and the
CommPlan with the normalised windows (``Engine::build_plan``,
src/runtime.cpp:89-274) -- which ``engine.Engine`` uploads through the C ABI.
Restated from the reference's published definitions:

* mappings (affine, annulus, bilinear, curve sum of segments / arcs) and their
  Jacobians / inversion        include/fcs/geometry.hpp:57-136, src/geometry.cpp:35-99
* Patch.contains / max_spacing  src/geometry.cpp:161-208
* subdivide_Q / subdivide_L     src/geometry.cpp:210-334
* classify_end / fringe_mask    src/geometry.cpp:444-495
* check_min_overlap             src/geometry.cpp:502-560
* raw_window                    src/viscosity.cpp:253-293
* init_subpatch_data            src/subpatch_data.cpp:69-154
* build_plan                    src/runtime.cpp:57-274
* fcs-mesh v1 JSON              src/geometry.cpp:17-31,71-135,573-629 (mesh_to_json,
                                mesh_from_json, save_mesh, load_mesh)

Scalar arithmetic follows the reference's operation order (Python floats are
IEEE doubles and the reference is compiled without FMA contraction), so the
geometry and the plan match the reference's to round-off; tests/
test_multipatch.py checks them against the compiled reference.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .geometry import (INFLOW, NOSLIP_ADIABATIC, OUTFLOW_PRESSURE, SLIP_WALL, SUPERSONIC_OUTFLOW,  # noqa: F401
                       ZERO_NORMAL_ALL, BcSpec, DecompositionError, Plan, SideInfo)


class GeometryError(RuntimeError):
    """include/fcs/errors.hpp:18-21"""


def _hypot(x, y):
    return math.hypot(x, y)


def _inv(J):
    """Mat2::inverse (include/fcs/linalg.hpp:20-27): J = (a, b, c, d) = [[a, b], [c, d]]"""
    a, b, c, d = J
    dt = a * d - b * c
    return (d / dt, -b / dt, -c / dt, a / dt)


# ---------------------------------------------------------------------------
# mappings (q1, q2) -> (x, y)


class Mapping:
    def __call__(self, q1, q2):
        raise NotImplementedError

    def jacobian(self, q1, q2):
        raise NotImplementedError

    def invert(self, x, seed, tol=1e-10, max_iter=50):
        """damped Newton (src/geometry.cpp:41-62)"""
        q = seed
        mx, my = self(q[0], q[1])
        res = _hypot(mx - x[0], my - x[1])
        for _ in range(max_iter):
            if res <= tol:
                return q
            J = self.jacobian(q[0], q[1])
            a, b, c, d = J
            if abs(a * d - b * c) < 1e-300:
                return None
            ia, ib, ic, id_ = _inv(J)
            mx, my = self(q[0], q[1])
            vx, vy = x[0] - mx, x[1] - my
            dq = (ia * vx + ib * vy, ic * vx + id_ * vy)
            step = 1.0
            for h in range(8):
                qn = (q[0] + step * dq[0], q[1] + step * dq[1])
                nx, ny = self(qn[0], qn[1])
                rn = _hypot(nx - x[0], ny - x[1])
                if rn < res:
                    q, res = qn, rn
                    break
                step *= 0.5
                if h == 7:
                    return None
        return q if res <= tol else None


class AffineMap(Mapping):
    """origin + q1 e1 + q2 e2"""

    def __init__(self, origin, e1, e2):
        self.o, self.e1, self.e2 = tuple(origin), tuple(e1), tuple(e2)

    def __call__(self, q1, q2):
        o, a, b = self.o, self.e1, self.e2
        return (o[0] + q1 * a[0]) + q2 * b[0], (o[1] + q1 * a[1]) + q2 * b[1]

    def jacobian(self, q1, q2):
        return (self.e1[0], self.e2[0], self.e1[1], self.e2[1])

    def invert(self, x, seed=None, tol=1e-10, max_iter=50):
        J = self.jacobian(0.0, 0.0)
        a, b, c, d = J
        if abs(a * d - b * c) < 1e-300:
            return None
        ia, ib, ic, id_ = _inv(J)
        vx, vy = x[0] - self.o[0], x[1] - self.o[1]
        return (ia * vx + ib * vy, ic * vx + id_ * vy)


class AnnulusMap(Mapping):
    """ring around a circle: q1 = angle fraction, q2 = radial fraction"""

    def __init__(self, center, r0, r1, theta0, theta_extent):
        self.c, self.r0, self.r1, self.t0, self.dt = tuple(center), r0, r1, theta0, theta_extent

    def __call__(self, q1, q2):
        th = self.t0 + q1 * self.dt
        r = self.r0 + q2 * (self.r1 - self.r0)
        return self.c[0] + r * math.cos(th), self.c[1] + r * math.sin(th)

    def jacobian(self, q1, q2):
        th = self.t0 + q1 * self.dt
        r = self.r0 + q2 * (self.r1 - self.r0)
        dr = self.r1 - self.r0
        return (-r * self.dt * math.sin(th), dr * math.cos(th), r * self.dt * math.cos(th), dr * math.sin(th))

    def invert(self, x, seed=(0.0, 0.0), tol=1e-10, max_iter=50):
        dx, dy = x[0] - self.c[0], x[1] - self.c[1]
        r = _hypot(dx, dy)
        if r < 1e-300:
            return None
        q2 = (r - self.r0) / (self.r1 - self.r0)
        th = math.atan2(dy, dx)
        q1 = (th - self.t0) / self.dt
        period = 2 * math.pi / abs(self.dt)
        t = (q1 - seed[0]) / period
        rt = math.copysign(math.floor(abs(t) + 0.5), t)  # std::round
        q1 -= period * rt
        return (q1, q2)


class BilinearMap(Mapping):
    """quadrilateral with corners p00, p10, p01, p11"""

    def __init__(self, p00, p10, p01, p11):
        self.a = tuple(p00)
        self.b = (p10[0] - p00[0], p10[1] - p00[1])
        self.c = (p01[0] - p00[0], p01[1] - p00[1])
        self.d = (((p11[0] - p10[0]) - p01[0]) + p00[0], ((p11[1] - p10[1]) - p01[1]) + p00[1])

    def __call__(self, q1, q2):
        a, b, c, d = self.a, self.b, self.c, self.d
        qq = q1 * q2
        return ((a[0] + q1 * b[0]) + q2 * c[0]) + qq * d[0], ((a[1] + q1 * b[1]) + q2 * c[1]) + qq * d[1]

    def jacobian(self, q1, q2):
        b, c, d = self.b, self.c, self.d
        return (b[0] + q2 * d[0], c[0] + q1 * d[0], b[1] + q2 * d[1], c[1] + q1 * d[1])


class Segment:
    def __init__(self, a, b):
        self.a, self.b = tuple(a), tuple(b)

    def point(self, t):
        return self.a[0] + t * (self.b[0] - self.a[0]), self.a[1] + t * (self.b[1] - self.a[1])

    def derivative(self, t):
        return self.b[0] - self.a[0], self.b[1] - self.a[1]


class CircularArc:
    """include/fcs/geometry.hpp:37-55: center c, radius r, angle t0 -> t1"""

    def __init__(self, center, radius, theta0, theta1):
        self.c, self.r, self.t0, self.t1 = tuple(center), radius, theta0, theta1

    def point(self, t):
        cos, sin = (np.cos, np.sin) if isinstance(t, np.ndarray) else (math.cos, math.sin)
        th = self.t0 + t * (self.t1 - self.t0)
        return self.c[0] + self.r * cos(th), self.c[1] + self.r * sin(th)

    def derivative(self, t):
        cos, sin = (np.cos, np.sin) if isinstance(t, np.ndarray) else (math.cos, math.sin)
        th = self.t0 + t * (self.t1 - self.t0)
        return -self.r * (self.t1 - self.t0) * sin(th), self.r * (self.t1 - self.t0) * cos(th)


class CurveSumMap(Mapping):
    """corner mapping l_A(q1) + l_B(q2) - C"""

    def __init__(self, A, B, corner):
        self.A, self.B, self.C = A, B, tuple(corner)

    def __call__(self, q1, q2):
        ax, ay = self.A.point(q1)
        bx, by = self.B.point(q2)
        return (ax + bx) - self.C[0], (ay + by) - self.C[1]

    def jacobian(self, q1, q2):
        da, db = self.A.derivative(q1), self.B.derivative(q2)
        return (da[0], db[0], da[1], db[1])


# ---------------------------------------------------------------------------
# patches and subpatches

S, C1, C2, I = "S", "C1", "C2", "I"


@dataclass
class Subpatch:
    """include/fcs/geometry.hpp:150-169"""

    patch_index: int
    local_index: int
    i0: int
    i1: int
    j0: int
    j1: int
    i_cut: int = 0
    j_cut: int = 0
    l_shaped: bool = False
    global_id: int = -1

    @property
    def ni(self):
        return self.i1 - self.i0 + 1

    @property
    def nj(self):
        return self.j1 - self.j0 + 1

    def valid(self, i, j):
        if i < self.i0 or i > self.i1 or j < self.j0 or j > self.j1:
            return False
        return not (i < self.i_cut and j < self.j_cut)

    def row_begin(self, j):
        return self.i0 if j >= self.j_cut else self.i_cut

    def col_begin(self, i):
        return self.j0 if i >= self.i_cut else self.j_cut


@dataclass
class Patch:
    """include/fcs/geometry.hpp:171-215"""

    kind: str
    map: Mapping
    sides: list  # 4 SideInfo: W, E, S, N
    periodic1: bool = False
    wall_q1: SideInfo = field(default_factory=SideInfo)
    wall_q2: SideInfo = field(default_factory=SideInfo)
    index: int = -1
    r: int = 1
    s: int = 1
    n_cell: int = 83
    nv: int = 9
    np1: int = 0
    np2: int = 0
    h1: float = 0.0
    h2: float = 0.0
    i_corner: int = -1
    j_corner: int = -1
    subpatches: list = field(default_factory=list)

    def physical(self, i, j):
        return self.map(i * self.h1, j * self.h2)

    def lattice_valid(self, i, j):
        if i < 0 or i >= self.np1 or j < 0 or j >= self.np2:
            return False
        if self.kind == C1:
            return i >= self.i_corner or j >= self.j_corner
        return True

    def invert_point(self, x):
        """src/geometry.cpp:161-176: seed from a 10 x 10 sample, then invert"""
        best_q, best = (0.5, 0.5), 1e300
        ns = 9
        for a in range(ns + 1):
            for b in range(ns + 1):
                q1, q2 = a / ns, b / ns
                if self.kind == C1 and q1 < 0.5 and q2 < 0.5:
                    continue
                mx, my = self.map(q1, q2)
                d = _hypot(mx - x[0], my - x[1])
                if d < best:
                    best, best_q = d, (q1, q2)
        return self.map.invert(x, best_q, 1e-10, 50)

    def contains(self, x, margin):
        """src/geometry.cpp:178-191: the parameter point of x, or None"""
        q = self.invert_point(x)
        if q is None:
            return None
        mx, my = self.map(q[0], q[1])
        if _hypot(mx - x[0], my - x[1]) > 1e-8:
            return None
        lo, hi = -margin, 1.0 + margin
        if self.periodic1:
            if q[1] < lo or q[1] > hi:
                return None
        elif q[0] < lo or q[0] > hi or q[1] < lo or q[1] > hi:
            return None
        if self.kind == C1 and q[0] < 0.5 - margin and q[1] < 0.5 - margin:
            return None
        return q

    def max_spacing(self):
        """src/geometry.cpp:193-208"""
        ms0 = ms1 = 0.0
        wrap = self.np1 if self.periodic1 else self.np1 - 1
        for j in range(self.np2):
            for i in range(wrap):
                inn = (i + 1) % self.np1 if self.periodic1 else i + 1
                if not self.lattice_valid(i, j) or not self.lattice_valid(inn, j):
                    continue
                ax, ay = self.map(i * self.h1, j * self.h2)
                bx, by = self.map((i + 1) * self.h1, j * self.h2)
                ms0 = max(ms0, _hypot(bx - ax, by - ay))
        for j in range(self.np2 - 1):
            for i in range(self.np1):
                if not self.lattice_valid(i, j) or not self.lattice_valid(i, j + 1):
                    continue
                ax, ay = self.map(i * self.h1, j * self.h2)
                bx, by = self.map(i * self.h1, (j + 1) * self.h2)
                ms1 = max(ms1, _hypot(bx - ax, by - ay))
        return ms0, ms1


def subdivide_Q(p: Patch, r: int, s: int, n0: int, nv: int):
    """src/geometry.cpp:210-255"""
    if r < 1 or s < 1:
        raise ValueError("subdivide_Q: r, s must be >= 1")
    if p.kind == C1:
        raise ValueError("subdivide_Q: use subdivide_L for C1")
    p.r, p.s, p.n_cell, p.nv = r, s, n0, nv
    p.i_corner = p.j_corner = -1
    if p.periodic1:
        p.np1 = r * (n0 - 1)
        p.h1 = 1.0 / p.np1
    else:
        p.np1 = r * (n0 - 1) + 2 * nv + 1
        p.h1 = 1.0 / (p.np1 - 1)
    p.np2 = s * (n0 - 1) + 2 * nv + 1
    p.h2 = 1.0 / (p.np2 - 1)
    p.subpatches = []
    for b in range(s):
        for a in range(r):
            if p.periodic1:
                i0, i1 = a * (n0 - 1) - nv, (a + 1) * (n0 - 1) + nv
                if r == 1:
                    i0, i1 = 0, p.np1 - 1
            else:
                i0, i1 = a * (n0 - 1), (a + 1) * (n0 - 1) + 2 * nv
            j0, j1 = b * (n0 - 1), (b + 1) * (n0 - 1) + 2 * nv
            p.subpatches.append(Subpatch(p.index, b * r + a, i0, i1, j0, j1, i0, j0))


def subdivide_L(p: Patch, r: int, n1: int, nv: int):
    """src/geometry.cpp:257-334"""
    if r < 2 or r % 2:
        raise ValueError("subdivide_L: r must be even and >= 2")
    if p.kind != C1:
        raise ValueError("subdivide_L: patch must be C1")
    p.r = p.s = r
    p.n_cell, p.nv = n1, nv
    N = r * (n1 + 1) - 1
    p.np1 = p.np2 = N + 2 * nv
    p.h1 = p.h2 = 1.0 / (N + 2 * nv - 1)
    m = r // 2
    ic = (nv - 1) + m * (n1 + 1)
    p.i_corner = p.j_corner = ic
    NP = p.np1

    def cell_lo(a):
        return (nv - 1) + a * (n1 + 1)

    p.subpatches = []
    h0 = Subpatch(p.index, 0, max(0, cell_lo(m - 1) - nv), min(NP - 1, cell_lo(m + 1) + nv),
                  max(0, cell_lo(m - 1) - nv), min(NP - 1, cell_lo(m + 1) + nv), ic, ic, True)
    p.subpatches.append(h0)
    li = [1]

    def add_cell(a, b):
        i0, i1 = max(0, cell_lo(a) - nv), min(NP - 1, cell_lo(a + 1) + nv)
        j0, j1 = max(0, cell_lo(b) - nv), min(NP - 1, cell_lo(b + 1) + nv)
        if not (i0 >= ic or j0 >= ic):
            if j1 < ic:
                i0 = max(i0, ic)
            elif i1 < ic:
                j0 = max(j0, ic)
            else:
                raise GeometryError("subdivide_L: unexpected L-shaped cell subpatch")
        p.subpatches.append(Subpatch(p.index, li[0], i0, i1, j0, j1, i0, j0))
        li[0] += 1

    for b in range(m, 2 * m):
        for a in range(m):
            if not (a == m - 1 and b == m):
                add_cell(a, b)
    for b in range(m, 2 * m):
        for a in range(m, 2 * m):
            if not (a == m and b == m):
                add_cell(a, b)
    for b in range(m):
        for a in range(m, 2 * m):
            if not (a == m and b == m - 1):
                add_cell(a, b)


def _det_sign_sweep(p: Patch, n_samples: int = 100):
    """src/geometry.cpp:334-347: the mapping's Jacobian keeps one sign"""
    sign = 0
    for a in range(n_samples + 1):
        for b in range(n_samples + 1):
            q1, q2 = a / n_samples, b / n_samples
            if p.kind == C1 and q1 < 0.5 and q2 < 0.5:
                continue
            J = p.map.jacobian(q1, q2)
            d = J[0] * J[3] - J[1] * J[2]
            if abs(d) < 1e-14:
                raise GeometryError("mapping Jacobian vanishes")
            sg = 1 if d > 0 else -1
            if sign == 0:
                sign = sg
            if sg != sign:
                raise GeometryError("mapping Jacobian changes sign")


def _corner_checks(ellA, ellB, corner, t, who):
    pa0, pa1 = ellA.point(0.0), ellA.point(1.0)
    scale = max(1e-12, _hypot(pa0[0] - pa1[0], pa0[1] - pa1[1]))
    for c in (ellA, ellB):
        q = c.point(t)
        if _hypot(q[0] - corner[0], q[1] - corner[1]) > 1e-8 * scale:
            where = "pass through the corner at t=1/2" if t == 0.5 else "end at the corner (t=1)"
            raise GeometryError(f"{who}: curves must {where}")
    ta, tb = ellA.derivative(t), ellB.derivative(t)
    if abs(ta[0] * tb[1] - ta[1] * tb[0]) < 1e-12 * _hypot(*ta) * _hypot(*tb):
        raise GeometryError(f"{who}: tangents at the corner are parallel")


def build_c1_patch(ellA, ellB, corner, wall_tag="wall"):
    """src/geometry.cpp:351-369: convex-corner patch l_A(q1) + l_B(q2) - C,
    the curves crossing at the corner at t = 1/2; L-shaped point set"""
    _corner_checks(ellA, ellB, corner, 0.5, "build_c1_patch")
    p = Patch(C1, CurveSumMap(ellA, ellB, corner), [SideInfo() for _ in range(4)],
              wall_q1=SideInfo(True, wall_tag), wall_q2=SideInfo(True, wall_tag))
    _det_sign_sweep(p)
    return p


def build_c2_patch(ellA, ellB, corner, wall_tag="wall"):
    """src/geometry.cpp:371-389: concave-corner patch l_A(q1) + l_B(q2) - C,
    both curves ending at the corner (t = 1): E (= l_B) and N (= l_A) are
    walls, W and S interior"""
    _corner_checks(ellA, ellB, corner, 1.0, "build_c2_patch")
    p = Patch(C2, CurveSumMap(ellA, ellB, corner),
              [SideInfo(), SideInfo(True, wall_tag), SideInfo(), SideInfo(True, wall_tag)])
    _det_sign_sweep(p)
    return p


def classify_end(p: Patch, sp: Subpatch, axis: int, line: int, high: bool):
    """src/geometry.cpp:444-469: (internal, side)"""
    side = None
    if axis == 0:
        j = line
        e = sp.i1 if high else sp.row_begin(j)
        if not p.periodic1 and e == 0:
            side = p.sides[0]
        elif not p.periodic1 and e == p.np1 - 1:
            side = p.sides[1]
        elif p.kind == C1 and e == p.i_corner and j < p.j_corner:
            side = p.wall_q1
    else:
        i = line
        e = sp.j1 if high else sp.col_begin(i)
        if e == 0:
            side = p.sides[2]
        elif e == p.np2 - 1:
            side = p.sides[3]
        elif p.kind == C1 and e == p.j_corner and i < p.i_corner:
            side = p.wall_q2
    return not (side is not None and side.on_gamma), side


def fringe_mask(p: Patch, sp: Subpatch, nf: int) -> np.ndarray:
    """src/geometry.cpp:471-495"""
    ni, nj = sp.ni, sp.nj
    m = np.zeros((nj, ni), dtype=np.uint8)
    for j in range(sp.j0, sp.j1 + 1):
        m[j - sp.j0, sp.row_begin(j) - sp.i0:] = 1
    for j in range(sp.j0, sp.j1 + 1):
        ib = sp.row_begin(j)
        if classify_end(p, sp, 0, j, False)[0]:
            for k in range(nf):
                if ib + k <= sp.i1:
                    m[j - sp.j0, ib + k - sp.i0] = 2
        if classify_end(p, sp, 0, j, True)[0]:
            for k in range(nf):
                if sp.i1 - k >= ib:
                    m[j - sp.j0, sp.i1 - k - sp.i0] = 2
    for i in range(sp.i0, sp.i1 + 1):
        jb = sp.col_begin(i)
        if classify_end(p, sp, 1, i, False)[0]:
            for k in range(nf):
                if jb + k <= sp.j1:
                    m[jb + k - sp.j0, i - sp.i0] = 2
        if classify_end(p, sp, 1, i, True)[0]:
            for k in range(nf):
                if sp.j1 - k >= jb:
                    m[sp.j1 - k - sp.j0, i - sp.i0] = 2
    return m


def raw_window(p: Patch, sp: Subpatch, u: float, v: float, nf: int) -> float:
    """src/viscosity.cpp:253-293"""
    band = 2.0 * p.nv
    eps = 1e-9

    def ramp(dist):
        t = min(max((dist - nf) / (band - nf), 0.0), 1.0)
        s = math.sin(0.5 * math.pi * t)
        return s * s

    w = 1.0
    lo = sp.i_cut if v < sp.j_cut - eps else sp.i0
    internal = True
    if not p.periodic1 and lo == 0 and p.sides[0].on_gamma:
        internal = False
    if p.kind == C1 and lo == p.i_corner and v < p.j_corner - eps:
        internal = not p.wall_q1.on_gamma
    if internal:
        w *= ramp(u - lo)
    internal = not (not p.periodic1 and sp.i1 == p.np1 - 1 and p.sides[1].on_gamma)
    if internal:
        w *= ramp(sp.i1 - u)
    lo = sp.j_cut if u < sp.i_cut - eps else sp.j0
    internal = True
    if lo == 0 and p.sides[2].on_gamma:
        internal = False
    if p.kind == C1 and lo == p.j_corner and u < p.i_corner - eps:
        internal = not p.wall_q2.on_gamma
    if internal:
        w *= ramp(v - lo)
    internal = not (sp.j1 == p.np2 - 1 and p.sides[3].on_gamma)
    if internal:
        w *= ramp(sp.j1 - v)
    return w


def check_min_overlap(patches: list, nv: int):
    """src/geometry.cpp:502-560: raises DecompositionError listing the first
    orphan layer points / C1 corners no S patch reaches"""
    depth = 2 * nv + 1
    orphans = []
    for pi, p in enumerate(patches):
        def test(side, i, j):
            if not p.lattice_valid(i, j):
                return
            x = p.physical(i, j)
            for po, p2 in enumerate(patches):
                if po != pi and p2.contains(x, 1e-9) is not None:
                    return
            orphans.append((pi, side, i, j, x))

        if not p.periodic1:
            if not p.sides[0].on_gamma:
                for j in range(p.np2):
                    for i in range(min(depth, p.np1)):
                        test(0, i, j)
            if not p.sides[1].on_gamma:
                for j in range(p.np2):
                    for i in range(max(0, p.np1 - depth), p.np1):
                        test(1, i, j)
        if not p.sides[2].on_gamma:
            for i in range(p.np1):
                for j in range(min(depth, p.np2)):
                    test(2, i, j)
        if not p.sides[3].on_gamma:
            for i in range(p.np1):
                for j in range(max(0, p.np2 - depth), p.np2):
                    test(3, i, j)
    c1_fail = []
    for p in patches:
        if p.kind != C1:
            continue
        corner = p.map(0.5, 0.5)
        reached = False
        for ps in patches:
            if ps.kind != S:
                continue
            q = ps.contains(corner, 1e-7)
            if q is None:
                continue
            tol = 1e-6
            if ((ps.sides[0].on_gamma and abs(q[0]) < tol) or (ps.sides[1].on_gamma and abs(q[0] - 1) < tol)
                    or (ps.sides[2].on_gamma and abs(q[1]) < tol) or (ps.sides[3].on_gamma and abs(q[1] - 1) < tol)):
                reached = True
                break
        if not reached:
            c1_fail.append(f"C1 patch {p.index}: no S patch reaches its corner point")
    if orphans or c1_fail:
        lines = [f"FAIL: {len(orphans)} orphan layer points"]
        lines += [f"  patch {a} side {b} ({i},{j}) at ({x[0]:g},{x[1]:g})" for a, b, i, j, x in orphans[:8]]
        lines += ["  " + m for m in c1_fail]
        raise DecompositionError("minimum-overlap check failed:\n" + "\n".join(lines))


# ---------------------------------------------------------------------------
# subpatch data and the plan


@dataclass
class SubData:
    """One SubpatchData (include/fcs/subpatch_data.hpp:15-63) as the engine takes it."""

    sp: Subpatch
    patch: int
    ni: int
    nj: int
    h1: float
    h2: float
    cut_i: int
    cut_j: int
    mask: np.ndarray
    x: np.ndarray
    y: np.ndarray
    iq1x: np.ndarray
    iq2x: np.ndarray
    iq1y: np.ndarray
    iq2y: np.ndarray
    h_min: np.ndarray
    h_max: np.ndarray
    w_norm: np.ndarray
    bc_row_lo: list
    bc_row_hi: list
    bc_col_lo: list
    bc_col_hi: list
    det: np.ndarray = None  # |det J| (SubpatchData::det, src/subpatch_data.cpp:110): quadrature


def init_subpatch_data(p: Patch, sp: Subpatch, nf: int, bcs: dict) -> SubData:
    """src/subpatch_data.cpp:69-154"""
    ni, nj = sp.ni, sp.nj
    mask = fringe_mask(p, sp, nf)
    sh = (nj, ni)
    x, y = np.zeros(sh), np.zeros(sh)
    iq1x, iq2x, iq1y, iq2y = (np.zeros(sh) for _ in range(4))
    hmin, hmax = np.zeros(sh), np.zeros(sh)
    detJ = np.zeros(sh)
    M = p.map
    for j in range(sp.j0, sp.j1 + 1):
        for i in range(sp.i0, sp.i1 + 1):
            if not sp.valid(i, j):
                continue
            il, jl = i - sp.i0, j - sp.j0
            q1, q2 = i * p.h1, j * p.h2
            xp = M(q1, q2)
            x[jl, il], y[jl, il] = xp
            Jm = M.jacobian(q1, q2)
            Ji = _inv(Jm)
            iq1x[jl, il], iq2x[jl, il], iq1y[jl, il], iq2y[jl, il] = Ji[0], Ji[2], Ji[1], Ji[3]
            detJ[jl, il] = abs(Jm[0] * Jm[3] - Jm[1] * Jm[2])
            a, b = M(q1 + p.h1, q2), M(q1 - p.h1, q2)
            c, d = M(q1, q2 + p.h2), M(q1, q2 - p.h2)
            h1p = max(_hypot(a[0] - xp[0], a[1] - xp[1]), _hypot(xp[0] - b[0], xp[1] - b[1]))
            h2p = max(_hypot(c[0] - xp[0], c[1] - xp[1]), _hypot(xp[0] - d[0], xp[1] - d[1]))
            hmin[jl, il], hmax[jl, il] = min(h1p, h2p), max(h1p, h2p)

    def resolve(axis, line, high):
        internal, side = classify_end(p, sp, axis, line, high)
        if internal or side is None:
            return None
        if side.tag not in bcs:
            raise ValueError(f"no boundary condition for side tag '{side.tag}'")
        bc = bcs[side.tag]
        return (bc.kind, tuple(bc.state), bc.pressure)

    l_cut = sp.i_cut > sp.i0 and sp.j_cut > sp.j0
    return SubData(sp, p.index, ni, nj, p.h1, p.h2, sp.i_cut - sp.i0 if l_cut else 0,
                   sp.j_cut - sp.j0 if l_cut else 0, mask, x, y, iq1x, iq2x, iq1y, iq2y, hmin, hmax,
                   np.zeros(sh),
                   [resolve(0, j, False) for j in range(sp.j0, sp.j1 + 1)],
                   [resolve(0, j, True) for j in range(sp.j0, sp.j1 + 1)],
                   [resolve(1, i, False) for i in range(sp.i0, sp.i1 + 1)],
                   [resolve(1, i, True) for i in range(sp.i0, sp.i1 + 1)], detJ)


def _place(p: Patch, sp: Subpatch, u, v, eps):
    """place_in_subpatch (src/runtime.cpp:61-73)"""
    if p.periodic1:
        np1 = float(p.np1)
        while u < sp.i0 - eps:
            u += np1
        while u > sp.i1 + eps:
            u -= np1
    if u < sp.i0 - eps or u > sp.i1 + eps or v < sp.j0 - eps or v > sp.j1 + eps:
        return None
    if u < sp.i_cut - eps and v < sp.j_cut - eps:
        return None
    return u, v


def _lagrange(t, origin):
    """lagrange_weights (src/runtime.cpp:75-85)"""
    w = []
    for a in range(6):
        num, den = 1.0, 1.0
        for b in range(6):
            if a == b:
                continue
            num *= t - (origin + b)
            den *= float(a - b)
        w.append(num / den)
    return w


def _lround(x):
    return int(math.copysign(math.floor(abs(x) + 0.5), x))


def build_plan(patches: list, subs: list, nf: int) -> Plan:
    """Engine::build_plan (src/runtime.cpp:89-274): window normalisation
    (sets SubData.w_norm), viscosity-blend entries and the fringe solution
    entries (copies from the deepest-window interior donor of the same patch,
    else 6x6 interpolation from another patch)."""
    by_gid = {d.sp.global_id: (d, patches[d.patch]) for d in subs}
    boxes = {}
    for d in subs:
        valid = d.mask != 0
        b = boxes.setdefault(d.patch, [1e300, -1e300, 1e300, -1e300])
        b[0] = min(b[0], float(d.x[valid].min()))
        b[1] = max(b[1], float(d.x[valid].max()))
        b[2] = min(b[2], float(d.y[valid].min()))
        b[3] = max(b[3], float(d.y[valid].max()))
    margin = {p.index: 2.0 * max(p.max_spacing()) for p in patches}
    sol_c, vis_c, sol_i, vis_i = [], [], [], []

    def build_interp(c, slack):
        ds, _ = by_gid[c["sub"]]
        sp2 = ds.sp
        tu, tv = c["u"] - sp2.i0, c["v"] - sp2.j0
        bi, bj = math.floor(tu) - 2, math.floor(tv) - 2
        best, best_pen = None, 1e300
        for dj in range(-4, 5):
            for di in range(-4, 5):
                si, sj = bi + di, bj + dj
                if si < 0 or si + 5 >= ds.ni or sj < 0 or sj + 5 >= ds.nj:
                    continue
                out_u = max(0.0, si - tu, tu - (si + 5))
                out_v = max(0.0, sj - tv, tv - (sj + 5))
                if out_u > slack or out_v > slack:
                    continue
                if not (ds.mask[sj:sj + 6, si:si + 6] == 1).all():
                    continue
                pen = out_u + out_v + 0.01 * (abs(di) + abs(dj))
                if pen < best_pen:
                    best_pen, best = pen, (si, sj)
        if best is None:
            return None
        return c["sub"], best[0], best[1], _lagrange(tu, best[0]), _lagrange(tv, best[1])

    for d in subs:
        p = patches[d.patch]
        sp = d.sp
        gid = sp.global_id
        for j in range(sp.j0, sp.j1 + 1):
            for i in range(sp.row_begin(j), sp.i1 + 1):
                il, jl = i - sp.i0, j - sp.j0
                dst = jl * d.ni + il
                x = (float(d.x[jl, il]), float(d.y[jl, il]))
                contrib = []
                w_own = raw_window(p, sp, i, j, nf)
                for sp2 in p.subpatches:
                    if sp2.global_id == gid:
                        continue
                    pl = _place(p, sp2, float(i), float(j), 1e-9)
                    if pl is None:
                        continue
                    u, v = pl
                    i2, j2 = _lround(u), _lround(v)
                    ni2 = sp2.ni
                    contrib.append(dict(copy=True, sub=sp2.global_id, src=(j2 - sp2.j0) * ni2 + (i2 - sp2.i0),
                                        u=u, v=v, w=raw_window(p, sp2, u, v, nf)))
                for p2 in patches:
                    if p2.index == p.index:
                        continue
                    bb, m = boxes[p2.index], margin[p2.index]
                    if x[0] < bb[0] - m or x[0] > bb[1] + m or x[1] < bb[2] - m or x[1] > bb[3] + m:
                        continue
                    q = p2.contains(x, 1e-9)
                    if q is None:
                        continue
                    uu, vv = q[0] / p2.h1, q[1] / p2.h2
                    for sp2 in p2.subpatches:
                        pl = _place(p2, sp2, uu, vv, 1e-7)
                        if pl is None:
                            continue
                        u, v = pl
                        contrib.append(dict(copy=False, sub=sp2.global_id, u=u, v=v,
                                            w=raw_window(p2, sp2, u, v, nf)))
                denom = w_own
                for c in contrib:
                    denom += c["w"]
                if not denom > 1e-14:
                    raise DecompositionError(f"window partition vanishes at ({x[0]:f}, {x[1]:f}), subpatch {gid}")
                d.w_norm[jl, il] = w_own / denom
                for c in contrib:
                    w = c["w"] / denom
                    if w <= 1e-15:
                        continue
                    if c["copy"]:
                        vis_c.append((gid, dst, c["sub"], c["src"], w))
                    else:
                        ie = build_interp(c, 2.5)
                        if ie is None:
                            raise DecompositionError(f"no admissible viscosity stencil in donor subpatch {c['sub']} "
                                                     f"for ({x[0]:f}, {x[1]:f})")
                        vis_i.append((gid, dst) + ie + (w,))
                if d.mask[jl, il] == 2:
                    best = None
                    for c in contrib:
                        if not c["copy"]:
                            continue
                        ds2, _ = by_gid[c["sub"]]
                        if ds2.mask.reshape(-1)[c["src"]] != 1:
                            continue
                        if best is None or c["w"] > best["w"]:
                            best = c
                    if best is not None:
                        sol_c.append((gid, dst, best["sub"], best["src"]))
                    else:
                        cand = sorted((c for c in contrib if not c["copy"]), key=lambda c: -c["w"])
                        for c in cand:
                            ie = build_interp(c, 0.5)
                            if ie is not None:
                                sol_i.append((gid, dst) + ie)
                                break
                        else:
                            raise DecompositionError(f"orphan fringe point at ({x[0]:f}, {x[1]:f}), subpatch {gid}")

    def cols(rows, n):
        return [np.array([r[k] for r in rows]) for k in range(n)] if rows else [np.zeros(0)] * n

    sc = cols(sol_c, 4)
    vc = cols(vis_c, 5)
    i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731

    def interps(rows, with_w):
        if not rows:
            out = dict(dst_sub=i32([]), dst=i32([]), src_sub=i32([]), si0=i32([]), sj0=i32([]),
                       wx=np.zeros((0, 6)), wy=np.zeros((0, 6)))
            if with_w:
                out["w"] = np.zeros(0)
            return out
        out = dict(dst_sub=i32([r[0] for r in rows]), dst=i32([r[1] for r in rows]),
                   src_sub=i32([r[2] for r in rows]), si0=i32([r[3] for r in rows]), sj0=i32([r[4] for r in rows]),
                   wx=np.array([r[5] for r in rows]), wy=np.array([r[6] for r in rows]))
        if with_w:
            out["w"] = np.array([r[7] for r in rows])
        return out

    return Plan(i32(sc[0]), i32(sc[1]), i32(sc[2]), i32(sc[3]), i32(vc[0]), i32(vc[1]), i32(vc[2]), i32(vc[3]),
                np.asarray(vc[4], dtype=np.float64), sol_interps=interps(sol_i, False),
                visc_interps=interps(vis_i, True))


@dataclass
class MultiPatchDecomposition:
    """What engine.Engine consumes: subs (SubData, global id order) and plan."""

    patches: list
    subs: list
    plan: Plan
    bcs: dict
    nf: int = 5

    def total_points(self):
        return int(sum(int((d.mask != 0).sum()) for d in self.subs))

    def initial_state(self, ic, sub):
        """Engine::apply_ic at the points of the set (src/runtime.cpp:276-283)"""
        d = self.subs[sub]
        e = np.asarray(ic(d.x, d.y), dtype=np.float64)
        return np.ascontiguousarray(e * (d.mask != 0)[None])


def build_decomposition(patches: list, bcs: dict, nv: int, nf: int = 5, validate_overlap: bool = True,
                        fast: bool = False):
    """Engine::init's geometry part (src/runtime.cpp:293-305): ids, overlap
    check, SubpatchData, plan. Patches must already be subdivided. fast: the
    vectorised path (same results; for large decompositions)."""
    for k, p in enumerate(patches):
        p.index = k
        if p.nv <= nf:
            raise ValueError(f"window construction requires nv > nf (got nv={p.nv}, nf={nf})")
    gid = 0
    for p in patches:
        for sp in p.subpatches:
            sp.patch_index = p.index
            sp.global_id = gid
            gid += 1
    if validate_overlap:
        (_check_min_overlap_fast if fast else check_min_overlap)(patches, nv)
    init = _init_subpatch_data_fast if fast else init_subpatch_data
    subs = [init(p, sp, nf, bcs) for p in patches for sp in p.subpatches]
    plan = (_build_plan_fast if fast else build_plan)(patches, subs, nf)
    return MultiPatchDecomposition(patches, subs, plan, bcs, nf)


# ---------------------------------------------------------------------------
# vectorised builder: the same computations as above on numpy arrays (one
# subpatch or one patch side at a time), for decompositions of millions of
# points. build_decomposition(..., fast=True) uses it; tests/
# test_multipatch.py checks it against the scalar path.


def _map_arr(M, q1, q2):
    if isinstance(M, AnnulusMap):
        th = M.t0 + q1 * M.dt
        r = M.r0 + q2 * (M.r1 - M.r0)
        return M.c[0] + r * np.cos(th), M.c[1] + r * np.sin(th)
    return M(q1, q2)


def _jac_arr(M, q1, q2):
    if isinstance(M, AnnulusMap):
        th = M.t0 + q1 * M.dt
        r = M.r0 + q2 * (M.r1 - M.r0)
        dr = M.r1 - M.r0
        return (-r * M.dt * np.sin(th), dr * np.cos(th), r * M.dt * np.cos(th), dr * np.sin(th))
    if isinstance(M, AffineMap):
        J = M.jacobian(0.0, 0.0)
        z = np.zeros_like(np.asarray(q1, dtype=np.float64))
        return tuple(z + v for v in J)
    return M.jacobian(q1, q2)


def _invert_arr(M, X, Y, s1, s2, tol=1e-10, max_iter=50):
    """Mapping.invert for arrays of points: (ok, q1, q2)"""
    n = X.shape[0]
    if isinstance(M, AffineMap):
        a, b, c, d = M.jacobian(0.0, 0.0)
        if abs(a * d - b * c) < 1e-300:
            return np.zeros(n, bool), X * 0, Y * 0
        ia, ib, ic, id_ = _inv((a, b, c, d))
        vx, vy = X - M.o[0], Y - M.o[1]
        return np.ones(n, bool), ia * vx + ib * vy, ic * vx + id_ * vy
    if isinstance(M, AnnulusMap):
        dx, dy = X - M.c[0], Y - M.c[1]
        r = np.hypot(dx, dy)
        ok = ~(r < 1e-300)
        q2 = (r - M.r0) / (M.r1 - M.r0)
        th = np.arctan2(dy, dx)
        q1 = (th - M.t0) / M.dt
        period = 2 * math.pi / abs(M.dt)
        t = (q1 - s1) / period
        q1 = q1 - period * (np.sign(t) * np.floor(np.abs(t) + 0.5))
        return ok, q1, q2
    q1, q2 = s1.astype(np.float64).copy(), s2.astype(np.float64).copy()
    mx, my = _map_arr(M, q1, q2)
    res = np.hypot(mx - X, my - Y)
    active = np.ones(n, bool)   # still iterating
    failed = np.zeros(n, bool)
    for _ in range(max_iter):
        active &= ~(res <= tol)
        if not active.any():
            break
        idx = np.nonzero(active)[0]
        a, b, c, d = _jac_arr(M, q1[idx], q2[idx])
        det = a * d - b * c
        sing = np.abs(det) < 1e-300
        ia, ib, ic, id_ = d / det, -b / det, -c / det, a / det
        mx, my = _map_arr(M, q1[idx], q2[idx])
        vx, vy = X[idx] - mx, Y[idx] - my
        dq1, dq2 = ia * vx + ib * vy, ic * vx + id_ * vy
        step = np.ones(idx.size)
        done = sing.copy()
        for h in range(8):
            qn1, qn2 = q1[idx] + step * dq1, q2[idx] + step * dq2
            nx, ny = _map_arr(M, qn1, qn2)
            rn = np.hypot(nx - X[idx], ny - Y[idx])
            take = ~done & (rn < res[idx])
            q1[idx[take]], q2[idx[take]], res[idx[take]] = qn1[take], qn2[take], rn[take]
            done |= take
            step = np.where(done, step, step * 0.5)
        stalled = ~done
        fail_idx = idx[sing | stalled]
        failed[fail_idx] = True
        active[fail_idx] = False
    ok = ~failed & (res <= tol)
    return ok, q1, q2


def _contains_arr(p: Patch, X, Y, margin):
    """Patch.contains for arrays of points: (ok, q1, q2)"""
    ns = 9
    samp = [(a / ns, b / ns) for a in range(ns + 1) for b in range(ns + 1)
            if not (p.kind == C1 and a / ns < 0.5 and b / ns < 0.5)]
    sx = np.array([p.map(q1, q2)[0] for q1, q2 in samp])
    sy = np.array([p.map(q1, q2)[1] for q1, q2 in samp])
    best = np.full(X.shape[0], 1e300)
    bq1 = np.full(X.shape[0], 0.5)
    bq2 = np.full(X.shape[0], 0.5)
    for k, (q1, q2) in enumerate(samp):
        dd = np.hypot(sx[k] - X, sy[k] - Y)
        better = dd < best
        best = np.where(better, dd, best)
        bq1 = np.where(better, q1, bq1)
        bq2 = np.where(better, q2, bq2)
    ok, q1, q2 = _invert_arr(p.map, X, Y, bq1, bq2)
    mx, my = _map_arr(p.map, q1, q2)
    ok &= ~(np.hypot(mx - X, my - Y) > 1e-8)
    lo, hi = -margin, 1.0 + margin
    if p.periodic1:
        ok &= ~((q2 < lo) | (q2 > hi))
    else:
        ok &= ~((q1 < lo) | (q1 > hi) | (q2 < lo) | (q2 > hi))
    if p.kind == C1:
        ok &= ~((q1 < 0.5 - margin) & (q2 < 0.5 - margin))
    return ok, q1, q2


def _raw_window_arr(p: Patch, sp: Subpatch, u, v, nf):
    band = 2.0 * p.nv
    eps = 1e-9

    def ramp(dist):
        t = np.minimum(np.maximum((dist - nf) / (band - nf), 0.0), 1.0)
        s = np.sin(0.5 * math.pi * t)
        return s * s

    w = np.ones(np.broadcast(u, v).shape)
    lo = np.where(v < sp.j_cut - eps, sp.i_cut, sp.i0).astype(np.float64)
    internal = np.ones(w.shape, bool)
    if not p.periodic1 and p.sides[0].on_gamma:
        internal &= ~(lo == 0)
    if p.kind == C1:
        sel = (lo == p.i_corner) & (v < p.j_corner - eps)
        internal = np.where(sel, not p.wall_q1.on_gamma, internal)
    w = np.where(internal, w * ramp(u - lo), w)
    if not (not p.periodic1 and sp.i1 == p.np1 - 1 and p.sides[1].on_gamma):
        w = w * ramp(sp.i1 - u)
    lo = np.where(u < sp.i_cut - eps, sp.j_cut, sp.j0).astype(np.float64)
    internal = np.ones(w.shape, bool)
    if p.sides[2].on_gamma:
        internal &= ~(lo == 0)
    if p.kind == C1:
        sel = (lo == p.j_corner) & (u < p.i_corner - eps)
        internal = np.where(sel, not p.wall_q2.on_gamma, internal)
    w = np.where(internal, w * ramp(v - lo), w)
    if not (sp.j1 == p.np2 - 1 and p.sides[3].on_gamma):
        w = w * ramp(sp.j1 - v)
    return w


def _place_arr(p: Patch, sp: Subpatch, u, v, eps):
    u = np.array(u, dtype=np.float64, copy=True)
    if p.periodic1:
        np1 = float(p.np1)
        while True:
            m = u < sp.i0 - eps
            if not m.any():
                break
            u[m] += np1
        while True:
            m = u > sp.i1 + eps
            if not m.any():
                break
            u[m] -= np1
    ok = ~((u < sp.i0 - eps) | (u > sp.i1 + eps) | (v < sp.j0 - eps) | (v > sp.j1 + eps))
    ok &= ~((u < sp.i_cut - eps) & (v < sp.j_cut - eps))
    return ok, u


def _init_subpatch_data_fast(p: Patch, sp: Subpatch, nf: int, bcs: dict) -> SubData:
    ni, nj = sp.ni, sp.nj
    mask = fringe_mask(p, sp, nf)
    I, J = np.meshgrid(np.arange(sp.i0, sp.i1 + 1), np.arange(sp.j0, sp.j1 + 1))
    valid = mask != 0
    q1, q2 = I * p.h1, J * p.h2
    M = p.map
    x, y = _map_arr(M, q1, q2)
    a, b, c, dd = _jac_arr(M, q1, q2)
    det = a * dd - b * c
    ia, ib, ic, id_ = dd / det, -b / det, -c / det, a / det
    ax, ay = _map_arr(M, q1 + p.h1, q2)
    bx, by = _map_arr(M, q1 - p.h1, q2)
    cx, cy = _map_arr(M, q1, q2 + p.h2)
    dx, dy = _map_arr(M, q1, q2 - p.h2)
    h1p = np.maximum(np.hypot(ax - x, ay - y), np.hypot(x - bx, y - by))
    h2p = np.maximum(np.hypot(cx - x, cy - y), np.hypot(x - dx, y - dy))
    z = lambda arr: np.where(valid, arr, 0.0)  # noqa: E731
    base = init_subpatch_data_lines(p, sp, bcs)
    l_cut = sp.i_cut > sp.i0 and sp.j_cut > sp.j0
    return SubData(sp, p.index, ni, nj, p.h1, p.h2, sp.i_cut - sp.i0 if l_cut else 0,
                   sp.j_cut - sp.j0 if l_cut else 0, mask, z(x), z(y), z(ia), z(ic), z(ib), z(id_),
                   z(np.minimum(h1p, h2p)), z(np.maximum(h1p, h2p)), np.zeros((nj, ni)), *base, z(np.abs(det)))


def init_subpatch_data_lines(p: Patch, sp: Subpatch, bcs: dict):
    """the resolved line-end BCs of init_subpatch_data (rows lo, hi; cols lo, hi)"""
    def resolve(axis, line, high):
        internal, side = classify_end(p, sp, axis, line, high)
        if internal or side is None:
            return None
        if side.tag not in bcs:
            raise ValueError(f"no boundary condition for side tag '{side.tag}'")
        bc = bcs[side.tag]
        return (bc.kind, tuple(bc.state), bc.pressure)

    return ([resolve(0, j, False) for j in range(sp.j0, sp.j1 + 1)],
            [resolve(0, j, True) for j in range(sp.j0, sp.j1 + 1)],
            [resolve(1, i, False) for i in range(sp.i0, sp.i1 + 1)],
            [resolve(1, i, True) for i in range(sp.i0, sp.i1 + 1)])


def _check_min_overlap_fast(patches: list, nv: int):
    depth = 2 * nv + 1
    orphans = []
    for pi, p in enumerate(patches):
        pts = []
        if not p.periodic1:
            if not p.sides[0].on_gamma:
                pts += [(0, i, j) for j in range(p.np2) for i in range(min(depth, p.np1))]
            if not p.sides[1].on_gamma:
                pts += [(1, i, j) for j in range(p.np2) for i in range(max(0, p.np1 - depth), p.np1)]
        if not p.sides[2].on_gamma:
            pts += [(2, i, j) for i in range(p.np1) for j in range(min(depth, p.np2))]
        if not p.sides[3].on_gamma:
            pts += [(3, i, j) for i in range(p.np1) for j in range(max(0, p.np2 - depth), p.np2)]
        pts = [t for t in pts if p.lattice_valid(t[1], t[2])]
        if not pts:
            continue
        arr = np.array(pts)
        X, Y = _map_arr(p.map, arr[:, 1] * p.h1, arr[:, 2] * p.h2)
        covered = np.zeros(len(pts), bool)
        for po, p2 in enumerate(patches):
            if po == pi:
                continue
            idx = np.nonzero(~covered)[0]
            if idx.size == 0:
                break
            ok, _, _ = _contains_arr(p2, X[idx], Y[idx], 1e-9)
            covered[idx[ok]] = True
        for k in np.nonzero(~covered)[0]:
            orphans.append((pi, int(arr[k, 0]), int(arr[k, 1]), int(arr[k, 2]), (float(X[k]), float(Y[k]))))
    if orphans:
        lines = [f"FAIL: {len(orphans)} orphan layer points"]
        lines += [f"  patch {a} side {b} ({i},{j}) at ({x[0]:g},{x[1]:g})" for a, b, i, j, x in orphans[:8]]
        raise DecompositionError("minimum-overlap check failed:\n" + "\n".join(lines))
    _check_c1_corners(patches)  # the S-C1 corner rule (few points: scalar path)


def _check_c1_corners(patches):
    fails = []
    for p in patches:
        if p.kind != C1:
            continue
        corner = p.map(0.5, 0.5)
        reached = False
        for ps in patches:
            if ps.kind != S:
                continue
            q = ps.contains(corner, 1e-7)
            if q is None:
                continue
            tol = 1e-6
            if ((ps.sides[0].on_gamma and abs(q[0]) < tol) or (ps.sides[1].on_gamma and abs(q[0] - 1) < tol)
                    or (ps.sides[2].on_gamma and abs(q[1]) < tol) or (ps.sides[3].on_gamma and abs(q[1] - 1) < tol)):
                reached = True
                break
        if not reached:
            fails.append(f"C1 patch {p.index}: no S patch reaches its corner point")
    if fails:
        raise DecompositionError("minimum-overlap check failed:\nFAIL: 0 orphan layer points\n  " + "\n  ".join(fails))


def _stencil_ok(mask):
    """ok[sj, si]: the 6x6 block at (si, sj) is all interior (mask == 1)"""
    m = (mask == 1).astype(np.int32)
    c = np.zeros((m.shape[0] + 1, m.shape[1] + 1), np.int64)
    c[1:, 1:] = m.cumsum(0).cumsum(1)
    nj, ni = m.shape
    if nj < 6 or ni < 6:
        return np.zeros((max(nj - 5, 0), max(ni - 5, 0)), bool)
    s = c[6:, 6:] - c[:-6, 6:] - c[6:, :-6] + c[:-6, :-6]
    return s == 36


def _lagrange_arr(t, origin):
    w = []
    for a in range(6):
        num = np.ones_like(t)
        den = 1.0
        for b in range(6):
            if a == b:
                continue
            num = num * (t - (origin + b))
            den *= float(a - b)
        w.append(num / den)
    return np.stack(w, axis=-1)


def _build_interp_arr(ds: SubData, okst, u, v, slack):
    """build_interp (src/runtime.cpp:115-146) for arrays of points of one donor:
    (found, si0, sj0, wx, wy)"""
    sp2 = ds.sp
    tu, tv = u - sp2.i0, v - sp2.j0
    bi = np.floor(tu).astype(np.int64) - 2
    bj = np.floor(tv).astype(np.int64) - 2
    n = u.shape[0]
    best_pen = np.full(n, 1e300)
    bsi = np.full(n, -1, np.int64)
    bsj = np.full(n, -1, np.int64)
    for dj in range(-4, 5):
        for di in range(-4, 5):
            si, sj = bi + di, bj + dj
            inb = (si >= 0) & (si + 5 < ds.ni) & (sj >= 0) & (sj + 5 < ds.nj)
            out_u = np.maximum(np.maximum(0.0, si - tu), tu - (si + 5))
            out_v = np.maximum(np.maximum(0.0, sj - tv), tv - (sj + 5))
            cand = inb & ~(out_u > slack) & ~(out_v > slack)
            ok = np.zeros(n, bool)
            ci = np.nonzero(cand)[0]
            ok[ci] = okst[sj[ci], si[ci]]
            pen = out_u + out_v + 0.01 * (abs(di) + abs(dj))
            take = ok & (pen < best_pen)
            best_pen = np.where(take, pen, best_pen)
            bsi = np.where(take, si, bsi)
            bsj = np.where(take, sj, bsj)
    found = bsi >= 0
    wx = _lagrange_arr(tu, bsi.astype(np.float64))
    wy = _lagrange_arr(tv, bsj.astype(np.float64))
    return found, bsi, bsj, wx, wy


def _build_plan_fast(patches: list, subs: list, nf: int) -> Plan:
    by_gid = {d.sp.global_id: d for d in subs}
    boxes = {}
    for d in subs:
        valid = d.mask != 0
        b = boxes.setdefault(d.patch, [1e300, -1e300, 1e300, -1e300])
        b[0], b[1] = min(b[0], float(d.x[valid].min())), max(b[1], float(d.x[valid].max()))
        b[2], b[3] = min(b[2], float(d.y[valid].min())), max(b[3], float(d.y[valid].max()))
    margin = {p.index: 2.0 * max(p.max_spacing()) for p in patches}
    okst = {d.sp.global_id: _stencil_ok(d.mask) for d in subs}
    sol_c, vis_c, sol_i, vis_i = [], [], [], []
    for d in subs:
        p = patches[d.patch]
        sp = d.sp
        gid = sp.global_id
        # the recipient points in the reference's order (rows, then along the row)
        jl, il = np.nonzero(d.mask != 0)
        I, J = (il + sp.i0).astype(np.float64), (jl + sp.j0).astype(np.float64)
        dst = jl * d.ni + il
        X, Y = d.x[jl, il], d.y[jl, il]
        n = dst.size
        w_own = _raw_window_arr(p, sp, I, J, nf)
        slots = []  # contributors in the reference's order: (copy, sub, ok, u, v, w, src)
        for sp2 in p.subpatches:
            if sp2.global_id == gid:
                continue
            ok, u = _place_arr(p, sp2, I, J, 1e-9)
            if not ok.any():
                continue
            v = J
            i2 = np.sign(u) * np.floor(np.abs(u) + 0.5)
            j2 = np.sign(v) * np.floor(np.abs(v) + 0.5)
            src = ((j2 - sp2.j0) * sp2.ni + (i2 - sp2.i0)).astype(np.int64)
            w = np.where(ok, _raw_window_arr(p, sp2, u, v, nf), 0.0)
            slots.append((True, sp2.global_id, ok, u, v, w, src))
        for p2 in patches:
            if p2.index == p.index:
                continue
            bb, m = boxes[p2.index], margin[p2.index]
            inbox = ~((X < bb[0] - m) | (X > bb[1] + m) | (Y < bb[2] - m) | (Y > bb[3] + m))
            idx = np.nonzero(inbox)[0]
            if idx.size == 0:
                continue
            okc, q1, q2 = _contains_arr(p2, X[idx], Y[idx], 1e-9)
            uu = np.zeros(n)
            vv = np.zeros(n)
            has = np.zeros(n, bool)
            has[idx[okc]] = True
            uu[idx] = q1 / p2.h1
            vv[idx] = q2 / p2.h2
            for sp2 in p2.subpatches:
                ok, u = _place_arr(p2, sp2, uu, vv, 1e-7)
                ok &= has
                if not ok.any():
                    continue
                w = np.where(ok, _raw_window_arr(p2, sp2, u, vv, nf), 0.0)
                slots.append((False, sp2.global_id, ok, u, vv, w, None))
        denom = w_own.copy()
        for s_ in slots:
            denom = np.where(s_[2], denom + s_[5], denom)
        if not (denom > 1e-14).all():
            k = int(np.nonzero(~(denom > 1e-14))[0][0])
            raise DecompositionError(f"window partition vanishes at ({X[k]:f}, {Y[k]:f}), subpatch {gid}")
        d.w_norm[jl, il] = w_own / denom
        for copy, sub, ok, u, v, w, src in slots:
            wn = w / denom
            sel = ok & ~(wn <= 1e-15)
            if not sel.any():
                continue
            k = np.nonzero(sel)[0]
            if copy:
                vis_c.append((np.full(k.size, gid), dst[k], np.full(k.size, sub), src[k], wn[k]))
            else:
                ds = by_gid[sub]
                found, si, sj, wx, wy = _build_interp_arr(ds, okst[sub], u[k], v[k], 2.5)
                if not found.all():
                    kk = k[np.nonzero(~found)[0][0]]
                    raise DecompositionError(f"no admissible viscosity stencil in donor subpatch {sub} for "
                                             f"({X[kk]:f}, {Y[kk]:f})")
                vis_i.append((np.full(k.size, gid), dst[k], np.full(k.size, sub), si, sj, wx, wy, wn[k]))
        # solution entries of the fringe points
        fringe = d.mask[jl, il] == 2
        best_w = np.full(n, -1.0)
        best_sub = np.full(n, -1, np.int64)
        best_src = np.zeros(n, np.int64)
        for copy, sub, ok, u, v, w, src in slots:
            if not copy:
                continue
            dm = by_gid[sub].mask.reshape(-1)
            good = ok & fringe
            gi = np.nonzero(good)[0]
            good[gi] = dm[src[gi]] == 1
            take = good & ((best_sub < 0) | (w > best_w))
            best_w = np.where(take, w, best_w)
            best_sub = np.where(take, sub, best_sub)
            best_src = np.where(take, src, best_src)
        hc = fringe & (best_sub >= 0)
        k = np.nonzero(hc)[0]
        if k.size:
            sol_c.append((np.full(k.size, gid), dst[k], best_sub[k], best_src[k]))
        need = np.nonzero(fringe & (best_sub < 0))[0]
        if need.size:
            cands = [(s_[1], s_[2], s_[3], s_[4], s_[5]) for s_ in slots if not s_[0]]
            done = np.zeros(need.size, bool)
            res = {}
            # candidates by raw window, largest first (stable on ties)
            W = np.stack([c[4][need] for c in cands], axis=1) if cands else np.zeros((need.size, 0))
            OK = np.stack([c[1][need] for c in cands], axis=1) if cands else np.zeros((need.size, 0), bool)
            order = np.argsort(-np.where(OK, W, -np.inf), axis=1, kind="stable")
            for rank in range(len(cands)):
                todo = np.nonzero(~done)[0]
                if todo.size == 0:
                    break
                ci = order[todo, rank]
                for cidx in np.unique(ci):
                    sel = todo[ci == cidx]
                    sel = sel[OK[sel, cidx]]
                    if sel.size == 0:
                        continue
                    sub, ok, u, v, w = cands[cidx]
                    pts = need[sel]
                    found, si, sj, wx, wy = _build_interp_arr(by_gid[sub], okst[sub], u[pts], v[pts], 0.5)
                    for q, f in enumerate(found):
                        if f:
                            res[int(sel[q])] = (sub, int(si[q]), int(sj[q]), wx[q], wy[q])
                    done[sel[found]] = True
            if not done.all():
                kk = need[np.nonzero(~done)[0][0]]
                raise DecompositionError(f"orphan fringe point at ({X[kk]:f}, {Y[kk]:f}), subpatch {gid}")
            keys = sorted(res)
            sol_i.append((np.full(len(keys), gid), dst[need[keys]],
                          np.array([res[q][0] for q in keys]), np.array([res[q][1] for q in keys]),
                          np.array([res[q][2] for q in keys]), np.array([res[q][3] for q in keys]),
                          np.array([res[q][4] for q in keys])))
    i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731

    def cat(parts, k, dt):
        return np.concatenate([np.asarray(x[k], dtype=dt) for x in parts]) if parts else np.zeros(0, dt)

    def cat6(parts, k):
        return np.concatenate([np.asarray(x[k], dtype=np.float64).reshape(-1, 6) for x in parts]) if parts \
            else np.zeros((0, 6))

    # viscosity entries were gathered contributor by contributor; the
    # reference lists them point by point, contributors in order: a stable
    # sort by (recipient, point) restores that order
    def point_major(parts):
        if not parts:
            return parts
        cols = [np.concatenate([np.asarray(x[k]) for x in parts]) for k in range(len(parts[0]))]
        o = np.lexsort((cols[1], cols[0]))
        return [tuple(c[o] for c in cols)]

    vis_c = point_major(vis_c)
    vis_i = point_major(vis_i)
    return Plan(i32(cat(sol_c, 0, np.int64)), i32(cat(sol_c, 1, np.int64)), i32(cat(sol_c, 2, np.int64)),
                i32(cat(sol_c, 3, np.int64)), i32(cat(vis_c, 0, np.int64)), i32(cat(vis_c, 1, np.int64)),
                i32(cat(vis_c, 2, np.int64)), i32(cat(vis_c, 3, np.int64)), cat(vis_c, 4, np.float64),
                sol_interps=dict(dst_sub=i32(cat(sol_i, 0, np.int64)), dst=i32(cat(sol_i, 1, np.int64)),
                                 src_sub=i32(cat(sol_i, 2, np.int64)), si0=i32(cat(sol_i, 3, np.int64)),
                                 sj0=i32(cat(sol_i, 4, np.int64)), wx=cat6(sol_i, 5), wy=cat6(sol_i, 6)),
                visc_interps=dict(dst_sub=i32(cat(vis_i, 0, np.int64)), dst=i32(cat(vis_i, 1, np.int64)),
                                  src_sub=i32(cat(vis_i, 2, np.int64)), si0=i32(cat(vis_i, 3, np.int64)),
                                  sj0=i32(cat(vis_i, 4, np.int64)), wx=cat6(vis_i, 5), wy=cat6(vis_i, 6),
                                  w=cat(vis_i, 7, np.float64)))


# ---------------------------------------------------------------------------
# fcs-mesh v1 JSON (DomainDecomposition::to_json / from_json,
# src/geometry.cpp:573-629; curves and mappings :17-31, :71-135): the
# reference's mesh file, read and written with the same keys and values, so a
# decomposition moves between the two codes. Python's float repr and
# nlohmann::json both print the shortest round-trip form, so the numbers
# survive either way exactly.

MESH_FORMAT, MESH_VERSION = "fcs-mesh", 1


def curve_to_json(c) -> dict:
    if isinstance(c, Segment):
        return {"type": "segment", "a": list(c.a), "b": list(c.b)}
    if isinstance(c, CircularArc):
        return {"type": "arc", "center": list(c.c), "r": c.r, "theta0": c.t0, "theta1": c.t1}
    raise GeometryError(f"curve has no fcs-mesh form: {type(c).__name__}")


def curve_from_json(j: dict):
    t = j["type"]
    if t == "segment":
        return Segment(tuple(j["a"]), tuple(j["b"]))
    if t == "arc":
        return CircularArc(tuple(j["center"]), j["r"], j["theta0"], j["theta1"])
    raise GeometryError("unknown curve type: " + t)


def mapping_to_json(M) -> dict:
    if isinstance(M, AffineMap):
        return {"type": "affine", "o": list(M.o), "e1": list(M.e1), "e2": list(M.e2)}
    if isinstance(M, AnnulusMap):
        return {"type": "annulus", "center": list(M.c), "r0": M.r0, "r1": M.r1, "theta0": M.t0,
                "theta_extent": M.dt}
    if isinstance(M, BilinearMap):
        a, b, c, d = M.a, M.b, M.c, M.d
        p10 = (a[0] + b[0], a[1] + b[1])
        p01 = (a[0] + c[0], a[1] + c[1])
        p11 = (((a[0] + b[0]) + c[0]) + d[0], ((a[1] + b[1]) + c[1]) + d[1])
        return {"type": "bilinear", "p00": list(a), "p10": list(p10), "p01": list(p01), "p11": list(p11)}
    if isinstance(M, CurveSumMap):
        return {"type": "curve_sum", "a": curve_to_json(M.A), "b": curve_to_json(M.B), "corner": list(M.C)}
    raise GeometryError(f"mapping has no fcs-mesh form: {type(M).__name__}")


def mapping_from_json(j: dict) -> Mapping:
    t = j["type"]
    if t == "affine":
        return AffineMap(tuple(j["o"]), tuple(j["e1"]), tuple(j["e2"]))
    if t == "annulus":
        return AnnulusMap(tuple(j["center"]), j["r0"], j["r1"], j["theta0"], j["theta_extent"])
    if t == "bilinear":
        return BilinearMap(tuple(j["p00"]), tuple(j["p10"]), tuple(j["p01"]), tuple(j["p11"]))
    if t == "curve_sum":
        return CurveSumMap(curve_from_json(j["a"]), curve_from_json(j["b"]), tuple(j["corner"]))
    raise GeometryError("unknown mapping type: " + t)


def mesh_to_json(patches: list, nv: int, n0: int = 83, n1: int = 43, nf: int = 5) -> dict:
    """DomainDecomposition::to_json (src/geometry.cpp:573-594) of subdivided
    patches; nv, n0, n1, nf are the decomposition's fields."""
    jp = []
    for p in patches:
        pj = {"kind": p.kind, "mapping": mapping_to_json(p.map), "r": p.r, "s": p.s, "n_cell": p.n_cell,
              "nv": p.nv, "periodic1": bool(p.periodic1),
              "sides": [{"on_gamma": bool(sd.on_gamma), "tag": sd.tag} for sd in p.sides]}
        if p.kind == C1:
            pj["wall_q1_tag"] = p.wall_q1.tag
            pj["wall_q2_tag"] = p.wall_q2.tag
        pj["subpatches"] = [[sp.i0, sp.i1, sp.j0, sp.j1, sp.i_cut, sp.j_cut] for sp in p.subpatches]
        jp.append(pj)
    return {"format": MESH_FORMAT, "version": MESH_VERSION, "nv": nv, "n0": n0, "n1": n1, "nf": nf,
            "patches": jp}


def mesh_from_json(j: dict):
    """DomainDecomposition::from_json (src/geometry.cpp:596-629): patches
    rebuilt from their mapping, sides and subdivision parameters (the
    subpatch table is only checked for its length, as in the reference).
    Returns (patches, {"nv", "n0", "n1", "nf"})."""
    if j.get("format", "") != MESH_FORMAT or j.get("version", 0) != MESH_VERSION:
        raise GeometryError("mesh file: unknown format/version")
    patches = []
    for idx, pj in enumerate(j["patches"]):
        kind = pj["kind"]
        if kind not in (S, C1, C2, I):
            raise GeometryError("unknown patch kind: " + str(kind))
        sides = [SideInfo(bool(pj["sides"][k]["on_gamma"]), pj["sides"][k]["tag"]) for k in range(4)]
        p = Patch(kind, mapping_from_json(pj["mapping"]), sides, periodic1=bool(pj.get("periodic1", False)),
                  index=idx)
        if kind == C1:
            p.wall_q1 = SideInfo(True, pj.get("wall_q1_tag", "wall"))
            p.wall_q2 = SideInfo(True, pj.get("wall_q2_tag", "wall"))
            subdivide_L(p, pj["r"], pj["n_cell"], pj["nv"])
        else:
            subdivide_Q(p, pj["r"], pj["s"], pj["n_cell"], pj["nv"])
        if "subpatches" in pj and len(pj["subpatches"]) != len(p.subpatches):
            raise GeometryError("mesh file: subpatch table does not match r/s parameters")
        patches.append(p)
    gid = 0
    for p in patches:
        for sp in p.subpatches:
            sp.patch_index = p.index
            sp.global_id = gid
            gid += 1
    return patches, {k: j[k] for k in ("nv", "n0", "n1", "nf")}


def save_mesh(path: str, patches: list, nv: int, n0: int = 83, n1: int = 43, nf: int = 5):
    import json
    with open(path, "w") as f:
        json.dump(mesh_to_json(patches, nv, n0, n1, nf), f, indent=2)


def load_mesh(path: str):
    import json
    with open(path) as f:
        return mesh_from_json(json.load(f))
