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

* mappings (affine, annulus, bilinear, curve sum of segments) and their
  Jacobians / inversion        include/fcs/geometry.hpp:57-136, src/geometry.cpp:35-99
* Patch.contains / max_spacing  src/geometry.cpp:161-208
* subdivide_Q / subdivide_L     src/geometry.cpp:210-334
* classify_end / fringe_mask    src/geometry.cpp:444-495
* check_min_overlap             src/geometry.cpp:502-560
* raw_window                    src/viscosity.cpp:253-293
* init_subpatch_data            src/subpatch_data.cpp:69-154
* build_plan                    src/runtime.cpp:57-274

Scalar arithmetic follows the reference's operation order (Python floats are
IEEE doubles and the reference is compiled without FMA contraction), so the
geometry and the plan match the reference's to round-off; tests/
test_multipatch.py checks them against the compiled reference.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .geometry import BcSpec, DecompositionError, Plan, SideInfo  # noqa: F401  (re-exported)


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


def build_c1_patch(ellA: Segment, ellB: Segment, corner, wall_tag="wall"):
    """src/geometry.cpp:351-369 (without its Jacobian sign sweep)"""
    return Patch(C1, CurveSumMap(ellA, ellB, corner), [SideInfo() for _ in range(4)],
                 wall_q1=SideInfo(True, wall_tag), wall_q2=SideInfo(True, wall_tag))


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


def init_subpatch_data(p: Patch, sp: Subpatch, nf: int, bcs: dict) -> SubData:
    """src/subpatch_data.cpp:69-154"""
    ni, nj = sp.ni, sp.nj
    mask = fringe_mask(p, sp, nf)
    sh = (nj, ni)
    x, y = np.zeros(sh), np.zeros(sh)
    iq1x, iq2x, iq1y, iq2y = (np.zeros(sh) for _ in range(4))
    hmin, hmax = np.zeros(sh), np.zeros(sh)
    M = p.map
    for j in range(sp.j0, sp.j1 + 1):
        for i in range(sp.i0, sp.i1 + 1):
            if not sp.valid(i, j):
                continue
            il, jl = i - sp.i0, j - sp.j0
            q1, q2 = i * p.h1, j * p.h2
            xp = M(q1, q2)
            x[jl, il], y[jl, il] = xp
            Ji = _inv(M.jacobian(q1, q2))
            iq1x[jl, il], iq2x[jl, il], iq1y[jl, il], iq2y[jl, il] = Ji[0], Ji[2], Ji[1], Ji[3]
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
                   [resolve(1, i, True) for i in range(sp.i0, sp.i1 + 1)])


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


def build_decomposition(patches: list, bcs: dict, nv: int, nf: int = 5, validate_overlap: bool = True):
    """Engine::init's geometry part (src/runtime.cpp:293-305): ids, overlap
    check, SubpatchData, plan. Patches must already be subdivided."""
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
        check_min_overlap(patches, nv)
    subs = [init_subpatch_data(p, sp, nf, bcs) for p in patches for sp in p.subpatches]
    plan = build_plan(patches, subs, nf)
    return MultiPatchDecomposition(patches, subs, plan, bcs, nf)
