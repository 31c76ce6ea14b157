"""Synthetic BASELINE workloads (host side): decompositions + seeded initial data.

No dataset is involved: BASELINE.json's configurations are synthetic, and the
seeded generators here produce them with the stated shapes and value ranges.
Random numbers use splitmix64 with uniform() = (next() >> 11) * 2^-53, the
same generator as the reference's private Rng (src/viscosity.cpp:300-313).

* ``fc_lines_config1``  config 1: 4096 lines of N=256 on [0,1],
  f = sum_k a_k sin(w_k x + phi_k) + sum_j b_j x^j.
* ``riemann_quadrants`` config 2: one 512x512 I patch on [0,1]^2, four-quadrant
  Riemann data split at (0.5, 0.5), zero_normal_all sides (as riemann4,
  src/problems.cpp:57-81), CFL 0.5.
* ``vortex_tiles``      config 5: one I patch tiled by 256x256 subpatches
  (subdivide_Q(r, s, 238, 9): 19-point intra-patch overlap), isentropic vortex
  plus 1e-3 seeded noise on the primitives.
* ``cylinder_flow``     config 3: Mach 3 flow past a unit cylinder in
  [-4, 12] x [-6, 6]: a periodic annulus (2048 x 147) around the body and four
  Cartesian I patches of 256 x 256 subpatches around it (multipatch.py).
* ``step_flow``         config 4: Mach 3 forward-facing step; C1 corner patch
  (L-shaped subpatch), S and I patches (multipatch.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import geometry as G

GAMMA = 1.4
MASK64 = (1 << 64) - 1


class SplitMix64:
    """src/viscosity.cpp:300-313"""

    def __init__(self, seed: int):
        self.s = seed & MASK64 if seed else 0x9E3779B97F4A7C15

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self, a=0.0, b=1.0) -> float:
        return a + (b - a) * ((self.next() >> 11) * 2.0 ** -53)


def splitmix_uniform_array(seeds: np.ndarray, k: int) -> np.ndarray:
    """k uniforms in [0,1) per seed (vectorised splitmix64, uint64 wraparound)."""
    s = seeds.astype(np.uint64).copy()
    out = np.empty(seeds.shape + (k,))
    with np.errstate(over="ignore"):
        for j in range(k):
            s = s + np.uint64(0x9E3779B97F4A7C15)
            z = s.copy()
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            out[..., j] = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return out


def conservative(rho, u, v, p):
    """src/euler.cpp:10-12"""
    return np.stack(np.broadcast_arrays(rho, rho * u, rho * v, p / (GAMMA - 1.0) + 0.5 * rho * (u * u + v * v)))


def fc_lines_config1(n_lines=4096, n=256, seed=1):
    rng = SplitMix64(seed)
    x = np.arange(n) / (n - 1)
    f = np.zeros((n_lines, n))
    df = np.zeros((n_lines, n))
    for l in range(n_lines):
        for _ in range(4):
            a, w, ph = rng.uniform(-1, 1), rng.uniform(1, 20), rng.uniform(0, 2 * math.pi)
            f[l] += a * np.sin(w * x + ph)
            df[l] += a * w * np.cos(w * x + ph)
        b = [rng.uniform(-1, 1) for _ in range(4)]
        for j in range(4):
            f[l] += b[j] * x ** j
            if j:
                df[l] += j * b[j] * x ** (j - 1)
    return x, f, df


def riemann_quadrants(n=512, seed=2, nv=9):
    """BASELINE config 2 (n=512) or a smaller n for parity tests."""
    zero_normal = G.BcSpec(G.ZERO_NORMAL_ALL)
    dec = G.rect_decomposition((0.0, 0.0), 1.0, 1.0, 1, 1, n - 2 * nv, nv, [zero_normal] * 4)
    rng = SplitMix64(seed)
    q = [(rng.uniform(0.1, 1.5), rng.uniform(-0.75, 0.75), rng.uniform(-0.75, 0.75), rng.uniform(0.03, 1.5))
         for _ in range(4)]

    def ic(x, y):
        e = np.zeros((4,) + x.shape)
        quads = [(x >= 0.5) & (y >= 0.5), (x < 0.5) & (y >= 0.5), (x < 0.5) & (y < 0.5), (x >= 0.5) & (y < 0.5)]
        for k, m in enumerate(quads):
            e[:, m] = np.asarray(conservative(*q[k]), dtype=np.float64).reshape(4, 1)
        return e

    return dec, ic, {"cfl": 0.5, "quadrant_states": q}


def vortex_tiles(r=8, s=8, seed=5, n0=238, nv=9, noise=1e-3, beta=5.0):
    """BASELINE config 5: an (r x s) tiling of 256x256 subpatches (n0=238)."""
    zero_normal = G.BcSpec(G.ZERO_NORMAL_ALL)
    h = 1.0 / (n0 - 1)  # fixed spacing: each preliminary cell is a unit square
    lx = (r * (n0 - 1) + 2 * nv) * h
    ly = (s * (n0 - 1) + 2 * nv) * h
    dec = G.rect_decomposition((0.0, 0.0), lx, ly, r, s, n0, nv, [zero_normal] * 4)
    p = dec.patches[0]
    xc, yc = 0.5 * lx, 0.5 * ly
    R = 0.25 * min(lx, ly) / 2.0  # vortex radius scale

    def ic(x, y, I=None, J=None):
        dx, dy = (x - xc) / R, (y - yc) / R
        r2 = dx * dx + dy * dy
        f = beta / (2 * math.pi) * np.exp(0.5 * (1 - r2))
        u = -dy * f * 0.2
        v = dx * f * 0.2
        T = 1.0 - (GAMMA - 1.0) * (0.2 * beta) ** 2 / (8 * GAMMA * math.pi ** 2) * np.exp(1 - r2)
        rho = T ** (1.0 / (GAMMA - 1.0))
        pr = rho * T
        if noise and I is not None:
            lid = (I.astype(np.int64) * p.np2 + J.astype(np.int64)) + np.int64(seed) * np.int64(1 << 40)
            un = splitmix_uniform_array(lid, 4) * 2.0 - 1.0
            rho = rho * (1 + noise * un[..., 0])
            u = u + noise * un[..., 1]
            v = v + noise * un[..., 2]
            pr = pr * (1 + noise * un[..., 3])
        return conservative(rho, u, v, pr)

    return dec, ic, {"cfl": 0.5}


def rotated_channel(theta=0.3, r=2, s=1, n0=30, nv=9, mach=0.6):
    """A rotated affine channel (every metric term nonzero) with one side of
    each boundary-condition kind: W inflow, E outflow_pressure, S slip wall,
    N no-slip adiabatic wall; a smooth subsonic flow along the channel with a
    Gaussian density bump. Exercises the general stage passes and
    src/euler.cpp:105-165."""
    c, sn = math.cos(theta), math.sin(theta)
    L, H = 2.0, 1.0
    e1 = (L * c, L * sn)
    e2 = (-H * sn, H * c)
    rho0, p0 = 1.0, 1.0 / GAMMA
    u0 = mach * math.sqrt(GAMMA * p0 / rho0)
    inflow = tuple(float(v) for v in conservative(rho0, u0 * c, u0 * sn, p0))
    bcs = [G.BcSpec(G.INFLOW, inflow), G.BcSpec(G.OUTFLOW_PRESSURE, pressure=p0), G.BcSpec(G.SLIP_WALL),
           G.BcSpec(G.NOSLIP_ADIABATIC)]
    dec = G.affine_decomposition((0.0, 0.0), e1, e2, r, s, n0, nv, bcs)

    def ic(x, y):
        # channel coordinates
        xi = x * c + y * sn
        eta = -x * sn + y * c
        rho = rho0 * (1.0 + 0.2 * np.exp(-((xi - 0.8) ** 2 + (eta - 0.5) ** 2) / 0.02))
        return conservative(rho, u0 * c, u0 * sn, p0 * (rho / rho0) ** GAMMA)

    return dec, ic, {"cfl": 0.5, "e1": e1, "e2": e2, "kinds": [G.INFLOW, G.OUTFLOW_PRESSURE, G.SLIP_WALL,
                                                              G.NOSLIP_ADIABATIC], "inflow": inflow,
                     "pressure": p0}


def initial_state(dec, ic, sub):
    """Evaluate an IC on one subpatch (Engine::apply_ic, src/runtime.cpp:276-283)."""
    d = dec.subs[sub]
    try:
        I, J = np.meshgrid(np.arange(d.sp.i0, d.sp.i1 + 1), np.arange(d.sp.j0, d.sp.j1 + 1))
        return np.ascontiguousarray(ic(d.x, d.y, I, J))
    except TypeError:
        return np.ascontiguousarray(ic(d.x, d.y))


def cylinder_flow(full=True, fine=False, body="slip"):
    """BASELINE config 3 (multi-patch, curvilinear). The reference's own
    cylinder decomposition fails its overlap check, so
    the patches are laid out here: an annulus r in [1, 2.2] around the body
    (periodic q1, slip wall at r = 1; subdivide_Q(16, 1, 129, 9): 2048 x 147,
    SURVEY D4) and four Cartesian I patches covering the rest of
    [-4, 12] x [-6, 6] (inflow on the left, supersonic outflow on the right,
    slip walls at y = +-6) with 256 x 256 subpatches; free stream rho = 1.4,
    p = 1, u = 3 (Mach 3). full=False: the same layout at about a quarter of
    the resolution (0.70M points; ring 512 x 83, Cartesian 138 x 138).
    body="noslip": the body as the reference's flow-cylinder has it
    (noslip_adiabatic, src/problems.cpp:205) instead of a slip wall.
    fine=True: BASELINE's ~4M points -- the ring at 3072 x 147 and the
    Cartesian patches cut into 6, 36, 4 and 4 subpatches of 256 x 256 (the
    cells anisotropic where a patch side does not divide evenly)."""
    from . import multipatch as M
    SI = M.SideInfo
    ring = M.Patch(M.S, M.AnnulusMap((0.0, 0.0), 1.0, 2.2, -math.pi, 2 * math.pi),
                   [SI(), SI(), SI(True, "body"), SI()], periodic1=True)
    left = M.Patch(M.I, M.AffineMap((-4.0, -6.0), (2.8, 0.0), (0.0, 12.0)),
                   [SI(True, "in"), SI(), SI(True, "wall"), SI(True, "wall")])
    right = M.Patch(M.I, M.AffineMap((1.2, -6.0), (10.8, 0.0), (0.0, 12.0)),
                    [SI(), SI(True, "out"), SI(True, "wall"), SI(True, "wall")])
    top = M.Patch(M.I, M.AffineMap((-1.7, 1.2), (3.4, 0.0), (0.0, 4.8)), [SI(), SI(), SI(), SI(True, "wall")])
    bottom = M.Patch(M.I, M.AffineMap((-1.7, -6.0), (3.4, 0.0), (0.0, 4.8)), [SI(), SI(), SI(True, "wall"), SI()])
    patches = [ring, left, right, top, bottom]
    for k, p in enumerate(patches):
        p.index = k
    ring_r, ring_n0, n0 = (16, 129, 238) if full else (8, 65, 120)
    cuts = ((1, 5), (5, 5), (1, 2), (1, 2))
    if fine:
        ring_r, cuts = 24, ((1, 6), (6, 6), (2, 2), (2, 2))
    M.subdivide_Q(ring, ring_r, 1, ring_n0, 9)
    for p, (r, s) in zip((left, right, top, bottom), cuts):
        M.subdivide_Q(p, r, s, n0, 9)
    free = tuple(float(v) for v in conservative(1.4, 3.0, 0.0, 1.0))
    body_bc = M.BcSpec(M.SLIP_WALL) if body == "slip" else M.BcSpec(M.NOSLIP_ADIABATIC)
    bcs = {"in": M.BcSpec(M.INFLOW, free), "out": M.BcSpec(M.SUPERSONIC_OUTFLOW), "wall": M.BcSpec(M.SLIP_WALL),
           "body": body_bc}
    dec = M.build_decomposition(patches, bcs, 9, fast=True)

    def ic(x, y):
        return np.broadcast_to(np.asarray(free).reshape(4, 1, 1), (4,) + np.shape(x)).copy()

    return dec, ic, {"cfl": 0.5, "free_stream": free}



def step_flow(scale=1, cfl=0.25):
    """BASELINE config 4: Mach 3 flow over a forward-facing step in
    [0, 3] x [0, 1] (step of height 0.2 at x = 0.6). The reference's own
    corner-patch problems fail their overlap checks, so
    the layout is ours: a convex-corner C1 patch at the step's top (0.6, 0.2)
    (arms of 0.15 along the step top and face: one L-shaped subpatch at scale
    1), an S patch along the step top, a concave-corner C2 patch at the
    step's foot (0.6, 0) between the floor and the face, and two Cartesian I
    patches;
    inflow rho = 1.4, p = 1, u = 3 on the left, supersonic outflow on the
    right, slip walls. The I and S patches are split into 256 x 256
    subpatches (as config 5); scale k multiplies the cells per patch side
    (about 0.87M k^2 points; the C1 patch gets 2k cells of 60 points).
    CFL 0.25: the reference runs every problem with C1 patches at 0.25
    (src/problems.cpp:88,284)."""
    from . import multipatch as M
    SI = M.SideInfo
    c, a = (0.6, 0.2), 0.15
    c1 = M.build_c1_patch(M.Segment((c[0] + a, c[1]), (c[0] - a, c[1])),
                          M.Segment((c[0], c[1] - a), (c[0], c[1] + a)), c, "wall")
    left = M.Patch(M.I, M.AffineMap((0.0, 0.0), (0.57, 0.0), (0.0, 1.0)),
                   [SI(True, "in"), SI(), SI(True, "wall"), SI(True, "wall")])
    top = M.Patch(M.I, M.AffineMap((0.4, 0.26), (2.6, 0.0), (0.0, 0.74)),
                  [SI(), SI(True, "out"), SI(), SI(True, "wall")])
    s_top = M.Patch(M.S, M.AffineMap((0.6, 0.2), (2.4, 0.0), (0.0, 0.25)),
                    [SI(), SI(True, "out"), SI(True, "wall"), SI()])
    # concave corner at the step's foot (0.6, 0): a C2 patch between the
    # floor and the step face, both ending at the corner (walls on E and N)
    s_face = M.build_c2_patch(M.Segment((0.3, 0.0), (0.6, 0.0)), M.Segment((0.6, 0.2), (0.6, 0.0)), (0.6, 0.0),
                              "wall")
    patches = [c1, left, top, s_top, s_face]
    for k, p in enumerate(patches):
        p.index = k
    k = int(scale)
    M.subdivide_L(c1, 2 * k, 59, 9)
    for p, (r, s) in zip(patches[1:], ((1, 2), (5, 1), (4, 1), (1, 1))):
        M.subdivide_Q(p, r * k, s * k, 238, 9)  # 256 x 256 subpatches, as config 5
    free = tuple(float(v) for v in conservative(1.4, 3.0, 0.0, 1.0))
    bcs = {"in": M.BcSpec(M.INFLOW, free), "out": M.BcSpec(M.SUPERSONIC_OUTFLOW), "wall": M.BcSpec(M.SLIP_WALL)}
    dec = M.build_decomposition(patches, bcs, 9, fast=True)

    def ic(x, y):
        return np.broadcast_to(np.asarray(free).reshape(4, 1, 1), (4,) + np.shape(x)).copy()

    return dec, ic, {"cfl": cfl, "free_stream": free}
