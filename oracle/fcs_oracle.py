"""CPU restatement of the reference FC-SDNN time step -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the CUDA product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference legs
may import it; the product never routes through it.

Every function restates one reference function (file:line relative to
``/root/reference/proj``) in numpy, vectorised over lines/points but keeping
the reference's arithmetic order where that order is observable at the
parity tolerances (1e-11 per FC line, 1e-8 per solution):

* FC operator       -> src/fc_core.cpp:55-152 (blend matrix, 120-digit LSQ),
                       :190-206 (sizes/profiles), :221-238 (continuation),
                       :257-284 (derivative), :286-306 (filters)
* line sweeps       -> src/subpatch_data.cpp:9-67
* Euler physics     -> src/euler.cpp:10-12,16-101,105-180,182-221,223-236
* SDNN viscosity    -> src/viscosity.cpp:13-29,48-59,63-89,108-133,143-208,211-251
                       (ann and fallback classifier variants)
* superstep         -> src/runtime.cpp:327-454,482-511

The blend matrix is also generalised to Gram degree d (degree 2 reproduces
the reference exactly; degree 4 is the BASELINE config-1 operator that the
reference cannot build, SURVEY.md D1 -- that case is pinned analytically).

Parity pin: ``tests/test_oracle_pins.py`` checks this module against the
unmodified reference compiled into ``oracle/_ref`` (when present) and against
the committed fixtures in ``tests/golden`` produced from it.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

GAMMA = 1.4
# src/fc_core.cpp:27-29
K_OVERSAMPLE = 10
K_ZERO_WIDTH = 3
K_MODES = 15
# include/fcs/fc_core.hpp:11-15
ALPHA = 23.025850929940457
P_FILTER = 7
P_SMEAR = 2
# include/fcs/viscosity.hpp:51,72-74
ABS_FLOOR = 1e-4
VISC_C = (1.5, 1.0, 0.25, 0.0)
# include/fcs/euler.hpp:14-30
B0 = 0.391752226571890
A20, A21, B1 = 0.444370493651235, 0.555629506348765, 0.368410593050371
A30, A32, B2 = 0.620101851488403, 0.379898148511597, 0.251891774271694
A40, A43, B3 = 0.178079954393132, 0.821920045606868, 0.544974750228521
C2, C3, D3, C4, D4 = (0.517231671970585, 0.096059710526147, 0.063692468666290,
                      0.386708617503269, 0.226007483236906)

BC_INFLOW, BC_OUTFLOW_P, BC_SLIP, BC_NOSLIP, BC_SUPERSONIC, BC_ZERO_NORMAL = range(6)


class InvalidState(RuntimeError):
    """include/fcs/errors.hpp:32-39 (InvalidStateError)."""


# ---------------------------------------------------------------------------
# FC operator tables


def gram_basis(d: int):
    """Orthonormal Gram basis on points {0..d}, Gram-Schmidt in double
    (src/fc_core.cpp:88-112; the reference hard-codes d=2)."""
    n = d + 1
    q = [[float(i ** m) for i in range(n)] for m in range(n)]
    cf = [[1.0 if a == b else 0.0 for b in range(n)] for a in range(n)]
    for k in range(n):
        for p in range(k):
            dot = 0.0
            for i in range(n):
                dot += q[p][i] * q[k][i]
            for i in range(n):
                q[k][i] -= dot * q[p][i]
            for m in range(n):
                cf[k][m] -= dot * cf[p][m]
        nrm = 0.0
        for i in range(n):
            nrm += q[k][i] * q[k][i]
        nrm = math.sqrt(nrm)
        for i in range(n):
            q[k][i] /= nrm
        for m in range(n):
            cf[k][m] /= nrm
    return q, cf


_BLEND_CACHE: dict = {}


def blend_matrix(n_cont: int, d: int = 2) -> np.ndarray:
    """(n_cont-1) x (d+1) blend-to-zero matrix (src/fc_core.cpp:55-152).

    Trig least-squares fit by normal equations solved with partial pivoting at
    400 bits (the reference's mpfr_float_backend<120>), residual guard 1e-13.
    """
    key = (n_cont, d)
    if key in _BLEND_CACHE:
        return _BLEND_CACHE[key]
    import mpmath as mp

    ctx = mp.mp.clone()
    ctx.prec = 400
    mpf = ctx.mpf
    lam = mpf(2) * (d + n_cont + K_ZERO_WIDTH)
    twopi = 2 * ctx.pi
    n_match = K_OVERSAMPLE * d + 1
    n_zero = K_OVERSAMPLE * (K_ZERO_WIDTH - 1) + 1
    rows = n_match + n_zero
    cols = 2 * K_MODES + 1
    zs = [mpf(d) * i / (n_match - 1) for i in range(n_match)]
    zs += [mpf(d + n_cont) + mpf(K_ZERO_WIDTH - 1) * i / (n_zero - 1) for i in range(n_zero)]
    B = [[mpf(0)] * cols for _ in range(rows)]
    for r in range(rows):
        B[r][0] = mpf(1)
        for m in range(1, K_MODES + 1):
            arg = twopi * m * zs[r] / lam
            B[r][2 * m - 1] = ctx.cos(arg)
            B[r][2 * m] = ctx.sin(arg)
    G0 = [[mpf(0)] * cols for _ in range(cols)]
    for i in range(cols):
        for j in range(i, cols):
            s = mpf(0)
            for r in range(rows):
                s += B[r][i] * B[r][j]
            G0[i][j] = s
            G0[j][i] = s
    pv, coef = gram_basis(d)
    n_gap = n_cont - 1
    A = np.zeros((n_gap, d + 1))
    for k in range(d + 1):
        rhs = [mpf(0)] * rows
        for r in range(n_match):
            z = zs[r]
            v = mpf(0)
            for m in range(d + 1):
                v += mpf(coef[k][m]) * z ** m
            rhs[r] = v
        btr = []
        for i in range(cols):
            s = mpf(0)
            for r in range(rows):
                s += B[r][i] * rhs[r]
            btr.append(s)
        G = [row[:] for row in G0]
        _solve_mp(G, btr, cols)
        resid = mpf(0)
        for r in range(rows):
            v = mpf(0)
            for i in range(cols):
                v += B[r][i] * btr[i]
            resid = max(resid, abs(v - rhs[r]))
        if resid > 1e-13:
            raise ValueError("blend matrix fit residual too large")
        for j in range(n_gap):
            z = mpf(d + 1 + j)
            val = btr[0]
            for m in range(1, K_MODES + 1):
                arg = twopi * m * z / lam
                val += btr[2 * m - 1] * ctx.cos(arg) + btr[2 * m] * ctx.sin(arg)
            for i in range(d + 1):
                A[j, i] += float(val) * pv[k][i]
    _BLEND_CACHE[key] = A
    return A


def _solve_mp(a, b, n):
    """Gaussian elimination with partial pivoting (src/fc_core.cpp:32-53)."""
    for k in range(n):
        piv = k
        for r in range(k + 1, n):
            if abs(a[r][k]) > abs(a[piv][k]):
                piv = r
        if piv != k:
            a[k], a[piv] = a[piv], a[k]
            b[k], b[piv] = b[piv], b[k]
        if a[k][k] == 0:
            raise ValueError("blend matrix solve: singular system")
        for r in range(k + 1, n):
            f = a[r][k] / a[k][k]
            for c in range(k, n):
                a[r][c] -= f * a[k][c]
            b[r] -= f * b[k]
    for k in range(n - 1, -1, -1):
        s = b[k]
        for c in range(k + 1, n):
            s -= a[k][c] * b[c]
        b[k] = s / a[k][k]


@dataclass
class FcOp:
    """FcOperator (include/fcs/fc_core.hpp:33-86, src/fc_core.cpp:190-306)."""

    n: int
    n_cont: int = 25
    degree: int = 2
    alpha: float = ALPHA
    p: int = P_FILTER
    p_smear: int = P_SMEAR
    A: np.ndarray = field(init=False)

    def __post_init__(self):
        if self.n < 10:
            raise ValueError("FcOperator: n_points must be >= 10")
        if self.n_cont < 4:
            raise ValueError("FcOperator: n_cont must be >= 4")
        self.n_ext = self.n + self.n_cont - 1
        self.period = self.n_ext / (self.n - 1)
        self.n_modes = self.n_ext // 2 + 1
        kmax = self.n_ext // 2
        r = np.arange(self.n_modes) / kmax
        self.filter_profile = np.exp(-self.alpha * r ** (2.0 * self.p))
        self.smear_profile = np.exp(-self.alpha * r ** (2.0 * self.p_smear))
        self.A = blend_matrix(self.n_cont, self.degree)

    # src/fc_core.cpp:221-238 ; lines along the last axis
    def continuation(self, f: np.ndarray) -> np.ndarray:
        d = self.degree
        right = f[..., self.n - 1 - d:]
        left_rev = f[..., d::-1]
        A = self.A
        gap = right @ A.T
        gap = gap + (left_rev @ A[::-1].T)
        return gap

    def _extend(self, f):
        return np.concatenate([f, self.continuation(f)], axis=-1)

    # src/fc_core.cpp:257-284
    def derivative(self, f: np.ndarray, order: int = 1) -> np.ndarray:
        if order not in (1, 2):
            raise ValueError("fc_derivative: order must be 1 or 2")
        ext = self._extend(np.asarray(f, dtype=np.float64))
        spec = np.fft.rfft(ext, axis=-1)
        nb = self.n_ext // 2 + 1
        w0 = 2.0 * math.pi / self.period
        k = np.arange(nb)
        if order == 1:
            w = w0 * k * (1.0 / self.n_ext)
            spec = spec * (1j * w)
            if self.n_ext % 2 == 0:
                spec[..., nb - 1] = 0.0
        else:
            w = w0 * k
            spec = spec * (-w * w * (1.0 / self.n_ext))
        spec[..., 0] = spec[..., 0].real
        if self.n_ext % 2 == 0:
            spec[..., nb - 1] = spec[..., nb - 1].real
        out = np.fft.irfft(spec, n=self.n_ext, axis=-1, norm="forward")
        return out[..., : self.n]

    # src/fc_core.cpp:286-306
    def apply_profile(self, f: np.ndarray, profile: np.ndarray) -> np.ndarray:
        ext = self._extend(np.asarray(f, dtype=np.float64))
        spec = np.fft.rfft(ext, axis=-1) * (profile * (1.0 / self.n_ext))
        spec[..., 0] = spec[..., 0].real
        if self.n_ext % 2 == 0:
            spec[..., -1] = spec[..., -1].real
        out = np.fft.irfft(spec, n=self.n_ext, axis=-1, norm="forward")
        return out[..., : self.n]

    def filter(self, f):
        return self.apply_profile(f, self.filter_profile)

    def strong_filter(self, f):
        return self.apply_profile(f, self.smear_profile)


_OP_CACHE: dict = {}


def get_op(n: int, n_cont: int = 25, degree: int = 2) -> FcOp:
    """OperatorCache::get (src/fc_core.cpp:391-402)."""
    key = (n, n_cont, degree)
    if key not in _OP_CACHE:
        _OP_CACHE[key] = FcOp(n, n_cont, degree)
    return _OP_CACHE[key]


# ---------------------------------------------------------------------------
# SDNN classifier (src/viscosity.cpp)


@dataclass
class Mlp:
    """MlpClassifier (src/viscosity.cpp:63-133), FCNN v1 weight format."""

    weights: list
    biases: list
    activation: int = 1

    @staticmethod
    def load(path: str) -> "Mlp":
        with open(path, "rb") as fh:
            buf = fh.read()
        if buf[:4] != b"FCNN":
            raise ValueError("bad weight file magic")
        version, act, nl = struct.unpack_from("<III", buf, 4)
        if version != 1:
            raise ValueError("unsupported weight file version")
        off = 16
        W, b = [], []
        for _ in range(nl):
            r, c = struct.unpack_from("<II", buf, off)
            off += 8
            w = np.frombuffer(buf, dtype="<f8", count=r * c, offset=off).reshape(r, c).copy()
            off += 8 * r * c
            bb = np.frombuffer(buf, dtype="<f8", count=r, offset=off).copy()
            off += 8 * r
            W.append(w)
            b.append(bb)
        if W[0].shape[1] != 7 or W[-1].shape[0] != 4:
            raise ValueError("weight file has wrong input/output dimensions")
        return Mlp(W, b, act)

    def forward(self, x: np.ndarray) -> np.ndarray:
        """x: (..., 7) normalised stencils -> (..., 4) logits
        (src/viscosity.cpp:108-124: y_i = b_i + sum_j W_ij x_j, tanh hidden)."""
        y = np.asarray(x, dtype=np.float64)
        nl = len(self.weights)
        for l in range(nl):
            W, b = self.weights[l], self.biases[l]
            s = np.broadcast_to(b, y.shape[:-1] + b.shape).copy()
            for j in range(W.shape[1]):  # sequential j accumulation, as the reference
                s = s + W[:, j] * y[..., j : j + 1]
            y = np.tanh(s) if l + 1 < nl else s
        return y


def normalize_stencils(st: np.ndarray, abs_floor: float = ABS_FLOOR):
    """normalize_stencil (src/viscosity.cpp:48-59), vectorised; returns
    (normalised, ok) where ok=False is the class-4 guard."""
    lo = st.min(axis=-1, keepdims=True)
    hi = st.max(axis=-1, keepdims=True)
    span = hi - lo
    scale = np.maximum(np.maximum(np.abs(lo), np.abs(hi)), 1e-100)
    ok = ~((span <= 1e-13 * scale) | (span <= abs_floor))
    safe = np.where(ok, span, 1.0)
    out = 2.0 * (st - lo) / safe - 1.0
    return out, ok[..., 0]


def classify_lines(mlp: Mlp, lines: np.ndarray, abs_floor: float = ABS_FLOOR, width: int = 7):
    """Classifier::classify_line, ann variant (src/viscosity.cpp:143-160),
    for a batch of equal-length lines along the last axis. Also returns the
    logit margin (top1 - top2) so parity can be gated on it."""
    n = lines.shape[-1]
    if n < width:
        return np.full(lines.shape, 4, dtype=np.int32), np.full(lines.shape, np.inf)
    idx = np.arange(n)
    start = np.clip(idx - width // 2, 0, n - width)
    gather = start[:, None] + np.arange(width)[None, :]
    st = lines[..., gather]  # (..., n, 7)
    nrm, ok = normalize_stencils(st, abs_floor)
    logits = mlp.forward(nrm)
    best = np.zeros(logits.shape[:-1], dtype=np.int32)
    for k in range(1, 4):  # lowest index wins ties (src/viscosity.cpp:126-133)
        best = np.where(logits[..., k] > np.take_along_axis(logits, best[..., None], -1)[..., 0], k, best)
    srt = np.sort(logits, axis=-1)
    margin = srt[..., -1] - srt[..., -2]
    tau = np.where(ok, best + 1, 4).astype(np.int32)
    margin = np.where(ok, margin, np.inf)
    return tau, margin


def classify_lines_spectrum(lines: np.ndarray, window: int = 32, abs_floor: float = ABS_FLOOR,
                            n_cont: int = 25):
    """Classifier::classify_line, fallback variant (src/viscosity.cpp:161-208):
    FcOperator::spectrum (src/fc_core.cpp:308-316) of every window, then the
    log-log least-squares decay exponent of the top quarter of the modes.
    Returns (tau, margin) where margin is the distance of the decision
    variables from their thresholds (decay exponent from 1.6 / 2.6 / 3.6,
    tail peak from 2e-4, relative), for gating parity on near-ties."""
    n = lines.shape[-1]
    w = min(window, n)
    if w < 12:
        return np.full(lines.shape, 4, dtype=np.int32), np.full(lines.shape, np.inf)
    op = get_op(w, n_cont)
    nb = op.n_ext // 2 + 1
    k_lo = (3 * (nb - 1)) // 4
    idx = np.arange(n)
    start = np.clip(idx - w // 2, 0, n - w)
    gather = start[:, None] + np.arange(w)[None, :]
    st = lines[..., gather]  # (..., n, w)
    nrm, ok = normalize_stencils(st, abs_floor)
    ext = op._extend(nrm)
    mag = np.abs(np.fft.rfft(ext, axis=-1)) / op.n_ext
    tail = mag[..., k_lo:nb]
    ks = np.arange(k_lo, nb, dtype=np.float64)
    lx = np.log(ks)
    ly = np.log(np.maximum(tail, 1e-300))
    cnt = nb - k_lo
    sx, sxx = lx.sum(), (lx * lx).sum()
    sy = ly.sum(axis=-1)
    sxy = (ly * lx).sum(axis=-1)
    s = -(cnt * sxy - sx * sy) / (cnt * sxx - sx * sx)
    peak = tail.max(axis=-1)
    tau = np.where(peak < 2e-4, 4, np.where(s < 1.6, 1, np.where(s < 2.6, 2, np.where(s < 3.6, 3, 4))))
    margin = np.minimum(np.abs(peak - 2e-4) / 2e-4, np.min(np.abs(s[..., None] - np.array([1.6, 2.6, 3.6])), axis=-1))
    tau = np.where(ok, tau, 4).astype(np.int32)
    margin = np.where(ok, margin, np.inf)
    return tau, margin


def classify_field(mlp: Mlp, proxy: np.ndarray):
    """Classifier::classify for a rectangular subpatch (src/viscosity.cpp:211-238):
    rows, then columns combined by min. Returns (tau as float64, min margin)."""
    tr, mr = classify_lines(mlp, proxy)
    tc, mc = classify_lines(mlp, proxy.T)
    tau = np.minimum(tr, tc.T).astype(np.float64)
    return tau, np.minimum(mr, mc.T)


def proxy_mwsb(e: np.ndarray):
    """proxy_value / mwsb_value (src/viscosity.cpp:13-29), e = (4, nj, ni)."""
    rho, ru, rv, E = e
    if not np.all(rho > 0.0):
        raise InvalidState("nonpositive density")
    u = ru / rho
    v = rv / rho
    ke = 0.5 * rho * (u * u + v * v)
    p = (GAMMA - 1.0) * (E - ke)
    if not np.all(p > 0.0):
        raise InvalidState("nonpositive pressure")
    um = np.sqrt(u * u + v * v)
    return um * np.sqrt(rho / (GAMMA * p)), um + np.sqrt(GAMMA * p / rho)


# ---------------------------------------------------------------------------
# per-subpatch state and the superstep


@dataclass
class Sub:
    """The slice of SubpatchData (include/fcs/subpatch_data.hpp:19-63) the step
    touches, for a rectangular subpatch (all bounding-box points valid).

    bc_* : per line end a tuple (kind, state4, pressure) or None, ordered like
    rows[j].bc_lo/bc_hi and cols[i].bc_lo/bc_hi."""

    ni: int
    nj: int
    mask: np.ndarray  # uint8 (nj, ni)
    iq1x: np.ndarray
    iq2x: np.ndarray
    iq1y: np.ndarray
    iq2y: np.ndarray
    h_min: np.ndarray
    h_max: np.ndarray
    w_norm: np.ndarray
    inv_len1: float  # rows: 1/((ni-1) h1)
    inv_len2: float  # cols: 1/((nj-1) h2)
    bc_row_lo: object = None
    bc_row_hi: object = None
    bc_col_lo: object = None
    bc_col_hi: object = None
    e: np.ndarray = None
    n_cont: int = 25

    def __post_init__(self):
        z = lambda: np.zeros((4, self.nj, self.ni))
        if self.e is None:
            self.e = z()
        self.e0, self.e2, self.e3, self.rhs, self.rhs3 = z(), z(), z(), z(), z()
        shp = (self.nj, self.ni)
        self.mu_hat = np.zeros(shp)
        self.mu = np.zeros(shp)
        self.tau = np.full(shp, 4.0)
        self.speed = np.ones(shp)
        self.margin = np.full(shp, np.inf)
        self.op1 = get_op(self.ni, self.n_cont)
        self.op2 = get_op(self.nj, self.n_cont)

    # src/subpatch_data.cpp:9-28
    def d1(self, f):
        return self.op1.derivative(f) * self.inv_len1

    def d2(self, f):
        return (self.op2.derivative(f.T) * self.inv_len2).T

    # src/subpatch_data.cpp:30-42 (rows, then columns, in place)
    def filter_field(self, f):
        f = self.op1.filter(f)
        return self.op2.filter(f.T).T

    # src/subpatch_data.cpp:44-67
    def smear_field(self, f, m):
        s = self.op1.strong_filter(f)
        f = m * s + (1.0 - m) * f
        s = self.op2.strong_filter(f.T).T
        return m * s + (1.0 - m) * f


def euler_rhs(d: Sub, e: np.ndarray, mu: np.ndarray) -> np.ndarray:
    """src/euler.cpp:25-101 (rectangular subpatch: every point valid)."""
    rho, mx, my, E = e
    valid = d.mask != 0
    interior = d.mask == 1
    rs = np.where(rho != 0.0, rho, 1e-300)
    p = (GAMMA - 1.0) * (E - 0.5 * (mx * mx + my * my) / rs)
    bad = interior & (~(rho > 0.0) | ~(p > 0.0) | ~np.isfinite(p))
    if bad.any():
        raise InvalidState("nonpositive density or pressure")
    theta = p / rs
    out = np.zeros_like(e)
    for c in range(4):
        u = mx / rho
        pp = rho * theta
        fx = [mx, mx * u + pp, my * u, u * (E + pp)][c]
        a = d.iq1x * d.d1(fx) + d.iq2x * d.d2(fx)
        out[c] = np.where(valid, out[c] + -1.0 * a, out[c])
        v = my / rho
        fy = [my, mx * v, my * v + pp, v * (E + pp)][c]
        a = d.iq1y * d.d1(fy) + d.iq2y * d.d2(fy)
        out[c] = np.where(valid, out[c] + -1.0 * a, out[c])
    for c in range(4):
        w = e[c] if c < 3 else theta
        s2, s3 = d.d1(w), d.d2(w)
        gx = d.iq1x * s2 + d.iq2x * s3
        gy = d.iq1y * s2 + d.iq2y * s3
        s4 = mu * gx
        s5 = mu * gy
        a = d.iq1x * d.d1(s4) + d.iq2x * d.d2(s4)
        out[c] = np.where(valid, out[c] + 1.0 * a, out[c])
        a = d.iq1y * d.d1(s5) + d.iq2y * d.d2(s5)
        out[c] = np.where(valid, out[c] + 1.0 * a, out[c])
    return out


def _apply_bc_at(d: Sub, bc, il, jl, axis, direction):
    """apply_bc_at (src/euler.cpp:105-165)."""
    kind, state, pressure = bc
    e = d.e
    if kind == BC_INFLOW:
        e[:, jl, il] = state
    elif kind == BC_OUTFLOW_P:
        rho, mx, my = e[0, jl, il], e[1, jl, il], e[2, jl, il]
        e[3, jl, il] = pressure / (GAMMA - 1.0) + 0.5 * (mx * mx + my * my) / rho
    elif kind == BC_SLIP:
        if axis == 0:
            nx, ny = d.iq1x[jl, il], d.iq1y[jl, il]
        else:
            nx, ny = d.iq2x[jl, il], d.iq2y[jl, il]
        nn = math.hypot(nx, ny)
        nx /= nn
        ny /= nn
        rho, mx, my, E = e[:, jl, il]
        p = (GAMMA - 1.0) * (E - 0.5 * (mx * mx + my * my) / rho)
        mn = mx * nx + my * ny
        tmx, tmy = mx - mn * nx, my - mn * ny
        e[1, jl, il] = tmx
        e[2, jl, il] = tmy
        e[3, jl, il] = p / (GAMMA - 1.0) + 0.5 * (tmx * tmx + tmy * tmy) / rho
    elif kind == BC_NOSLIP:
        i1, j1 = il + (direction if axis == 0 else 0), jl + (direction if axis == 1 else 0)
        i2, j2 = il + (2 * direction if axis == 0 else 0), jl + (2 * direction if axis == 1 else 0)

        def th(i, j):
            rho, mx, my, E = e[:, j, i]
            return (GAMMA - 1.0) * (E - 0.5 * (mx * mx + my * my) / rho) / rho

        t = (4.0 * th(i1, j1) - th(i2, j2)) / 3.0
        rho = e[0, jl, il]
        e[1, jl, il] = 0.0
        e[2, jl, il] = 0.0
        e[3, jl, il] = rho * t / (GAMMA - 1.0)
    elif kind == BC_ZERO_NORMAL:
        i1, j1 = il + (direction if axis == 0 else 0), jl + (direction if axis == 1 else 0)
        i2, j2 = il + (2 * direction if axis == 0 else 0), jl + (2 * direction if axis == 1 else 0)
        e[:, jl, il] = (4.0 * e[:, j1, i1] - e[:, j2, i2]) / 3.0


def enforce_bc(d: Sub):
    """enforce_bc (src/euler.cpp:167-180): every row end, then every column end."""
    for jl in range(d.nj):
        if d.bc_row_lo and d.bc_row_lo[jl]:
            _apply_bc_at(d, d.bc_row_lo[jl], 0, jl, 0, +1)
        if d.bc_row_hi and d.bc_row_hi[jl]:
            _apply_bc_at(d, d.bc_row_hi[jl], d.ni - 1, jl, 0, -1)
    for il in range(d.ni):
        if d.bc_col_lo and d.bc_col_lo[il]:
            _apply_bc_at(d, d.bc_col_lo[il], il, 0, 1, +1)
        if d.bc_col_hi and d.bc_col_hi[il]:
            _apply_bc_at(d, d.bc_col_hi[il], il, d.nj - 1, 1, -1)


def ssprk_stage_update(d: Sub, stage: int, dt: float):
    """src/euler.cpp:182-221."""
    u, u0, r = d.e, d.e0, d.rhs
    if stage == 0:
        d.e = u0 + dt * B0 * r
    elif stage == 1:
        d.e = A20 * u0 + A21 * u + dt * B1 * r
        d.e2 = d.e.copy()
    elif stage == 2:
        d.e = A30 * u0 + A32 * u + dt * B2 * r
        d.e3 = d.e.copy()
    elif stage == 3:
        d.rhs3 = r.copy()
        d.e = A40 * u0 + A43 * u + dt * B3 * r
    else:
        d.e = C2 * d.e2 + C3 * d.e3 + dt * D3 * d.rhs3 + C4 * u + dt * D4 * r


def dt_bound_local(d: Sub) -> float:
    """src/euler.cpp:223-236."""
    m = d.mask == 1
    if not m.any():
        return math.inf
    h = d.h_min[m]
    rate = d.speed[m] / h + d.mu[m] / (h * h)
    if not np.all((rate > 0.0) & np.isfinite(rate)):
        raise InvalidState("nonfinite wave speed")
    return float(np.min(1.0 / rate))


@dataclass
class Plan:
    """CommPlan (include/fcs/runtime.hpp:16-49), copies only (intra-patch):
    per recipient, arrays (dst, src_sub, src, w)."""

    sol: list  # per sub: (dst, src_sub, src) int arrays
    visc: list  # per sub: (dst, src_sub, src, w)


class Engine:
    """Engine::run superstep (src/runtime.cpp:327-454,482-511) over rectangular
    subpatches with an intra-patch copy plan."""

    def __init__(self, subs, plan: Plan, mlp: Mlp, cfl=0.5, T=1e300, smear_radius=10):
        self.subs = subs
        self.plan = plan
        self.mlp = mlp
        self.cfl = cfl
        self.T = T
        self.smear_radius = smear_radius
        self.t = 0.0
        self.step_count = 0
        self.dt = 0.0

    def finish_ic(self):
        """apply_ic tail (src/runtime.cpp:284-286)."""
        for d in self.subs:
            enforce_bc(d)
        self.exchange()

    def phase0(self):
        for d in self.subs:
            proxy, speed = proxy_mwsb(d.e)
            d.speed = speed
            d.tau, d.margin = classify_field(self.mlp, proxy)
            t = np.clip(d.tau.astype(np.int64), 1, 4) - 1
            c = np.asarray(VISC_C)[t]
            d.mu_hat = np.where(d.mask == 1, c * d.h_max * d.speed, 0.0)

    def phase1(self):
        for k, d in enumerate(self.subs):
            mu = (d.w_norm * d.mu_hat).ravel()
            dst, src_sub, src, w = self.plan.visc[k]
            for n in range(len(dst)):  # sequential accumulation order
                mu[dst[n]] += w[n] * self.subs[src_sub[n]].mu_hat.ravel()[src[n]]
            d.mu = np.maximum(mu, 0.0).reshape(d.nj, d.ni)

    def phase2(self):
        for d in self.subs:
            rho, mx, my, E = d.e
            theta = (GAMMA - 1.0) * (E - 0.5 * (mx * mx + my * my) / rho) / rho
            if self.step_count == 0:
                tau_rho, _ = classify_field(self.mlp, d.e[0])
                seed = (d.tau <= 2.0) | (tau_rho <= 2.0)
                m01 = np.zeros((d.nj, d.ni))
                r = self.smear_radius
                for jl, il in zip(*np.nonzero(seed)):
                    m01[max(0, jl - r) : jl + r + 1, max(0, il - r) : il + r + 1] = 1.0
                d.m01 = m01
                rho = d.smear_field(rho, m01)
                mx = d.smear_field(mx, m01)
                my = d.smear_field(my, m01)
                theta = d.smear_field(theta, m01)
            else:
                rho = d.filter_field(rho)
                mx = d.filter_field(mx)
                my = d.filter_field(my)
                theta = d.filter_field(theta)
            E = rho * theta / (GAMMA - 1.0) + 0.5 * (mx * mx + my * my) / rho
            d.e = np.stack([rho, mx, my, E])
            enforce_bc(d)
            d.e0 = d.e.copy()
            d.dt_local = dt_bound_local(d)

    def reduce_dt(self):
        b = min(d.dt_local for d in self.subs)
        self.dt = self.cfl * b
        if self.t + self.dt > self.T:
            self.dt = self.T - self.t
        return self.dt

    def stage(self, s):
        for d in self.subs:
            d.rhs = euler_rhs(d, d.e, d.mu)
            ssprk_stage_update(d, s, self.dt)
            enforce_bc(d)
        self.exchange()

    def exchange(self):
        """phase 6 (src/runtime.cpp:433-454), copies only; every donor read
        happens after all stage updates (barrier)."""
        src_e = [np.ascontiguousarray(d.e).reshape(4, -1).copy() for d in self.subs]
        for k, d in enumerate(self.subs):
            dst, src_sub, src = self.plan.sol[k]
            if len(dst) == 0:
                continue
            e = np.ascontiguousarray(d.e)  # reshape below must be a view
            ef = e.reshape(4, -1)
            for s in np.unique(src_sub):
                m = src_sub == s
                ef[:, dst[m]] = src_e[s][:, src[m]]
            d.e = e

    def step(self):
        self.phase0()
        self.phase1()
        self.phase2()
        self.reduce_dt()
        for s in range(5):
            self.stage(s)
        self.t += self.dt
        self.step_count += 1
