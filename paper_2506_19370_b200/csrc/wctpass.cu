// Cartesian flux-form passes (and the phase-2 filter) of the N = 256 lines on
// the register-resident 8 x 35 transform (wct280.h): PassXc / PassYc of
// step_kernels.cu (euler_rhs, src/euler.cpp:25-101, as div(mu grad w - f),
// and the SSPRK(5,4) stage update, src/euler.cpp:182-221) with the line data
// in the lanes' registers from the global loads to the global stores.
//
// A warp transforms four complex lines at once; a line's two *halves* are the
// complex lines (rho, rho u) (half 0) and (rho v, theta) (half 1). Lane
// (c, r) -- c = lane / 8 the complex line, r = lane % 8 -- owns the positions
// r + 8 t (t < 32) of its line.
//  * Pass Y (columns): a unit is one half of four adjacent columns (c = the
//    column; an instruction reads 8 rows x 32 contiguous bytes: whole
//    sectors); the two halves of a column quad are consecutive units, so they
//    run on neighbouring warps of one CTA and the second one's loads hit L1.
//    Pass Y writes only tA, which it never reads: the halves are independent.
//  * Pass X (rows): a unit is both halves of two adjacent rows (c = 2 row +
//    half; the two halves' lanes load the same addresses in one instruction).
//    Pass X updates e in place and each half reads all four components, so a
//    row's halves must share a warp: the update follows every read of the
//    row in program order across the warp's synchronisations.
// Per pass and unit:
//
//   load e -> w -> [continuation, DFT-35] -> smem -> [140 x (DFT-8, multiplier,
//   inverse DFT-8)] -> smem -> [inverse DFT-35] -> Phi = mu iq D w - f ->
//   [continuation, DFT-35] -> ... -> [inverse DFT-35] -> X: rhs = tA + iq1x D1
//   Phi_x and the SSPRK update; Y: tA = iq2y D2 Phi_y
//
// i.e. four shared-memory round trips per pass and line (the per-stage
// prime-factor passes of wpass.cu take fourteen), no block barrier after the
// table staging, and every epilogue works on registers. The price is
// registers (35 complex values per lane: 8 warps per SM).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "wct280.h"
#include "wpass_common.h"

namespace fcsg {

namespace {

constexpr int kCtWarps = 8;  // warps per CTA (one CTA per SM: the registers of 35 complex values per lane)
constexpr int kCtThreads = kCtWarps * 32;

// the lane's line: point index of position 0, point stride along the line
// (rows: 1), subpatch slot, index across the lines (row / column), the
// line-length factor LineInfo::inv_len (src/subpatch_data.cpp:134) and the
// subpatch's uniform metric factor (uniform_q views)
struct CtLine {
    long base;
    long step;
    int sub, idx;
    bool ok;  // false: past the last line (the lane computes on line 0 and stores nothing)
    double inv_len, qc;
};

template <bool ROWS>
FCSG_HD int ct_half(int unit, int c) {
    return ROWS ? (c & 1) : (unit & 1);
}
template <bool ROWS>
FCSG_HD CtLine ct_line(const EngineDev& E, int unit, int c) {
    CtLine g;
    const int ni = E.ni, nj = E.nj;
    const bool uq = E.uniform_q != 0;
    if (ROWS) {
        const int gl = 2 * unit + (c >> 1);
        g.ok = gl < E.S * nj;
        const int l = g.ok ? gl : 0;
        g.sub = l / nj;
        g.idx = l - g.sub * nj;
        g.base = static_cast<long>(g.sub) * ni * nj + static_cast<long>(g.idx) * ni;
        g.step = 1;
        g.inv_len = 1.0 / ((wct::kN - 1) * E.h1[g.sub]);
        g.qc = uq ? E.iq1x_c[g.sub] : 0.0;
    } else {
        const int qps = (ni + 3) / 4;
        const int quad = unit >> 1;
        g.sub = quad / qps;
        const int col = (quad - g.sub * qps) * 4 + c;
        g.ok = col < ni;
        g.idx = g.ok ? col : 0;
        g.base = static_cast<long>(g.sub) * ni * nj + g.idx;
        g.step = ni;
        g.inv_len = 1.0 / ((wct::kN - 1) * E.h2[g.sub]);
        g.qc = uq ? E.iq2y_c[g.sub] : 0.0;
    }
    return g;
}
// work units of a pass (host and device)
#if FCSG_CUDA
#define FCSG_HOST_DEV __host__ __device__ inline
#else
#define FCSG_HOST_DEV inline
#endif
template <bool ROWS>
FCSG_HOST_DEV int ct_units(int S, int ni, int nj) {
    return ROWS ? (S * nj + 1) / 2 : 2 * S * ((ni + 3) / 4);
}

// the continuation's boundary samples of the lane's line: fr[i] = f[253 + i]
// is z[31] of lane 5 + i of the line's lane group, fl[i] = f[2 - i] is z[0]
// of lane 2 - i
#if FCSG_CUDA
__device__ __forceinline__ void ct_ends(int lane, const double2 (&z)[wct::kT], double2 (&fr)[wct::kD1],
                                        double2 (&fl)[wct::kD1]) {
    const int g = lane & ~7;
#pragma unroll
    for (int i = 0; i < wct::kD1; ++i) {
        fr[i] = mk2(__shfl_sync(0xffffffffu, z[31].x, g + 5 + i), __shfl_sync(0xffffffffu, z[31].y, g + 5 + i));
        fl[i] = mk2(__shfl_sync(0xffffffffu, z[0].x, g + 2 - i), __shfl_sync(0xffffffffu, z[0].y, g + 2 - i));
    }
}
#endif

// registers -> continuation -> DFT-35 -> the warp's buffer
FCSG_HD void ct_forward(int c, int r, double2 (&z)[wct::kT], const double2 (&fr)[wct::kD1],
                        const double2 (&fl)[wct::kD1], const double* blend, double2* buf) {
    wct::continuation(r, z, fr, fl, blend);
    wct::dft35<false>(z);
    wct::put35(buf, c, r, z);
}
// the warp's buffer -> inverse DFT-35 -> registers (t < 32: the line's points)
FCSG_HD void ct_inverse(int c, int r, const double2* buf, double2 (&z)[wct::kT]) {
    wct::get35(buf, c, r, z);
    wct::dft35<true>(z);
}

// ---------------------------------------------------------------------------
// Asynchronous point loads. A lane's global inputs arrive through a private
// ring in shared memory (kRingVals doubles per lane, value k of the lane at
// ring[k * 32 + lane]: conflict-free) filled by 8-byte cp.async copies: the
// inputs of point t + D are requested when point t has been consumed, and the
// first D points of a phase before the preceding shared-memory DFT-8 step, so
// a load's L2 latency overlaps D points of arithmetic (or a whole transform
// step) without holding registers -- the 35 complex values of the transform
// leave none for deep register prefetch. Every slot is written and read by
// its own lane only: cp.async.wait_group is all the synchronisation needed.
constexpr int kRingVals = 36;
constexpr int kRingSlots = kRingVals * 32;  // doubles per warp

FCSG_HD void cp8(double* smem, const double* gmem) {
#if FCSG_CUDA
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
#else
    *smem = *gmem;
#endif
}
FCSG_HD void cp_commit() {
#if FCSG_CUDA
    asm volatile("cp.async.commit_group;" ::: "memory");
#endif
}
template <int N>
FCSG_HD void cp_wait() {
#if FCSG_CUDA
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
#endif
}

constexpr size_t kCtSmem =
    (wct::kTabSlots + kCtWarps * wct::kBufSlots) * sizeof(double2) + kCtWarps * kRingSlots * sizeof(double);

// per-lane state of one unit
struct CtLane {
    CtLine g;
    int half, c, r;
    long step8;          // point stride of one t step (8 positions)
    double* ring;        // the lane's ring base (ring + lane)
    const double* src[5];  // e[0..3], mu at the lane's position r
};
template <bool ROWS>
FCSG_HD CtLane ct_lane(const EngineDev& E, int unit, int lane, double* ring) {
    CtLane L;
    L.c = lane >> 3;
    L.r = lane & 7;
    L.half = ct_half<ROWS>(unit, L.c);
    L.g = ct_line<ROWS>(E, unit, L.c);
    const long step = ROWS ? 1 : L.g.step;
    L.step8 = 8 * step;
    L.ring = ring + lane;
    const long p0 = L.g.base + L.r * step;
    for (int q = 0; q < 4; ++q) L.src[q] = E.e[q] + p0;
    L.src[4] = E.mu + p0;
    return L;
}

// the positivity diagnostic's failure path (src/euler.cpp:37-39: interior
// points only), out of line: it runs at most once per run
#if FCSG_CUDA
__device__ __noinline__
#else
inline
#endif
void ct_positivity_fail(const uint8_t* mask, StepScalars* sc, long p, int sub, int i, int j) {
    if (mask[p] == 1) raise_error(sc, 1, sub, i, j);
}

// point phase (both rounds): the conserved state and mu at the lane's points
// -> round 0: the half's complex line w = (rho, rho u) or (rho v, theta);
// round 1: Phi = mu iq D w - f from z = D w (unnormalised), f the x-fluxes
// (rows) or y-fluxes (columns) of the half's components (src/euler.cpp:44-55,
// 64-75). One code path: z <- ms z - f with ms = 0, f = -w in round 0 (exact).
// The positivity diagnostic of euler_rhs runs once per point and stage: in
// pass X, round 0, on half 0.
constexpr int kPtVals = 5;
constexpr int kPtDepth = kRingVals / kPtVals;
template <bool ROWS>
FCSG_HD void ct_point_issue(const CtLane& L, int t) {
    const long off = ROWS ? 8 * t : t * L.step8;
#pragma unroll
    for (int v = 0; v < kPtVals; ++v) cp8(L.ring + ((t % kPtDepth) * kPtVals + v) * 32, L.src[v] + off);
    cp_commit();
}
template <bool ROWS>
FCSG_HD void ct_point_prologue(const CtLane& L) {
#pragma unroll
    for (int t = 0; t < kPtDepth; ++t) ct_point_issue<ROWS>(L, t);
}
// points consumed per wait: their dependent chains (reciprocal + Newton steps
// -> pressure -> fluxes, ~25 FP64 operations deep) interleave; one point at a
// time left the chain's latency exposed at two warps per scheduler
constexpr int kPtChunk = 4;
static_assert(kPtChunk <= kPtDepth && 32 % kPtChunk == 0, "chunk within the ring");
template <bool ROWS>
FCSG_HD void ct_point_main(const EngineDev& E, const CtLane& L, int round, double2 (&z)[wct::kT]) {
    const CtLine& g = L.g;
    const int half = L.half;
    const bool uq = E.uniform_q != 0;
    const double* metric = (ROWS ? E.iq1x : E.iq2y) + g.base + L.r * (ROWS ? 1 : g.step);
#pragma unroll
    for (int t0 = 0; t0 < 32; t0 += kPtChunk) {
        cp_wait<kPtDepth - kPtChunk>();  // all but the newest D - C groups: points t0 .. t0 + C - 1 have landed
        double v[kPtChunk][kPtVals], a[kPtChunk];
#pragma unroll
        for (int k = 0; k < kPtChunk; ++k) {
            const double* s = L.ring + ((t0 + k) % kPtDepth) * kPtVals * 32;
#pragma unroll
            for (int q = 0; q < kPtVals; ++q) v[k][q] = s[32 * q];
            a[k] = (uq || round == 0) ? g.qc : ldg1(metric + (ROWS ? 8 * (t0 + k) : (t0 + k) * L.step8));
        }
#pragma unroll
        for (int k = 0; k < kPtChunk; ++k) {
            const int t = t0 + k;
            const PrimR q = prim_r(v[k][0], v[k][1], v[k][2], v[k][3]);
            double ms, f0, f1;
            if (round == 0) {
                if (ROWS && half == 0 && g.ok) {
                    const double pr = q.theta * ((q.rho != 0.0) ? q.rho : 1e-300);
                    if (!(q.rho > 0.0) || !(pr > 0.0) || !finite_d(pr))
                        ct_positivity_fail(E.mask, E.sc, g.base + L.r + 8 * t, E.sub_base + g.sub, L.r + 8 * t, g.idx);
                }
                ms = 0.0;
                f0 = half ? -q.my : -q.rho;
                f1 = half ? -q.theta : -q.mx;
            } else {
                ms = v[k][4] * (a[k] * g.inv_len);
                if (ROWS) {  // F = (mx, mx u + p | my u, u (E + p)): the half selects operands, not results
                    const double u = q.mx * q.ir;
                    const double my_u = q.my * u;
                    f0 = half ? my_u : q.mx;
                    f1 = fma(half ? q.E + q.p : q.mx, u, half ? 0.0 : q.p);
                } else {  // G = (my, mx v | my v + p, v (E + p))
                    const double vv = q.my * q.ir;
                    f0 = half ? fma(q.my, vv, q.p) : q.my;
                    f1 = (half ? q.E + q.p : q.mx) * vv;
                }
            }
            z[t] = mk2(fma(ms, z[t].x, -f0), fma(ms, z[t].y, -f1));
        }
#pragma unroll
        for (int k = 0; k < kPtChunk; ++k) {
            if (t0 + k + kPtDepth < 32) ct_point_issue<ROWS>(L, t0 + k + kPtDepth);
            else cp_commit();
        }
    }
    cp_wait<0>();
}

// SSPRK(5,4) stage update of pass X (src/euler.cpp:182-221; ssprk_update of
// pass_common.h), by stage class SC: 0 = stage 0 (inputs per component: e,
// tA), 1 = stages 1-3 (e, tA, e0), 2 = stage 4 (e, tA, e2, e3, rhs3).
//   e <- cA y + cU u + cR r     (stage 0: u + dt SB0 r; 1-3: SAx0 e0 + SAxy u + dt SBx r)
//   e <- SC2 e2 + SC3 e3 + dt SD3 rhs3 + SC4 u + dt SD4 r     (stage 4)
// with r = tA + iq1x D1 Phi_x, u = the stage's input state (pass Y does not
// write e, and a point of e is rewritten by the lane that read it last, after
// the warp's other half has read it: the phases are ordered by __syncwarp).
// The stage's extra store: 0: e0 <- u, 1: e2 <- e, 2: e3 <- e, 3: rhs3 <- r.
template <int SC>
struct UpdVals {
    static constexpr int kPerComp = SC == 0 ? 2 : (SC == 1 ? 3 : 5);
    static constexpr int kVals = 2 * kPerComp;
    static constexpr int kDepth = kRingVals / kVals;
};
struct UpdSrc {
    const double* f[10];  // per component: e, tA, then the stage's registers
    double* e[2];
    double* aux[2];
    double* rhs[2];
};
template <int SC>
FCSG_HD UpdSrc ct_update_src(const EngineDev& E, const CtLane& L, int stage) {
    UpdSrc U;
    const long p0 = L.g.base + L.r;
    constexpr int PC = UpdVals<SC>::kPerComp;
    for (int k = 0; k < 2; ++k) {
        const int q = 2 * L.half + k;
        U.e[k] = E.e[q] + p0;
        U.rhs[k] = E.rhs[0] ? E.rhs[q] + p0 : nullptr;
        double* aux = stage == 0 ? E.e0[q] : stage == 1 ? E.e2[q] : stage == 2 ? E.e3[q] : stage == 3 ? E.rhs3[q] : nullptr;
        U.aux[k] = aux ? aux + p0 : nullptr;
        U.f[k * PC + 0] = E.e[q] + p0;
        U.f[k * PC + 1] = E.tA[q] + p0;
        if (SC == 1) U.f[k * PC + 2] = E.e0[q] + p0;
        if (SC == 2) {
            U.f[k * PC + 2] = E.e2[q] + p0;
            U.f[k * PC + 3] = E.e3[q] + p0;
            U.f[k * PC + 4] = E.rhs3[q] + p0;
        }
    }
    return U;
}
template <int SC>
FCSG_HD void ct_update_issue(const CtLane& L, const UpdSrc& U, int t) {
    constexpr int NV = UpdVals<SC>::kVals, D = UpdVals<SC>::kDepth;
#pragma unroll
    for (int v = 0; v < NV; ++v) cp8(L.ring + ((t % D) * NV + v) * 32, U.f[v] + 8 * t);
    cp_commit();
}
template <int SC>
FCSG_HD void ct_update_prologue(const CtLane& L, const UpdSrc& U) {
#pragma unroll
    for (int t = 0; t < UpdVals<SC>::kDepth; ++t) ct_update_issue<SC>(L, U, t);
}
template <int SC>
FCSG_HD void ct_update_main(const EngineDev& E, const CtLane& L, const UpdSrc& U, int stage,
                            const double2 (&z)[wct::kT]) {
    constexpr int NV = UpdVals<SC>::kVals, D = UpdVals<SC>::kDepth, PC = UpdVals<SC>::kPerComp;
    constexpr int C = D >= 8 ? 4 : (D >= 4 ? 2 : 1);  // points per wait (their loads and chains interleave)
    const CtLine& g = L.g;
    const bool uq = E.uniform_q != 0;
    const double dt = E.sc->dt;
    const double cA = stage == 1 ? SA20 : stage == 2 ? SA30 : stage == 3 ? SA40 : 0.0;
    const double cU = stage == 1 ? SA21 : stage == 2 ? SA32 : stage == 3 ? SA43 : 1.0;
    const double cR = dt * (stage == 0 ? SB0 : stage == 1 ? SB1 : stage == 2 ? SB2 : SB3);
#pragma unroll
    for (int t0 = 0; t0 < 32; t0 += C) {
        cp_wait<D - C>();
        double v[C][NV], sa[C];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const double* s = L.ring + ((t0 + k) % D) * NV * 32;
#pragma unroll
            for (int q = 0; q < NV; ++q) v[k][q] = s[32 * q];
            sa[k] = (uq ? g.qc : ldg1(E.iq1x + g.base + L.r + 8 * (t0 + k))) * g.inv_len;
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int t = t0 + k;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double* sk = v[k] + h * PC;
                const double u = sk[0];
                const double r = fma(sa[k], h ? z[t].y : z[t].x, sk[1]);
                double nu;
                if (SC == 2) nu = SC2 * sk[2 % PC] + SC3 * sk[3 % PC] + dt * SD3 * sk[4 % PC] + SC4 * u + dt * SD4 * r;
                else nu = cA * (SC == 1 ? sk[2 % PC] : 0.0) + cU * u + cR * r;
                if (g.ok) {
                    if (U.rhs[h]) U.rhs[h][8 * t] = r;
                    U.e[h][8 * t] = nu;
                    if (SC != 2) U.aux[h][8 * t] = stage == 0 ? u : (stage == 3 ? r : nu);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
            if (t0 + k + D < 32) ct_update_issue<SC>(L, U, t0 + k + D);
            else cp_commit();
        }
    }
    cp_wait<0>();
}

// last phase of pass Y: tA = iq2y D2 Phi_y of the half's components
FCSG_HD void ct_store_ta(const EngineDev& E, const CtLane& L, const double2 (&z)[wct::kT]) {
    const CtLine& g = L.g;
    if (!g.ok) return;
    const bool uq = E.uniform_q != 0;
    const long p0 = g.base + L.r * g.step;
    double* tA0 = E.tA[2 * L.half] + p0;
    double* tA1 = E.tA[2 * L.half + 1] + p0;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
        const long off = t * L.step8;
        const double d = (uq ? g.qc : ldg1(E.iq2y + p0 + off)) * g.inv_len;
        tA0[off] = d * z[t].x;
        tA1[off] = d * z[t].y;
    }
}

// L2 prefetch of the lane group's share of one field over the unit's lines:
// rows, the line's 2 KB by its r = 0 lane; columns, one 32-byte sector per
// row of the quad by the c = 0 lanes
template <bool ROWS>
FCSG_HD void ct_prefetch(const double* f, const CtLine& g, int c, int r) {
    if (ROWS) {
        if (r == 0) pf_l2_bulk(f + g.base, wct::kN * sizeof(double));
    } else {
        if (c == 0)
#pragma unroll 4
            for (int t = 0; t < 32; ++t) pf_l2(f + g.base + (r + 8 * t) * g.step);
    }
}
// unit start: this unit's later inputs (pass X: tA and the RK registers of
// the update) and the next unit's state and mu into L2
template <bool ROWS>
FCSG_HD void ct_unit_prefetch(const EngineDev& E, const CtLane& L, int unit, int nunits, int stride, int stage) {
    const CtLine& g = L.g;
    const int c = L.c, r = L.r, half = L.half;
    if (!E.uniform_q) ct_prefetch<ROWS>(ROWS ? E.iq1x : E.iq2y, g, c, r);
    if (ROWS) {
        const bool e0r = stage >= 1 && stage <= 3;
        for (int k = 0; k < 2; ++k) {
            const int q = 2 * half + k;
            ct_prefetch<ROWS>(E.tA[q], g, c, r);
            if (e0r) ct_prefetch<ROWS>(E.e0[q], g, c, r);
            if (stage == 4) {
                ct_prefetch<ROWS>(E.e2[q], g, c, r);
                ct_prefetch<ROWS>(E.e3[q], g, c, r);
                ct_prefetch<ROWS>(E.rhs3[q], g, c, r);
            }
        }
    }
    const int nxt = unit + stride;
    if (nxt < nunits) {  // half 0 prefetches components 0, 1 and mu, half 1 components 2, 3
        const CtLine gn = ct_line<ROWS>(E, nxt, c);
        ct_prefetch<ROWS>(E.e[2 * half], gn, c, r);
        ct_prefetch<ROWS>(E.e[2 * half + 1], gn, c, r);
        if (half == 0) ct_prefetch<ROWS>(E.mu, gn, c, r);
    }
}

// One unit of a pass (per lane, split at the warp synchronisations):
//   prologue of the point loads
//   2 x { point phase -> continuation, DFT-35 -> smem | next prologue, 140 x
//         (DFT-8, multiplier, inverse DFT-8) | smem -> inverse DFT-35 }
//   X: SSPRK update; Y: tA store
// The two rounds share one loop body (the kernels' code must stay inside the
// instruction caches: fully unrolled per round it did not, and instruction
// fetch became the first stall).
#if FCSG_CUDA
template <bool ROWS, int SC>
__device__ __forceinline__ void ct_unit(const EngineDev& E, int unit, int nunits, int stride, int stage, int lane,
                                        double2* buf, double* ring, const double2* tabs) {
    const double2* mult = tabs;
    const double2* tw = tabs + wct::kNE;
    const double* blend = reinterpret_cast<const double*>(tabs + wct::kNE + wct::kTwSlots);
    const CtLane L = ct_lane<ROWS>(E, unit, lane, ring);
    ct_point_prologue<ROWS>(L);
    ct_unit_prefetch<ROWS>(E, L, unit, nunits, stride, stage);
    UpdSrc U;
    if (ROWS) U = ct_update_src<SC>(E, L, stage);
    double2 z[wct::kT];
#pragma unroll
    for (int t = 0; t < wct::kT; ++t) z[t] = mk2(0.0, 0.0);
#pragma unroll 1
    for (int round = 0; round < 2; ++round) {
        ct_point_main<ROWS>(E, L, round, z);
        double2 fr[wct::kD1], fl[wct::kD1];
        ct_ends(lane, z, fr, fl);
        ct_forward(L.c, L.r, z, fr, fl, blend, buf);
        __syncwarp();
        if (round == 0) ct_point_prologue<ROWS>(L);
        else if (ROWS) ct_update_prologue<SC>(L, U);
        wct::middle<32>(lane, buf, tw, mult);
        __syncwarp();
        ct_inverse(L.c, L.r, buf, z);
    }
    if (ROWS) ct_update_main<SC>(E, L, U, stage, z);
    else ct_store_ta(E, L, z);
    __syncwarp();
}

template <bool ROWS, int SC>
__global__ void __launch_bounds__(kCtThreads, 1) wctpass_kernel(const __grid_constant__ EngineDev E,
                                                               const double2* __restrict__ mult_pfa,
                                                               const double2* __restrict__ tw_src,
                                                               const double* __restrict__ blend_src, int stage) {
    extern __shared__ double2 wsm[];
    {
        wct::TableRegs<kCtThreads> tr;
        tr.load(threadIdx.x, mult_pfa, tw_src, blend_src);
        tr.store(threadIdx.x, wsm);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + wct::kTabSlots + warp * wct::kBufSlots;
    double* ring = reinterpret_cast<double*>(wsm + wct::kTabSlots + kCtWarps * wct::kBufSlots) + warp * kRingSlots;
    const int nunits = ct_units<ROWS>(E.S, E.ni, E.nj);
    const int stride = gridDim.x * kCtWarps;
    for (int unit = blockIdx.x * kCtWarps + warp; unit < nunits; unit += stride)
        ct_unit<ROWS, SC>(E, unit, nunits, stride, stage, lane, buf, ring, wsm);
}

template <bool ROWS, int SC>
void launch_ct(const EngineDev& E, const FcPlanDev& pl, int stage, cudaStream_t s) {
    static unsigned long long done = 0;
    static int resident[64];
    int d = 0;
    cudaGetDevice(&d);
    if (dev::first_on_device(&done)) {
        cudaFuncSetAttribute(wctpass_kernel<ROWS, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kCtSmem));
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wctpass_kernel<ROWS, SC>, kCtThreads, kCtSmem);
        resident[d & 63] = sms * (per > 0 ? per : 1);
    }
    const int nunits = ct_units<ROWS>(E.S, E.ni, E.nj);
    const int need = (nunits + kCtWarps - 1) / kCtWarps;
    const int grid = std::min(need, resident[d & 63]);
    wctpass_kernel<ROWS, SC><<<grid, kCtThreads, kCtSmem, s>>>(E, pl.mult_pfa, pl.tw, pl.blend, stage);
}
#else
// emulation: one warp at a time, every lane's registers kept across the
// phases' synchronisation points
template <bool ROWS, int SC>
void emulate_ct(const EngineDev& E, const FcPlanDev& pl, int stage) {
    std::vector<double2> tabs(wct::kTabSlots), buf(wct::kBufSlots);
    std::vector<double> ring(kRingSlots);
    wct::stage_tables(0, 1, pl.mult_pfa, pl.tw, pl.blend, tabs.data());
    const double2* mult = tabs.data();
    const double2* tw = tabs.data() + wct::kNE;
    const double* blend = reinterpret_cast<const double*>(tabs.data() + wct::kNE + wct::kTwSlots);
    const int nunits = ct_units<ROWS>(E.S, E.ni, E.nj);
    std::vector<double2> zz(32 * wct::kT);
    auto Z = [&](int lane) -> double2(&)[wct::kT] { return *reinterpret_cast<double2(*)[wct::kT]>(&zz[lane * wct::kT]); };
    for (int unit = 0; unit < nunits; ++unit) {
        CtLane L[32];
        UpdSrc U[32];
        for (int lane = 0; lane < 32; ++lane) {
            L[lane] = ct_lane<ROWS>(E, unit, lane, ring.data());
            if (ROWS) U[lane] = ct_update_src<SC>(E, L[lane], stage);
            for (int t = 0; t < wct::kT; ++t) Z(lane)[t] = mk2(0.0, 0.0);
            ct_point_prologue<ROWS>(L[lane]);
        }
        for (int round = 0; round < 2; ++round) {
            for (int lane = 0; lane < 32; ++lane) ct_point_main<ROWS>(E, L[lane], round, Z(lane));
            // the boundary samples of every lane group before any lane's transform overwrites them
            std::vector<double2> fr(32 * wct::kD1), fl(32 * wct::kD1);
            for (int lane = 0; lane < 32; ++lane) {
                const int g0 = lane & ~7;
                for (int i = 0; i < wct::kD1; ++i) {
                    fr[lane * wct::kD1 + i] = Z(g0 + 5 + i)[31];
                    fl[lane * wct::kD1 + i] = Z(g0 + 2 - i)[0];
                }
            }
            for (int lane = 0; lane < 32; ++lane) {
                double2 a[wct::kD1], b[wct::kD1];
                for (int i = 0; i < wct::kD1; ++i) {
                    a[i] = fr[lane * wct::kD1 + i];
                    b[i] = fl[lane * wct::kD1 + i];
                }
                ct_forward(lane >> 3, lane & 7, Z(lane), a, b, blend, buf.data());
            }
            for (int lane = 0; lane < 32; ++lane) {
                if (round == 0) ct_point_prologue<ROWS>(L[lane]);
                else if (ROWS) ct_update_prologue<SC>(L[lane], U[lane]);
            }
            for (int lane = 0; lane < 32; ++lane) wct::middle<32>(lane, buf.data(), tw, mult);
            for (int lane = 0; lane < 32; ++lane) ct_inverse(lane >> 3, lane & 7, buf.data(), Z(lane));
        }
        for (int lane = 0; lane < 32; ++lane) {
            if (ROWS) ct_update_main<SC>(E, L[lane], U[lane], stage, Z(lane));
            else ct_store_ta(E, L[lane], Z(lane));
        }
    }
}
#endif

}  // namespace

void launch_wctpass(const EngineDev& E, const FcPlanDev& pl, bool rows, int stage, void* stream) {
    if (E.S * (rows ? E.nj : E.ni) == 0) return;
#if FCSG_CUDA
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!rows) launch_ct<false, 0>(E, pl, stage, s);
    else if (stage == 0) launch_ct<true, 0>(E, pl, stage, s);
    else if (stage == 4) launch_ct<true, 2>(E, pl, stage, s);
    else launch_ct<true, 1>(E, pl, stage, s);
#else
    (void)stream;
    if (!rows) emulate_ct<false, 0>(E, pl, stage);
    else if (stage == 0) emulate_ct<true, 0>(E, pl, stage);
    else if (stage == 4) emulate_ct<true, 2>(E, pl, stage);
    else emulate_ct<true, 1>(E, pl, stage);
#endif
}

}  // namespace fcsg
