// Register-resident FC line transform for n_ext = 280 as 14 x 20 (N = 256
// points, the reference operator: n_cont = 25, degree 2), two complex lines
// (four real lines) per warp: the FcOperator pipeline of
// src/fc_core.cpp:221-238,257-297 (continuation -> DFT -> spectral multiplier
// -> inverse DFT) with two shared-memory round trips per transform, like the
// 8 x 35 form (wct280.h), but 20 instead of 35 complex values per lane: half
// the registers, so twice the warps per SM, and half the dependent work per
// warp -- the form for batches of a few thousand lines (config 1), which are
// bound by one warp's latency chain.
//
// Decomposition: Cooley-Tukey 280 = 14 x 20 in time. Lane (l, q) of the warp
// (l = lane / 14 the complex line, q = lane % 14; lanes 28-31 idle) owns the
// 20 positions p = q + 14 t (t < 20) of its line: t < 18 and (t = 18, q < 4)
// are the line's own points, read straight from global memory into
// registers (the fourteen lanes of a line read 112 contiguous bytes per
// instruction), the rest are the continuation points 256 + j with j = q - 4
// (t = 18, q >= 4) and j = 10 + q (t = 19). Then
//   1. DFT-20 over t in registers (prime-factor 4 x 5, no twiddles):
//        Y_q[k2] = sum_t x[q + 14 t] W20^(t k2)
//   2. shared memory, then per group (l, k2) (40 groups over 32 lanes):
//        twiddle W280^(q k2), DFT-14 over q -> k1 (prime-factor 2 x 7),
//        multiplier M[k2 + 20 k1], inverse DFT-14 over k1 -> q, twiddle
//        W280^(-q k2)
//   3. shared memory, then per lane the inverse DFT-20 over k2 -> t in
//        registers, stored straight to global memory.
// X[k2 + 20 k1] = sum_q W280^(q k2) W14^(q k1) Y_q[k2] is the length-280 DFT;
// unnormalised like FFTW's c2r (the multiplier tables carry 1/n_ext).
//
// Shared memory of one warp: value (l, q, k2) at l * kPL + q * kPQ + k2. The
// pitches kPQ = 21 = 5 (mod 8) and kPL = 294 = 6 (mod 8) keep the per-lane
// accesses (fixed k2, lanes over (l, q)) conflict-free, and the group
// accesses (fixed q, lanes over k2) read consecutive slots.
#pragma once

#include "fft_line.h"
#include "wct280.h"

namespace fcsg {
namespace w20 {

constexpr int kN = 256;   // points per line
constexpr int kNE = 280;  // n_ext
constexpr int kGap = 24;  // n_cont - 1
constexpr int kD1 = 3;    // degree + 1
constexpr int kQ = 14;    // lanes per complex line
constexpr int kT = 20;    // positions per lane
constexpr int kLines = 2;                // complex lines per warp
constexpr int kActive = kLines * kQ;     // 28 working lanes
constexpr int kPQ = 21;                  // pitch of q (double2)
constexpr int kPL = 294;                 // pitch of the line
constexpr int kBufSlots = kLines * kPL;  // double2 per warp
constexpr int kTwPitch = 15;             // twiddle table: W280^(q k2) at 15 k2 + q
constexpr int kTwSlots = kT * kTwPitch;  // 300
constexpr int kBlendSlots = (kGap * kD1 + 1) / 2;
constexpr int kTabSlots = kNE + kTwSlots + kBlendSlots;

// DFT-20 of z in place, natural order in and out. Prime-factor 4 x 5
// (Good-Thomas): t = (5 a + 4 b) mod 20, k = (5 a' + 16 b') mod 20, so
// W20^(t k) = W4^(a a') W5^(b b'); compile-time indices throughout.
template <bool INV>
FCSG_HD void dft20(double2 (&z)[kT]) {
    constexpr int KA = 5, KB = INV ? 16 : 4;   // first pass: index (KA a + KB b) of the input order
    constexpr int OA = 5, OB = INV ? 4 : 16;   // output order
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        double2 x[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) x[a] = z[(KA * a + KB * b) % 20];
        dft4<INV>(x);
#pragma unroll
        for (int a = 0; a < 4; ++a) z[(KA * a + KB * b) % 20] = x[a];
    }
    double2 y[kT];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double2 x[5];
#pragma unroll
        for (int b = 0; b < 5; ++b) x[b] = z[(KA * a + KB * b) % 20];
        dft_odd<5, INV>(x, nullptr, 5);
#pragma unroll
        for (int b = 0; b < 5; ++b) y[(OA * a + OB * b) % 20] = x[b];
    }
#pragma unroll
    for (int k = 0; k < kT; ++k) z[k] = y[k];
}

// DFT-14 of v in place, natural order in and out. Prime-factor 2 x 7:
// q = (7 a + 2 b) mod 14, k = (7 a' + 8 b') mod 14, W14^(q k) = W2^(a a') W7^(b b').
template <bool INV>
FCSG_HD void dft14(double2 (&v)[kQ]) {
    constexpr int KB = INV ? 8 : 2;  // input order (7 a + KB b)
    constexpr int OB = INV ? 2 : 8;  // output order
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        double2 x[7];
#pragma unroll
        for (int b = 0; b < 7; ++b) x[b] = v[(7 * a + KB * b) % 14];
        dft_odd<7, INV>(x, nullptr, 7);
#pragma unroll
        for (int b = 0; b < 7; ++b) v[(7 * a + KB * b) % 14] = x[b];
    }
    double2 y[kQ];
#pragma unroll
    for (int b = 0; b < 7; ++b) {
        const double2 p0 = v[(KB * b) % 14], p1 = v[(7 + KB * b) % 14];
        y[(OB * b) % 14] = cadd(p0, p1);
        y[(7 + OB * b) % 14] = csub(p0, p1);
    }
#pragma unroll
    for (int k = 0; k < kQ; ++k) v[k] = y[k];
}

// continuation points of lane q: g_j at z[18] (j = q - 4, lanes q >= 4) and
// z[19] (j = 10 + q) (FcOperator::continuation, src/fc_core.cpp:221-238:
// g_j = sum_i A[j][i] f[N-3+i] + sum_i A[23-j][i] f[2-i]); fl[i] = f[2-i],
// fr[i] = f[253+i] of the lane's complex line
FCSG_HD double2 cont_point(int j, const double2 (&fr)[kD1], const double2 (&fl)[kD1], const double* blend) {
    double2 a = mk2(0.0, 0.0), c = mk2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < kD1; ++i) {
        const double cr = blend[j * kD1 + i], cl = blend[(kGap - 1 - j) * kD1 + i];
        a = mk2(a.x + cr * fr[i].x, a.y + cr * fr[i].y);
        c = mk2(c.x + cl * fl[i].x, c.y + cl * fl[i].y);
    }
    return cadd(a, c);
}
FCSG_HD void continuation(int q, double2 (&z)[kT], const double2 (&fr)[kD1], const double2 (&fl)[kD1],
                          const double* blend) {
    if (q >= 4) z[18] = cont_point(q - 4, fr, fl, blend);
    z[19] = cont_point(10 + q, fr, fl, blend);
}

// lane (l, q): store Y_q[k2] (k2 < 20) of line l / load it back
FCSG_HD void put20(double2* buf, int l, int q, const double2 (&z)[kT]) {
    double2* p = buf + l * kPL + q * kPQ;
#pragma unroll
    for (int k = 0; k < kT; ++k) p[k] = z[k];
}
FCSG_HD void get20(const double2* buf, int l, int q, double2 (&z)[kT]) {
    const double2* p = buf + l * kPL + q * kPQ;
#pragma unroll
    for (int k = 0; k < kT; ++k) z[k] = p[k];
}

// step 2 for one group (l, k2): tw = W280^(q k2) at kTwPitch k2 + q, mult =
// the multiplier in natural frequency order
FCSG_HD void middle_group(double2* buf, int l, int k2, const double2* tw, const double2* mult) {
    double2* p = buf + l * kPL + k2;
    const double2* w = tw + kTwPitch * k2;
    double2 v[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) v[q] = p[q * kPQ];
#pragma unroll
    for (int q = 1; q < kQ; ++q) v[q] = cmul(v[q], w[q]);
    dft14<false>(v);
#pragma unroll
    for (int k1 = 0; k1 < kQ; ++k1) v[k1] = cmul(v[k1], mult[k2 + kT * k1]);
    dft14<true>(v);
#pragma unroll
    for (int q = 1; q < kQ; ++q) v[q] = cmulc(v[q], w[q]);
#pragma unroll
    for (int q = 0; q < kQ; ++q) p[q * kPQ] = v[q];
}
// the 40 groups of a warp buffer over 32 lanes: first every lane takes
// (l, k2) = (lane / 16, lane % 16), then lanes 0-3 and 8-11 take k2 = 16 + lane % 4
// of line lane / 8 (quarter-warps of one line each: conflict-free)
FCSG_HD void middle(int lane, double2* buf, const double2* tw, const double2* mult) {
    middle_group(buf, lane >> 4, lane & 15, tw, mult);
    if (lane < 16 && (lane & 7) < 4) middle_group(buf, lane >> 3, 16 + (lane & 3), tw, mult);
}

// the operator tables in a CTA's shared memory: multiplier of one mode in
// natural frequency order (from the prime-factor order of FcPlanDev::mult_pfa,
// wct::mult_entry), twiddles W280^(q k2) from the plan's exp(-2 pi i k / 280)
// table, the 24 x 3 blend matrix
FCSG_HD double2 tw_entry(const double2* tw_src, int k) {
    const int k2 = k / kTwPitch, q = k - kTwPitch * k2;
    return q < kQ ? ldg2(tw_src + q * k2) : mk2(1.0, 0.0);
}
FCSG_HD void stage_tables(int tid, int nthr, const double2* mult_pfa, const double2* tw_src, const double* blend_src,
                          double2* tabs) {
    double* blend = reinterpret_cast<double*>(tabs + kNE + kTwSlots);
    for (int f = tid; f < kNE; f += nthr) tabs[f] = wct::mult_entry(mult_pfa, f);
    for (int k = tid; k < kTwSlots; k += nthr) tabs[kNE + k] = tw_entry(tw_src, k);
    for (int k = tid; k < kGap * kD1; k += nthr) blend[k] = ldg1(blend_src + k);
}
template <int NT>
struct TableRegs {
    static constexpr int NM = (kNE + NT - 1) / NT, NW = (kTwSlots + NT - 1) / NT, NB = (kGap * kD1 + NT - 1) / NT;
    double2 m[NM], w[NW];
    double b[NB];
    FCSG_HD void load(int tid, const double2* mult_pfa, const double2* tw_src, const double* blend_src) {
#pragma unroll
        for (int i = 0; i < NM; ++i)
            if (tid + i * NT < kNE) m[i] = wct::mult_entry(mult_pfa, tid + i * NT);
#pragma unroll
        for (int i = 0; i < NW; ++i)
            if (tid + i * NT < kTwSlots) w[i] = tw_entry(tw_src, tid + i * NT);
#pragma unroll
        for (int i = 0; i < NB; ++i)
            if (tid + i * NT < kGap * kD1) b[i] = ldg1(blend_src + tid + i * NT);
    }
    FCSG_HD void store(int tid, double2* tabs) const {
        double* blend = reinterpret_cast<double*>(tabs + kNE + kTwSlots);
#pragma unroll
        for (int i = 0; i < NM; ++i)
            if (tid + i * NT < kNE) tabs[tid + i * NT] = m[i];
#pragma unroll
        for (int i = 0; i < NW; ++i)
            if (tid + i * NT < kTwSlots) tabs[kNE + tid + i * NT] = w[i];
#pragma unroll
        for (int i = 0; i < NB; ++i)
            if (tid + i * NT < kGap * kD1) blend[tid + i * NT] = b[i];
    }
};

}  // namespace w20
}  // namespace fcsg
