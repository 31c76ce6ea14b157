// Register-resident FC line transform for n_ext = 280 (N = 256 points, the
// reference operator: n_cont = 25, degree 2), four complex lines (eight real
// lines) per warp: the FcOperator pipeline of src/fc_core.cpp:221-238,257-297
// (continuation -> DFT -> spectral multiplier -> inverse DFT) with two
// shared-memory round trips per transform instead of the five of the
// per-stage prime-factor transform (wline.h).
//
// Decomposition: Cooley-Tukey 280 = 8 x 35 in time. Lane (c, r) of the warp
// (c = lane / 8 the complex line, r = lane % 8) owns the 35 positions
// p = r + 8 t (t < 35) of its line -- t < 32 are the line's own points, read
// straight from global memory into registers (the eight lanes of a line read
// 64 contiguous bytes per instruction), t = 32..34 the continuation points
// 256 + r + 8 q. Then
//   1. DFT-35 over t in registers (prime-factor 5 x 7, no twiddles):
//        Y_r[k2] = sum_t x[r + 8 t] W35^(t k2)
//   2. shared memory, then per group (c, k2) (140 groups over 32 lanes):
//        twiddle W280^(r k2), DFT-8 over r -> k1, multiplier M[k2 + 35 k1],
//        inverse DFT-8 over k1 -> r, twiddle W280^(-r k2)
//   3. shared memory, then per lane the inverse DFT-35 over k2 -> t in
//        registers, stored straight to global memory (t < 32).
// X[k2 + 35 k1] = sum_r W280^(r k2) W8^(r k1) Y_r[k2] is the length-280 DFT,
// and the inverse has the mirrored structure; unnormalised like FFTW's c2r
// (the multiplier tables carry 1/n_ext).
//
// Shared memory of one warp: value (c, r, k2) at c * kPC + r * 35 + k2. The
// line pitch kPC = 283 = 3 (mod 8) and the r pitch 35 = 3 (mod 8) keep both
// access patterns conflict-free: the eight lanes of a quarter-warp write
// (fixed c, r = 0..7: 35 r spans the eight 16-byte bank groups) and read
// consecutive groups G = 35 c + k2 (c * 283 + k2 = G mod 8).
#pragma once

#include "fft_line.h"

namespace fcsg {
namespace wct {

constexpr int kN = 256;   // points per line
constexpr int kNE = 280;  // n_ext
constexpr int kGap = 24;  // n_cont - 1
constexpr int kD1 = 3;    // degree + 1
constexpr int kT = 35;    // positions per lane
constexpr int kPC = 283;  // line pitch (double2) of a warp's buffer
constexpr int kLines = 4;                 // complex lines per warp
constexpr int kBufSlots = kLines * kPC;   // double2 per warp
constexpr int kTwPitch = 9;               // twiddle table: W280^(r k2) at 9 k2 + r
constexpr int kTwSlots = kT * kTwPitch;   // 315

// DFT-35 of z in place, natural order in and out. Prime-factor 5 x 7
// (Good-Thomas): t = (7 t2 + 5 t3) mod 35, k = (21 k1 + 15 k2) mod 35, so
// W35^(t k) = W5^(t2 k1) W7^(t3 k2); compile-time indices throughout.
template <bool INV>
FCSG_HD void dft35(double2 (&z)[kT]) {
    if constexpr (!INV) {
#pragma unroll
        for (int t3 = 0; t3 < 7; ++t3) {
            double2 x[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) x[q] = z[(7 * q + 5 * t3) % 35];
            dft_odd<5, false>(x, nullptr, 5);
#pragma unroll
            for (int q = 0; q < 5; ++q) z[(7 * q + 5 * t3) % 35] = x[q];
        }
        double2 y[kT];
#pragma unroll
        for (int k1 = 0; k1 < 5; ++k1) {
            double2 x[7];
#pragma unroll
            for (int q = 0; q < 7; ++q) x[q] = z[(7 * k1 + 5 * q) % 35];
            dft_odd<7, false>(x, nullptr, 7);
#pragma unroll
            for (int q = 0; q < 7; ++q) y[(21 * k1 + 15 * q) % 35] = x[q];
        }
#pragma unroll
        for (int k = 0; k < kT; ++k) z[k] = y[k];
    } else {
#pragma unroll
        for (int k2 = 0; k2 < 7; ++k2) {
            double2 x[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) x[q] = z[(21 * q + 15 * k2) % 35];
            dft_odd<5, true>(x, nullptr, 5);
#pragma unroll
            for (int q = 0; q < 5; ++q) z[(21 * q + 15 * k2) % 35] = x[q];
        }
        double2 y[kT];
#pragma unroll
        for (int t2 = 0; t2 < 5; ++t2) {
            double2 x[7];
#pragma unroll
            for (int q = 0; q < 7; ++q) x[q] = z[(21 * t2 + 15 * q) % 35];
            dft_odd<7, true>(x, nullptr, 7);
#pragma unroll
            for (int q = 0; q < 7; ++q) y[(7 * t2 + 5 * q) % 35] = x[q];
        }
#pragma unroll
        for (int k = 0; k < kT; ++k) z[k] = y[k];
    }
}

// continuation points of lane (c, r): g_j for j = r + 8 q (q < 3), position
// 256 + j = r + 8 (32 + q) (FcOperator::continuation, src/fc_core.cpp:221-238:
// g_j = sum_i A[j][i] f[N-3+i] + sum_i A[23-j][i] f[2-i]); fl[i] = f[2-i],
// fr[i] = f[253+i] of the lane's complex line
FCSG_HD void continuation(int r, double2 (&z)[kT], const double2 (&fr)[kD1], const double2 (&fl)[kD1],
                          const double* blend) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int j = r + 8 * q;
        double2 a = mk2(0.0, 0.0), c = mk2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < kD1; ++i) {
            const double cr = blend[j * kD1 + i], cl = blend[(kGap - 1 - j) * kD1 + i];
            a = mk2(a.x + cr * fr[i].x, a.y + cr * fr[i].y);
            c = mk2(c.x + cl * fl[i].x, c.y + cl * fl[i].y);
        }
        z[32 + q] = cadd(a, c);
    }
}

// lane (c, r): store Y_r[k2] (k2 < 35) of line c
FCSG_HD void put35(double2* buf, int c, int r, const double2 (&z)[kT]) {
    double2* p = buf + c * kPC + r * kT;
#pragma unroll
    for (int k = 0; k < kT; ++k) p[k] = z[k];
}
FCSG_HD void get35(const double2* buf, int c, int r, double2 (&z)[kT]) {
    const double2* p = buf + c * kPC + r * kT;
#pragma unroll
    for (int k = 0; k < kT; ++k) z[k] = p[k];
}

// step 2 for the groups G = lane, lane + NL, ... < 140 of one warp buffer:
// tw = W280^(r k2) at kTwPitch k2 + r (r = 1..7), mult = the multiplier in
// natural frequency order
template <int NL>
FCSG_HD void middle(int lane, double2* buf, const double2* tw, const double2* mult) {
    for (int G = lane; G < kLines * kT; G += NL) {
        const int c = G >= 105 ? 3 : G >= 70 ? 2 : G >= 35 ? 1 : 0;
        const int k2 = G - kT * c;
        double2* p = buf + c * kPC + k2;
        const double2* w = tw + kTwPitch * k2;
        double2 v[8], wr[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = p[r * kT];
#pragma unroll
        for (int r = 1; r < 8; ++r) {
            wr[r] = w[r];
            v[r] = cmul(v[r], wr[r]);
        }
        dft8<false>(v);
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) v[k1] = cmul(v[k1], mult[k2 + kT * k1]);
        dft8<true>(v);
#pragma unroll
        for (int r = 1; r < 8; ++r) v[r] = cmulc(v[r], wr[r]);
#pragma unroll
        for (int r = 0; r < 8; ++r) p[r * kT] = v[r];
    }
}

// the operator tables in a CTA's shared memory: the multiplier of one mode
// in natural frequency order (permuted from the prime-factor order of
// FcPlanDev::mult_pfa: entry (k1 * 5 + k2) * 7 + k3 holds frequency
// f with k1 = f mod 8, k2 = f mod 5, k3 = f mod 7), the twiddles W280^(r k2)
// (from the plan's exp(-2 pi i k / 280) table) and the 24 x 3 blend matrix
constexpr int kBlendSlots = (kGap * kD1 + 1) / 2;
constexpr int kTabSlots = kNE + kTwSlots + kBlendSlots;
FCSG_HD double2 mult_entry(const double2* mult_pfa, int f) {
    return ldg2(mult_pfa + ((f % 8) * 5 + f % 5) * 7 + f % 7);
}
FCSG_HD double2 tw_entry(const double2* tw_src, int k) {
    const int k2 = k / kTwPitch, r = k - kTwPitch * k2;
    return r < 8 ? ldg2(tw_src + r * k2) : mk2(1.0, 0.0);
}
FCSG_HD void stage_tables(int tid, int nthr, const double2* mult_pfa, const double2* tw_src, const double* blend_src,
                          double2* tabs) {
    double2* mult = tabs;
    double2* tw = tabs + kNE;
    double* blend = reinterpret_cast<double*>(tabs + kNE + kTwSlots);
    for (int f = tid; f < kNE; f += nthr) mult[f] = mult_entry(mult_pfa, f);
    for (int k = tid; k < kTwSlots; k += nthr) tw[k] = tw_entry(tw_src, k);
    for (int k = tid; k < kGap * kD1; k += nthr) blend[k] = ldg1(blend_src + k);
}
// the same in two halves for a CTA of NT threads: every table load issued at
// once into registers (load), stored to shared memory later (store), so the
// L2 latency of the tables overlaps the line loads instead of preceding them
template <int NT>
struct TableRegs {
    static constexpr int NM = (kNE + NT - 1) / NT, NW = (kTwSlots + NT - 1) / NT, NB = (kGap * kD1 + NT - 1) / NT;
    double2 m[NM], w[NW];
    double b[NB];
    FCSG_HD void load(int tid, const double2* mult_pfa, const double2* tw_src, const double* blend_src) {
#pragma unroll
        for (int i = 0; i < NM; ++i)
            if (tid + i * NT < kNE) m[i] = mult_entry(mult_pfa, tid + i * NT);
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

}  // namespace wct
}  // namespace fcsg
