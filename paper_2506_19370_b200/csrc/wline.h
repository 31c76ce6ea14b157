// Warp-owned FC line transform for n_ext = 280 = 8 * 5 * 7 (N = 256 points,
// the reference operator: n_cont = 25, degree 2): the FcOperator pipeline of
// src/fc_core.cpp:221-238,257-297 (continuation -> DFT -> spectral multiplier
// -> inverse DFT) for ONE complex line (two real lines) per warp, with no
// block-level barrier: the line lives in a per-warp shared-memory buffer and
// the lanes synchronise with __syncwarp only.
//
// The DFT is a prime-factor (Good-Thomas) algorithm: the factors 8, 5 and 7
// are coprime, so with the index maps
//     n = (35 n1 + 56 n2 + 40 n3) mod 280          (input, CRT/Ruritanian)
//     k = (105 k1 + 56 k2 + 120 k3) mod 280        (output, CRT)
// (35*105 = 35 (mod 280), 56*56 = 56, 40*120 = 40, every cross product a
// multiple of 280) the length-280 DFT is exactly the 3-D DFT of the array
// A[n1][n2][n3] = x[n(n1,n2,n3)] of shape 8 x 5 x 7 -- no twiddle factors
// between the stages. The inverse DFT has the same structure, so the input
// map places the data, the spectral multiplier is stored in (k1,k2,k3) order
// (FcTables::mult_pfa) and the inverse's output lands back on the input map:
// no permutation pass. Stages: DFT-8 over n1 (35 butterflies), DFT-5 over n2
// (56), then DFT-7 over n3 fused with the multiplier and the inverse DFT-7
// (40), inverse DFT-5, inverse DFT-8. Each butterfly is held in registers;
// the radix-5/7/8 kernels are fft_line.h's (compile-time roots).
//
// Shared-memory layout of the 8 x 5 x 7 array: slot(n1,n2,n3) =
// 39 n1 + 7 n2 + n3 (312 slots of 16 bytes). The pitch 39 = 7 (mod 8) keeps
// the DFT-8 and DFT-5 stages free of bank conflicts (consecutive lanes on
// consecutive 16-byte bank groups).
#pragma once

#include "fft_line.h"

#if FCSG_CUDA
#define FCSG_SYNCWARP() __syncwarp()
#else
#define FCSG_SYNCWARP() ((void)0)
#endif

namespace fcsg {
namespace w280 {

constexpr int kN = 256;      // points per line
constexpr int kNE = 280;     // n_ext
constexpr int kGap = 24;     // n_cont - 1
constexpr int kD1 = 3;       // degree + 1
constexpr int kP1 = 39;      // slot pitch of n1
constexpr int kSlots = 8 * kP1;  // 312 double2 per line buffer

// slot of natural position i (0 <= i < 280): n1 = 3 i mod 8, n2 = i mod 5,
// n3 = 3 i mod 7 (the inverse of the input map)
FCSG_HD int slot_of(int i) {
    const int n1 = (3 * i) & 7;
    const int n2 = i - 5 * ((i * 205) >> 10);           // i mod 5, i < 1024
    const int t = 3 * i;
    const int n3 = t - 7 * ((t * 2341) >> 14);          // t mod 7, t < 2340
    return kP1 * n1 + 7 * n2 + n3;
}

// The transform of NLINES complex lines held in buffers buf + l * pitch
// (natural position i at slot_of(i), i < 256, already written and
// synchronised by the caller): continuation (FcOperator::continuation,
// src/fc_core.cpp:221-238: g_j = sum_i A[j][i] f[N-3+i] + sum_i A[23-j][i]
// f[2-i]), forward PFA DFT, multiplier
// `mult` (280 double2 in (k1,k2,k3) order, k3 fastest), inverse PFA DFT.
// Unnormalised like FFTW's c2r: the multiplier tables carry 1/n_ext. blend
// and mult are the kernels' shared-memory copies of the operator tables. The
// butterflies of all lines share each stage's loop, so two lines per warp
// fill 70 / 112 / 80 butterfly slots per stage instead of 35 / 56 / 40 (the
// remainder iterations of one line leave most lanes idle). Ends
// synchronised; result at slot_of(i).
template <int NL, int NLINES>
FCSG_HD void transform(int lane, double2* buf, int pitch, const double2* mult, const double* blend) {
    for (int t = lane; t < NLINES * kGap; t += NL) {
        const int l = t / kGap, j = t - l * kGap;
        double2* b = buf + l * pitch;
        double2 a = mk2(0.0, 0.0), c = mk2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < kD1; ++i) {
            const double2 fr = b[slot_of(kN - kD1 + i)];
            const double2 fl = b[slot_of(kD1 - 1 - i)];
            const double cr = blend[j * kD1 + i], cl = blend[(kGap - 1 - j) * kD1 + i];
            a = mk2(a.x + cr * fr.x, a.y + cr * fr.y);
            c = mk2(c.x + cl * fl.x, c.y + cl * fl.y);
        }
        b[slot_of(kN + j)] = cadd(a, c);
    }
    FCSG_SYNCWARP();
    // DFT-8 over n1: butterfly bb = (n2, n3) at slots bb + 39 n1
    for (int b = lane; b < NLINES * 35; b += NL) {
        const int l = b / 35;
        double2* p = buf + l * pitch + (b - 35 * l);
        double2 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = p[kP1 * q];
        dft8<false>(x);
#pragma unroll
        for (int q = 0; q < 8; ++q) p[kP1 * q] = x[q];
    }
    FCSG_SYNCWARP();
    // DFT-5 over n2: butterfly bb = 7 n1 + n3 at slots 39 n1 + n3 + 7 q
    for (int b = lane; b < NLINES * 56; b += NL) {
        const int l = b / 56, bb = b - 56 * l;
        const int n1 = (bb * 37) >> 8;  // bb / 7 for bb < 56
        double2* p = buf + l * pitch + kP1 * n1 + (bb - 7 * n1);
        double2 x[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) x[q] = p[7 * q];
        dft_odd<5, false>(x, nullptr, 5);
#pragma unroll
        for (int q = 0; q < 5; ++q) p[7 * q] = x[q];
    }
    FCSG_SYNCWARP();
    // DFT-7 over n3, multiplier, inverse DFT-7: butterfly bb = k1 + 8 k2 at
    // slots 39 k1 + 7 k2 + q (k1 fastest across lanes: 39 k1 = 7 k1 mod 8
    // spreads 8 lanes over the 8 bank groups); multiplier index
    // 7 (5 k1 + k2) + q
    for (int b = lane; b < NLINES * 40; b += NL) {
        const int l = b / 40, bb = b - 40 * l;
        const int k1 = bb & 7, k2 = bb >> 3;
        double2* p = buf + l * pitch + kP1 * k1 + 7 * k2;
        const double2* mk = mult + 7 * (5 * k1 + k2);
        double2 x[7];
#pragma unroll
        for (int q = 0; q < 7; ++q) x[q] = p[q];
        dft_odd<7, false>(x, nullptr, 7);
#pragma unroll
        for (int q = 0; q < 7; ++q) x[q] = cmul(x[q], mk[q]);
        dft_odd<7, true>(x, nullptr, 7);
#pragma unroll
        for (int q = 0; q < 7; ++q) p[q] = x[q];
    }
    FCSG_SYNCWARP();
    for (int b = lane; b < NLINES * 56; b += NL) {
        const int l = b / 56, bb = b - 56 * l;
        const int n1 = (bb * 37) >> 8;
        double2* p = buf + l * pitch + kP1 * n1 + (bb - 7 * n1);
        double2 x[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) x[q] = p[7 * q];
        dft_odd<5, true>(x, nullptr, 5);
#pragma unroll
        for (int q = 0; q < 5; ++q) p[7 * q] = x[q];
    }
    FCSG_SYNCWARP();
    for (int b = lane; b < NLINES * 35; b += NL) {
        const int l = b / 35;
        double2* p = buf + l * pitch + (b - 35 * l);
        double2 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = p[kP1 * q];
        dft8<true>(x);
#pragma unroll
        for (int q = 0; q < 8; ++q) p[kP1 * q] = x[q];
    }
    FCSG_SYNCWARP();
}

}  // namespace w280
}  // namespace fcsg
