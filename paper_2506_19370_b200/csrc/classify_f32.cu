// Steady-step SDNN classifier (phase 0, Classifier::classify over the proxy,
// src/viscosity.cpp:211-251) with an FP32 screening pass and an exact FP64
// decision wherever the screen is not conclusive.
//
// The classifier's output is an argmax (classify_stencil, src/viscosity.cpp:
// 126-133), so an approximate evaluation decides the class exactly whenever
// its logit margin (top1 - top2) exceeds twice a rigorous bound of its error
// against the exact-arithmetic MLP (mlp_f32_margin): then every evaluation
// within that bound -- the reference's FP64 one included, which is within
// ~1e-13 -- has the same argmax. One thread per point:
//   * the row and column windows (start = clamp(pos - 3, 0, n - 7), row /
//     column segments of L-shaped subpatches) are read from the proxy field
//     and normalised in FP64 exactly as normalize_stencil (src/viscosity.cpp:
//     48-59), guard included (class 4);
//   * the 7 -> 16 -> 16 -> 16 -> 16 -> 4 MLP runs in FP32 FMAs with the
//     weights as kernel parameters (constant bank, broadcast to the warp),
//     the point's row and column stencils packed in FFMA2 pairs, tanh on the
//     SFU (|error| <= 4e-7);
//   * a point with a stencil whose FP32 margin is not above the bound is
//     appended to a list, and a second kernel classifies the listed points
//     again in FP64 (classify_stencil: FP64 FMAs, the table tanh) -- ~0.2% of
//     the stencils of the config-5 vortex;
//   * tau = min(row, column), mu_hat = c(tau) h_max S on interior points
//     (preliminary_viscosity, src/viscosity.cpp:240-251).
// The FP64 tensor-core classifier (classify_mma_kernel) stays for step 0,
// where the density windows are classified too.
#include "classify_f32.h"

#include <algorithm>
#include <cmath>

#include "dev.h"
#include "fft_line.h"  // ldg1

namespace fcsg {

// Rigorous bound of |logit_fp32 - logit_exact| for inputs |x| <= 1 (the
// normalised stencil, and tanh outputs for the hidden layers), doubled: with
// u = 2^-24, per layer the error of a pre-activation is at most
//   sum_j |W_ij| E_j  (propagated)  +  (gamma_{n+1} + 2u) (|b_i| + sum_j |W_ij|)
// (n FMAs in sequence plus the bias: gamma_{n+1} = (n+1)u / (1 - (n+1)u);
// 2u for rounding W and b to float), E_0 = u (rounding x to float); tanh is
// 1-Lipschitz and tanh_f32 is within kTanhErr of tanh.
double mlp_f32_margin(const std::vector<double>& w) {
    constexpr double u = 0x1p-24, kTanhErr = 1e-6;  // tanh_f32: 2.5x its measured worst case (4e-7)
    const int rows[kMlpLayers] = {16, 16, 16, 16, 4}, cols[kMlpLayers] = {7, 16, 16, 16, 16};
    std::vector<double> err(7, u), nxt;
    int off = 0;
    double bound = 0.0;
    for (int l = 0; l < kMlpLayers; ++l) {
        const int n = cols[l];
        const double g = (n + 1) * u / (1.0 - (n + 1) * u) + 2.0 * u;
        nxt.assign(rows[l], 0.0);
        for (int i = 0; i < rows[l]; ++i) {
            double prop = 0.0, mag = std::fabs(w[off + rows[l] * n + i]);
            for (int j = 0; j < n; ++j) {
                prop += std::fabs(w[off + i * n + j]) * err[j];
                mag += std::fabs(w[off + i * n + j]);
            }
            nxt[i] = (prop + g * mag) * (1.0 + 1e-12) + (l + 1 < kMlpLayers ? kTanhErr : 0.0);
            if (l + 1 == kMlpLayers) bound = std::max(bound, nxt[i]);
        }
        err = nxt;
        off += rows[l] * n + rows[l];
    }
    if (!std::isfinite(bound)) return INFINITY;
    return 2.0 * bound + 1e-9;
}

MlpF32 mlp_f32_weights(const std::vector<double>& w) {
    MlpF32 m{};
    for (int k = 0; k < kMlpWeights; ++k) m.w[k] = static_cast<float>(w[k]);
    return m;
}

#if FCSG_CUDA
namespace {

constexpr int kF32Threads = 256;

// The point's row and column stencils run as the two halves of packed FP32
// pairs: Blackwell's FFMA2 does both FMAs in one instruction, with the weight
// broadcast from a uniform register (LDCU.128 fetches four), so the MLP costs
// 944 FFMA2 per point instead of 1888 FFMA. Each half rounds exactly as a
// scalar FFMA (IEEE round-to-nearest), so mlp_f32_margin bounds both.
__device__ __forceinline__ float2 dup(float w) { return make_float2(w, w); }

__device__ __forceinline__ float2 tanh_f32x2(float2 z) {
    const float2 a = __fmul2_rn(make_float2(fabsf(z.x), fabsf(z.y)), dup(2.8853900817779268f));  // 2|x| log2 e
    float tx, ty, rx, ry;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(tx) : "f"(a.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ty) : "f"(a.y));
    const float2 d = __fadd2_rn(make_float2(tx, ty), dup(1.0f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rx) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ry) : "f"(d.y));
    const float2 y = __ffma2_rn(dup(-2.0f), make_float2(rx, ry), dup(1.0f));  // 1 - 2 / (e^(2|x|) + 1)
    return make_float2(copysignf(fmaxf(y.x, 0.0f), z.x), copysignf(fmaxf(y.y, 0.0f), z.y));
}

// FP32 forward pass of two normalised stencils (row in .x, column in .y)
__device__ __forceinline__ void forward_f32x2(const MlpF32& W, const float2* x, float2* lg) {
    constexpr int L0 = 16 * 7 + 16, LH = 16 * 16 + 16;
    float2 h[16], g[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        float2 acc = dup(W.w[16 * 7 + i]);
#pragma unroll
        for (int j = 0; j < 7; ++j) acc = __ffma2_rn(dup(W.w[i * 7 + j]), x[j], acc);
        h[i] = tanh_f32x2(acc);
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const int b = L0 + l * LH;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float2 acc = dup(W.w[b + 256 + i]);
#pragma unroll
            for (int j = 0; j < 16; ++j) acc = __ffma2_rn(dup(W.w[b + i * 16 + j]), h[j], acc);
            g[i] = tanh_f32x2(acc);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) h[i] = g[i];
    }
    constexpr int LO = L0 + 3 * LH;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 acc = dup(W.w[LO + 64 + i]);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc = __ffma2_rn(dup(W.w[LO + i * 16 + j]), h[j], acc);
        lg[i] = acc;
    }
}

// normalize_stencil (src/viscosity.cpp:48-59) in FP64: false = the class-4
// guard; else the normalised values rounded to float (the screen needs them
// to ~1e-16 relative, not the reference's exact rounding)
__device__ __forceinline__ bool normalise_f32(const EngineDev& E, const double* s, float* x) {
    double lo = s[0], hi = s[0];
#pragma unroll
    for (int k = 1; k < kMlpIn; ++k) {
        lo = s[k] < lo ? s[k] : lo;
        hi = s[k] > hi ? s[k] : hi;
    }
    const double span = hi - lo;
    double scale = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
    scale = scale > 1e-100 ? scale : 1e-100;
    if (span <= 1e-13 * scale || span <= E.abs_floor) return false;
    const double inv = 2.0 / span;
#pragma unroll
    for (int k = 0; k < kMlpIn; ++k) x[k] = static_cast<float>(fma(s[k] - lo, inv, -1.0));
    return true;
}

// class 1..4 of FP32 logits, 0 when the margin is not above the bound
__device__ __forceinline__ int screen_class(const EngineDev& E, float l0, float l1, float l2, float l3) {
    const float lg[4] = {l0, l1, l2, l3};
    int best = 0;
    float top = lg[0];
#pragma unroll
    for (int k = 1; k < 4; ++k)
        if (lg[k] > top) {
            top = lg[k];
            best = k;
        }
    float second = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (k != best) second = fmaxf(second, lg[k]);
    return static_cast<double>(top) - static_cast<double>(second) > E.cls_margin32 ? best + 1 : 0;
}

// window geometry of point p: subpatch base, (i, j), row / column segment
// begins and the window starts (-1: the segment is shorter than a stencil)
struct PointWin {
    long base;
    int i, j, rst, cst;
    bool inset;
};
__device__ __forceinline__ PointWin point_windows(const EngineDev& E, long p) {
    PointWin w;
    const unsigned pp = static_cast<unsigned>(p);
    const unsigned sub = fdiv(E.div_sz, pp);
    const unsigned loc = pp - sub * E.div_sz.d;
    w.j = static_cast<int>(fdiv(E.div_ni, loc));
    w.i = static_cast<int>(loc) - w.j * E.ni;
    w.base = static_cast<long>(sub) * E.ni * E.nj;
    const int ci = E.cut_i[sub], cj = E.cut_j[sub];
    w.inset = !(w.i < ci && w.j < cj);
    const int rb = w.j < cj ? ci : 0, cb = w.i < ci ? cj : 0;  // row / column segment begin
    w.rst = w.cst = -1;
    if (E.ni - rb >= kMlpIn) {
        const int st = w.i - rb - kMlpIn / 2;
        w.rst = rb + (st < 0 ? 0 : (st > E.ni - rb - kMlpIn ? E.ni - rb - kMlpIn : st));
    }
    if (E.nj - cb >= kMlpIn) {
        const int st = w.j - cb - kMlpIn / 2;
        w.cst = cb + (st < 0 ? 0 : (st > E.nj - cb - kMlpIn ? E.nj - cb - kMlpIn : st));
    }
    return w;
}
__device__ __forceinline__ void row_window(const EngineDev& E, const PointWin& w, double* s) {
    const double* f = E.proxy + w.base + static_cast<long>(w.j) * E.ni + w.rst;
#pragma unroll
    for (int k = 0; k < kMlpIn; ++k) s[k] = ldg1(f + k);
}
__device__ __forceinline__ void col_window(const EngineDev& E, const PointWin& w, double* s) {
    const double* f = E.proxy + w.base + static_cast<long>(w.cst) * E.ni + w.i;
#pragma unroll
    for (int k = 0; k < kMlpIn; ++k) s[k] = ldg1(f + static_cast<long>(k) * E.ni);
}
__device__ __forceinline__ void write_tau(const EngineDev& E, long p, int tau) {
    E.tau[p] = tau;
    E.mu_hat[p] = (E.mask[p] == 1) ? E.visc_c[tau - 1] * E.h_max[p] * E.speed[p] : 0.0;
}

__global__ void __launch_bounds__(kF32Threads, 3) classify_f32_kernel(const __grid_constant__ EngineDev E,
                                                                   const __grid_constant__ MlpF32 W) {
    // one point per thread and no grid-stride loop: in a loop the weights are
    // loop-invariant and ptxas keeps hundreds of them in registers
    const long p = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < E.npts) {
        const PointWin w = point_windows(E, p);
        // per window: 4 (guard / no window) or -1 (to the MLP)
        int cr = 4, cc = 4;
        float xr[kMlpIn], xc[kMlpIn];
        if (w.inset) {
            double s[kMlpIn];
            if (w.rst >= 0) {
                row_window(E, w, s);
                cr = normalise_f32(E, s, xr) ? -1 : 4;
            }
            if (w.cst >= 0) {
                col_window(E, w, s);
                cc = normalise_f32(E, s, xc) ? -1 : 4;
            }
        }
        if (cr < 0 || cc < 0) {
            float2 x[kMlpIn], lg[4];
#pragma unroll
            for (int k = 0; k < kMlpIn; ++k) x[k] = make_float2(cr < 0 ? xr[k] : 0.0f, cc < 0 ? xc[k] : 0.0f);
            forward_f32x2(W, x, lg);
            if (cr < 0) cr = screen_class(E, lg[0].x, lg[1].x, lg[2].x, lg[3].x);
            if (cc < 0) cc = screen_class(E, lg[0].y, lg[1].y, lg[2].y, lg[3].y);
        }
        if (cr == 0 || cc == 0) {  // exact FP64 classification of this point by classify_fix_kernel
            const unsigned k = atomicAdd(E.cls_fix_count, 1u);
            E.cls_fix_list[k] = static_cast<int>(p);
        } else {
            write_tau(E, p, cr < cc ? cr : cc);
        }
    }
}

// the listed points: both windows in FP64 (classify_stencil, as the reference)
__global__ void __launch_bounds__(kF32Threads) classify_fix_kernel(const __grid_constant__ EngineDev E) {
    const unsigned n = *E.cls_fix_count;
    if (static_cast<unsigned>(blockIdx.x) * blockDim.x >= n) return;  // (~0.2% of the points: most blocks idle)
    // the table tanh and the FP64 weights in shared memory: each listed point
    // is one thread's serial FP64 MLP, whose latency is the kernel's
    __shared__ double tab[kTanhTable];
    __shared__ double wt[kMlpWeights];
    for (int k = threadIdx.x; k < kTanhTable; k += blockDim.x) tab[k] = E.tanh_tab[k];
    for (int k = threadIdx.x; k < kMlpWeights; k += blockDim.x) wt[k] = E.mlp[k];
    __syncthreads();
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const long p = E.cls_fix_list[k];
        const PointWin w = point_windows(E, p);
        double s[kMlpIn];
        int tau = 4;
        if (w.rst >= 0) {
            row_window(E, w, s);
            tau = classify_stencil(MlpPtr{wt}, tab, s, E.abs_floor);
        }
        if (w.cst >= 0) {
            col_window(E, w, s);
            const int c = classify_stencil(MlpPtr{wt}, tab, s, E.abs_floor);
            tau = c < tau ? c : tau;
        }
        write_tau(E, p, tau);
    }
}

}  // namespace

void launch_classify_f32(const EngineDev& E, const MlpF32& W, void* stream) {
    if (E.npts == 0) return;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(E.cls_fix_count, 0, sizeof(unsigned), s);
    const long n = (E.npts + kF32Threads - 1) / kF32Threads;
    classify_f32_kernel<<<static_cast<int>(n), kF32Threads, 0, s>>>(E, W);
    // enough threads for one listed point each up to 2% of the points
    const long nfix = std::max(1L, std::min((E.npts / 50 + kF32Threads - 1) / kF32Threads, 148L * 16));
    classify_fix_kernel<<<static_cast<int>(nfix), kF32Threads, 0, s>>>(E);
}
#endif

}  // namespace fcsg
