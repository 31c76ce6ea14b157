// The SDNN classifier's exact FP64 pieces shared by the classifier kernels
// (step_kernels.cu, classify_f32.cu): the table tanh and the per-stencil
// MLP of MlpClassifier::forward / classify_stencil.
#pragma once

#include "fcsg_common.h"
#include "step_kernels.h"

namespace fcsg {

// tanh for the classifier: tanh(a + b) = (tanh a + tanh b) / (1 + tanh a tanh b)
// with a = k/64 from a table (tanh of the grid, correctly rounded, kept in
// shared memory) and |b| <= 1/128, where the odd Taylor polynomial through
// b^7 is exact to < 1e-20. Branch-free: |x| is clamped at 20 (tanh = 1.0 in
// double precision there), k = round(64 |x|) comes from the low mantissa bits
// of 64 |x| + 1.5 2^52, and on the GPU the quotient uses the hardware
// reciprocal approximation refined by two Newton steps (the denominator is in
// [1, 2)). Error <= 3 ulp, against ~1e-16 of libm differences between the
// reference and any other build; tau parity is gated on the logit margin
// (> 1e-9) anyway.
FCSG_HD double tanh_tab(double x, const double* tab) {
    constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double ax = fmin(fabs(x), 20.0);
    const double kd = fma(ax, 64.0, kMagic);
#if FCSG_CUDA
    const int k = __double2loint(kd);
#else
    unsigned long long bits;
    std::memcpy(&bits, &kd, 8);
    const int k = static_cast<int>(bits & 0xffffffffu);
#endif
    const double b = fma(kd - kMagic, -0.015625, ax);  // exact
    const double p = b * b;
    const double tb = fma(b * p, fma(p, fma(p, -17.0 / 315.0, 2.0 / 15.0), -1.0 / 3.0), b);
    const double ta = tab[k];
    const double n = ta + tb, d = fma(ta, tb, 1.0);
#if FCSG_CUDA
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    return copysign(n * y, x);
#else
    return std::copysign(n / d, x);
#endif
}

// weights read through a device pointer (FCNN order, per layer W then b)
struct MlpPtr {
    const double* p;
    FCSG_HD double operator()(int k) const { return p[k]; }
};

// MlpClassifier::forward + classify_stencil (src/viscosity.cpp:108-133) on a
// raw 7-point stencil, with normalize_stencil's guard (src/viscosity.cpp:48-59)
template <class WA>
FCSG_HD int classify_stencil(const WA& W, const double* tab, const double* s, double abs_floor) {
    double lo = s[0], hi = s[0];
#pragma unroll
    for (int k = 1; k < kMlpIn; ++k) {
        lo = s[k] < lo ? s[k] : lo;
        hi = s[k] > hi ? s[k] : hi;
    }
    const double span = hi - lo;
    double scale = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
    scale = scale > 1e-100 ? scale : 1e-100;
    if (span <= 1e-13 * scale || span <= abs_floor) return 4;
    double x[kMlpIn];
#pragma unroll
    for (int k = 0; k < kMlpIn; ++k) x[k] = 2.0 * (s[k] - lo) / span - 1.0;
    double h[kMlpHidden], g[kMlpHidden];
    constexpr int L0 = kMlpHidden * kMlpIn + kMlpHidden;     // layer 0 size (W then b)
    constexpr int LH = kMlpHidden * kMlpHidden + kMlpHidden;  // hidden layer size
#pragma unroll
    for (int i = 0; i < kMlpHidden; ++i) {
        double acc = W(kMlpHidden * kMlpIn + i);
#pragma unroll
        for (int j = 0; j < kMlpIn; ++j) acc += W(i * kMlpIn + j) * x[j];
        h[i] = tanh_tab(acc, tab);
    }
#pragma unroll
    for (int layer = 0; layer < 3; ++layer) {
        const int base = L0 + layer * LH;
#pragma unroll
        for (int i = 0; i < kMlpHidden; ++i) {
            double acc = W(base + kMlpHidden * kMlpHidden + i);
#pragma unroll
            for (int j = 0; j < kMlpHidden; ++j) acc += W(base + i * kMlpHidden + j) * h[j];
            g[i] = tanh_tab(acc, tab);
        }
#pragma unroll
        for (int i = 0; i < kMlpHidden; ++i) h[i] = g[i];
    }
    constexpr int LO = L0 + 3 * LH;
    double lg[kMlpOut];
#pragma unroll
    for (int i = 0; i < kMlpOut; ++i) {
        double acc = W(LO + kMlpOut * kMlpHidden + i);
#pragma unroll
        for (int j = 0; j < kMlpHidden; ++j) acc += W(LO + i * kMlpHidden + j) * h[j];
        lg[i] = acc;
    }
    int best = 0;
#pragma unroll
    for (int k = 1; k < kMlpOut; ++k)
        if (lg[k] > lg[best]) best = k;
    return best + 1;
}

}  // namespace fcsg
