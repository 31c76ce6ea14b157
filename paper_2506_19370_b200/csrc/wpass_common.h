// Helpers shared by the warp-pass translation units (wpass.cu, wctpass.cu):
// conservative -> primitive conversion and the Euler fluxes
// (src/euler.cpp:29-75), L2 prefetches, the positivity diagnostic.
#pragma once

#include "dev.h"
#include "pass_common.h"
#include "step_kernels.h"

namespace fcsg {

// conservative -> primitive as prim_of (src/euler.cpp:29-41) with one
// reciprocal of the density instead of four divisions per point (the
// products differ from the quotients by an ulp, far inside the parity gates)
// 1/x without the IEEE division's special-case branch: the SFU's approximate
// reciprocal (rcp.approx.ftz.f64, ~2^-23 relative) refined by three Newton
// steps (~2^-52: an ulp). x is a positive, finite density here (a
// nonpositive or non-finite one is reported by the positivity check
// regardless of its reciprocal).
FCSG_HD double recip(double x) {
#if FCSG_CUDA && !defined(FCSG_EXACT_DIV)
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return fma(r, fma(-x, r, 1.0), r);
#else
    return 1.0 / x;
#endif
}
struct PrimR {
    double rho, mx, my, E, ir, theta, p;
};
FCSG_HD PrimR prim_r(double rho, double mx, double my, double E) {
    PrimR q;
    q.rho = rho;
    q.mx = mx;
    q.my = my;
    q.E = E;
    q.ir = recip((rho != 0.0) ? rho : 1e-300);
    const double pr = kGm1 * (E - 0.5 * (mx * mx + my * my) * q.ir);
    q.theta = pr * q.ir;
    q.p = rho * q.theta;
    return q;
}
// x-flux F_c and y-flux G_c (src/euler.cpp:44-55, 64-75)
FCSG_HD double flux_x(const PrimR& q, int c) {
    const double u = q.mx * q.ir;
    switch (c) {
        case 0: return q.mx;
        case 1: return q.mx * u + q.p;
        case 2: return q.my * u;
        default: return u * (q.E + q.p);
    }
}
FCSG_HD double flux_y(const PrimR& q, int c) {
    const double v = q.my * q.ir;
    switch (c) {
        case 0: return q.my;
        case 1: return q.mx * v;
        case 2: return q.my * v + q.p;
        default: return v * (q.E + q.p);
    }
}

// L2 prefetch of one 32-byte sector (the epilogue inputs of the next round,
// issued before the transform so their DRAM latency hides behind it)
FCSG_HD void pf_l2(const double* p) {
#if FCSG_CUDA
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#else
    (void)p;
#endif
}
// L2 prefetch of a contiguous range (bytes a multiple of 16). The bulk
// prefetch needs a 16-byte aligned start; a group view's fields start at the
// group's first point, which is only 8-byte aligned after a group with an odd
// number of points -- then the range is prefetched from its first aligned byte.
FCSG_HD void pf_l2_bulk(const double* p, unsigned bytes) {
#if FCSG_CUDA
    const unsigned long long a = reinterpret_cast<unsigned long long>(p);
    if (a & 15) {
        p += 1;
        bytes -= 16;
    }
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
#else
    (void)p;
    (void)bytes;
#endif
}

// interior positivity diagnostic of euler_rhs (src/euler.cpp:37-39)
FCSG_HD void w_check_positive(const EngineDev& E, double rho, double theta, long p, int sub, int i, int j) {
    const double pr = theta * ((rho != 0.0) ? rho : 1e-300);
    if ((!(rho > 0.0) || !(pr > 0.0) || !finite_d(pr)) && E.mask[p] == 1)
        raise_error(E.sc, 1, E.sub_base + sub, i, j);
}

}  // namespace fcsg
