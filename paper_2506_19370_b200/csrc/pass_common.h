// Device helpers shared by the line-pass translation units (step_kernels.cu,
// wpass.cu): SSPRK(5,4) constants and stage update, conservative ->
// primitive conversion and fluxes (src/euler.cpp), the device error word.
#pragma once

#include <cstring>

#include "fft_line.h"
#include "step_kernels.h"

namespace fcsg {

namespace {
constexpr double kG = 1.4;
constexpr double kGm1 = kG - 1.0;
// include/fcs/euler.hpp:20-29
constexpr double SB0 = 0.391752226571890;
constexpr double SA20 = 0.444370493651235, SA21 = 0.555629506348765, SB1 = 0.368410593050371;
constexpr double SA30 = 0.620101851488403, SA32 = 0.379898148511597, SB2 = 0.251891774271694;
constexpr double SA40 = 0.178079954393132, SA43 = 0.821920045606868, SB3 = 0.544974750228521;
constexpr double SC2 = 0.517231671970585, SC3 = 0.096059710526147, SD3 = 0.063692468666290,
                 SC4 = 0.386708617503269, SD4 = 0.226007483236906;
constexpr int kThreads = 256;
}  // namespace

FCSG_HD void raise_error_at(StepScalars* sc, int code, int sub, int i, int j, long long gp) {
#if FCSG_CUDA
    if (atomicCAS(&sc->err.code, 0, code) == 0) {
        sc->err.sub = sub;
        sc->err.i = i;
        sc->err.j = j;
        sc->err.gp = gp;
    }
#else
    if (sc->err.code == 0) {
        sc->err.code = code;
        sc->err.sub = sub;
        sc->err.i = i;
        sc->err.j = j;
        sc->err.gp = gp;
    }
#endif
}
// (storage slot, i, j) of a group view / a global point index
FCSG_HD void raise_error(StepScalars* sc, int code, int sub, int i, int j) { raise_error_at(sc, code, sub, i, j, -1); }
FCSG_HD void raise_error_gp(StepScalars* sc, int code, long gp) { raise_error_at(sc, code, -1, 0, 0, gp); }

FCSG_HD unsigned long long dbits(double v) {
#if FCSG_CUDA
    return static_cast<unsigned long long>(__double_as_longlong(v));
#else
    unsigned long long u;
    std::memcpy(&u, &v, 8);
    return u;
#endif
}

// 6x6 tensor Lagrange interpolation of field f from stencil origin s0
// (row pitch, weights wx[6] then wy[6]) in the reference's summation order
// (src/runtime.cpp:359-368, 443-451)
FCSG_HD double interp66(const double* f, long s0, int pitch, const double* w) {
    double val = 0.0;
    for (int b = 0; b < 6; ++b) {
        const double* row = f + s0 + static_cast<long>(b) * pitch;
        double sa = 0.0;
        for (int a = 0; a < 6; ++a) sa += w[a] * row[a];
        val += w[6 + b] * sa;
    }
    return val;
}

FCSG_HD bool finite_d(double v) {
#if FCSG_CUDA
    return isfinite(v);
#else
    return std::isfinite(v);
#endif
}

// conservative -> (theta, p) exactly as euler_rhs (src/euler.cpp:29-41,44-55)
struct Prim {
    double rho, mx, my, E, theta, p;
};
// the conserved values at p on the read-only path: no pass reads e at a point
// after writing it there
FCSG_HD void fetch_e(const EngineDev& E, long p, double* v) {
    v[0] = ldg1(E.e[0] + p);
    v[1] = ldg1(E.e[1] + p);
    v[2] = ldg1(E.e[2] + p);
    v[3] = ldg1(E.e[3] + p);
}
FCSG_HD Prim prim_of(const double* v) {
    Prim q;
    q.rho = v[0];
    q.mx = v[1];
    q.my = v[2];
    q.E = v[3];
    const double rs = (q.rho != 0.0) ? q.rho : 1e-300;
    const double pr = kGm1 * (q.E - 0.5 * (q.mx * q.mx + q.my * q.my) / rs);
    q.theta = pr / rs;
    q.p = q.rho * q.theta;
    return q;
}
FCSG_HD Prim prim_rhs(const EngineDev& E, long p) {
    double v[4];
    fetch_e(E, p, v);
    return prim_of(v);
}

// flux pair (F_c, G_c) (src/euler.cpp:44-55, 64-75)
FCSG_HD double2 flux_pair(const Prim& q, int c) {
    const double u = q.mx / q.rho, v = q.my / q.rho;
    switch (c) {
        case 0: return mk2(q.mx, q.my);
        case 1: return mk2(q.mx * u + q.p, q.mx * v);
        case 2: return mk2(q.my * u, q.my * v + q.p);
        default: return mk2(u * (q.E + q.p), v * (q.E + q.p));
    }
}

// SSPRK(5,4) stage update of component c at point p (src/euler.cpp:182-221),
// u = current e[c][p]. The RK registers read here (e0, e2, e3, rhs3) are never
// written in the same stage, so they take the read-only path. At stage 0 the
// register e0 equals e (phase 2 copies e into e0 after the BCs,
// src/runtime.cpp:422), so it is written here instead of in phase 2.
FCSG_HD void ssprk_update(const EngineDev& E, int stage, int c, long p, double u, double r, double dt) {
    if (E.rhs[0]) E.rhs[c][p] = r;
    double* e = E.e[c];
    switch (stage) {
        case 0:
            E.e0[c][p] = u;
            e[p] = u + dt * SB0 * r;
            break;
        case 1: {
            const double nu = SA20 * ldg1(E.e0[c] + p) + SA21 * u + dt * SB1 * r;
            e[p] = nu;
            E.e2[c][p] = nu;
            break;
        }
        case 2: {
            const double nu = SA30 * ldg1(E.e0[c] + p) + SA32 * u + dt * SB2 * r;
            e[p] = nu;
            E.e3[c][p] = nu;
            break;
        }
        case 3:
            E.rhs3[c][p] = r;
            e[p] = SA40 * ldg1(E.e0[c] + p) + SA43 * u + dt * SB3 * r;
            break;
        default:
            e[p] = SC2 * ldg1(E.e2[c] + p) + SC3 * ldg1(E.e3[c] + p) + dt * SD3 * ldg1(E.rhs3[c] + p) + SC4 * u +
                   dt * SD4 * r;
            break;
    }
}

// ssprk_update with the register e0 already read (stages 1-3; other stages
// read what they need themselves)
FCSG_HD void ssprk_update_e0(const EngineDev& E, int stage, int c, long p, double u, double r, double e0v,
                             double dt) {
    if (stage < 1 || stage > 3) {
        ssprk_update(E, stage, c, p, u, r, dt);
        return;
    }
    if (E.rhs[0]) E.rhs[c][p] = r;
    double* e = E.e[c];
    if (stage == 1) {
        const double nu = SA20 * e0v + SA21 * u + dt * SB1 * r;
        e[p] = nu;
        E.e2[c][p] = nu;
    } else if (stage == 2) {
        const double nu = SA30 * e0v + SA32 * u + dt * SB2 * r;
        e[p] = nu;
        E.e3[c][p] = nu;
    } else {
        E.rhs3[c][p] = r;
        e[p] = SA40 * e0v + SA43 * u + dt * SB3 * r;
    }
}

}  // namespace fcsg
