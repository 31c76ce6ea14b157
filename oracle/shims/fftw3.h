/*
 * TEST INFRASTRUCTURE ONLY (oracle build shim) -- never linked into the product.
 *
 * Stand-in for the five FFTW3 entry points the reference's src/fc_core.cpp
 * uses (fc_core.cpp:3,185-186,211-216,263,282,291,295,312,327):
 *   fftw_plan_dft_r2c_1d / fftw_plan_dft_c2r_1d (FFTW_ESTIMATE|FFTW_UNALIGNED),
 *   fftw_execute_dft_r2c / fftw_execute_dft_c2r (new-array execute),
 *   fftw_destroy_plan.
 * FFTW is absent from this image and the reference pins no version, so this
 * header restates FFTW's published transform definitions:
 *   r2c: Y[k] = sum_j x[j] exp(-2 pi i j k / n), k = 0..n/2 (unnormalised)
 *   c2r: y[j] = sum_{k=0}^{n-1} Y[k] exp(+2 pi i j k / n) over the Hermitian
 *        extension of the n/2+1 input bins; the imaginary parts of the DC and
 *        (even n) Nyquist bins are ignored, as FFTW does (unnormalised).
 *
 * Algorithm (chosen so the CPU baseline is not handicapped by the shim; complex
 * products written out, see cmul):
 * even n uses the standard half-length packing (z_k = x_2k + i x_2k+1, one
 * complex FFT of n/2 and an O(n) split); the complex FFT is an iterative
 * Stockham autosort mixed-radix transform (split real / imaginary arrays,
 * per-stage twiddle tables precomputed in long double, hand-written radix
 * 2/3/4/5/8 butterflies, a symmetric-pair direct DFT for odd factors >= 7). Plans are immutable; execution uses thread_local scratch, so
 * one plan may run concurrently on several threads (fc_core.cpp:174).
 * Large prime factors (67 in n=536, 47, 283) cost O(p) per point here where
 * FFTW uses Rader's algorithm, so timings at such lengths are pessimistic.
 */
#ifndef ORACLE_SHIM_FFTW3_H
#define ORACLE_SHIM_FFTW3_H

#include <cmath>
#include <complex>
#include <vector>

typedef double fftw_complex[2];

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

namespace oracle_fftw {

using cd = std::complex<double>;

// complex products written out: std::complex's operator* goes through
// __muldc3 (the C99 Annex G infinity / NaN recovery, a library call per
// product) unless -fcx-limited-range; for finite operands the result is the
// same as this textbook form
inline cd cmul(cd a, cd b) {
    return cd(a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real());
}
inline cd mul_i(cd a, double s) { return cd(-s * a.imag(), s * a.real()); }  // a * (i s)

// Iterative Stockham (autosort) mixed-radix complex FFT: per stage of radix
// p with Ns = product of the earlier radices, butterfly j (< m/p) gathers
// x[j + r m/p] (r < p), multiplies by the stage twiddles exp(-+2 pi i r k /
// (Ns p)) (k = j mod Ns, precomputed in long double per stage), runs the
// p-point DFT and scatters to (j / Ns) Ns p + k + r Ns: natural order in and
// out, ping-pong buffers, no recursion, no index arithmetic beyond the loop.
struct CPlan {  // complex FFT of length m
    int m = 0;
    std::vector<int> factors;                 // radices in stage order (8s and 4s first)
    std::vector<std::vector<double>> twr, twi;  // per stage: Ns * p twiddles, [k][r]
    std::vector<std::vector<double>> pc, ps;    // per stage (odd p > 7): cos / sin(2 pi k / p)
};

inline void make_cplan(CPlan& c, int m) {
    c.m = m;
    const long double two_pi = 6.283185307179586476925286766559005768L;
    int r = m;
    while (r % 8 == 0) { c.factors.push_back(8); r /= 8; }
    while (r % 4 == 0) { c.factors.push_back(4); r /= 4; }
    while (r % 2 == 0) { c.factors.push_back(2); r /= 2; }
    for (int f = 3; f * f <= r; f += 2)
        while (r % f == 0) { c.factors.push_back(f); r /= f; }
    if (r > 1) c.factors.push_back(r);
    long ns = 1;
    for (int p : c.factors) {
        std::vector<double> tr(ns * p), ti(ns * p), co, si;
        for (long k = 0; k < ns; ++k)
            for (int q = 0; q < p; ++q) {
                const long double a = two_pi * static_cast<long double>(q * k) / static_cast<long double>(ns * p);
                tr[k * p + q] = static_cast<double>(cosl(a));
                ti[k * p + q] = static_cast<double>(-sinl(a));
            }
        if (p > 7 && p != 8) {
            co.resize(p);
            si.resize(p);
            for (int k = 0; k < p; ++k) {
                const long double a = two_pi * k / p;
                co[k] = static_cast<double>(cosl(a));
                si[k] = static_cast<double>(sinl(a));
            }
        }
        c.twr.push_back(std::move(tr));
        c.twi.push_back(std::move(ti));
        c.pc.push_back(std::move(co));
        c.ps.push_back(std::move(si));
        ns *= p;
    }
}

// y_q = sum_r t_r exp(sgn 2 pi i r q / p), in place on (re, im)[0..p);
// sgn = -1 forward, +1 inverse
template <int P>
inline void dft_fixed(double* re, double* im, double sg);

template <>
inline void dft_fixed<2>(double* re, double* im, double) {
    const double ar = re[0], ai = im[0];
    re[0] = ar + re[1];
    im[0] = ai + im[1];
    re[1] = ar - re[1];
    im[1] = ai - im[1];
}
template <>
inline void dft_fixed<3>(double* re, double* im, double sg) {
    const double s3 = 0.86602540378443864676 * sg;
    const double ar = re[1] + re[2], ai = im[1] + im[2];
    const double br = re[1] - re[2], bi = im[1] - im[2];
    const double mr = re[0] - 0.5 * ar, mi = im[0] - 0.5 * ai;
    re[0] += ar;
    im[0] += ai;
    // b * (i s3) = (-s3 bi, s3 br)
    re[1] = mr - s3 * bi;
    im[1] = mi + s3 * br;
    re[2] = mr + s3 * bi;
    im[2] = mi - s3 * br;
}
template <>
inline void dft_fixed<4>(double* re, double* im, double sg) {
    const double ar = re[0] + re[2], ai = im[0] + im[2], br = re[0] - re[2], bi = im[0] - im[2];
    const double dr = re[1] + re[3], di = im[1] + im[3];
    const double er = -sg * (im[1] - im[3]), ei = sg * (re[1] - re[3]);  // (x1 - x3) (i sg)
    re[0] = ar + dr;
    im[0] = ai + di;
    re[2] = ar - dr;
    im[2] = ai - di;
    re[1] = br + er;
    im[1] = bi + ei;
    re[3] = br - er;
    im[3] = bi - ei;
}
template <>
inline void dft_fixed<5>(double* re, double* im, double sg) {
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double s1 = 0.95105651629515357212 * sg, s2 = 0.58778525229247312917 * sg;
    const double a1r = re[1] + re[4], a1i = im[1] + im[4], b1r = re[1] - re[4], b1i = im[1] - im[4];
    const double a2r = re[2] + re[3], a2i = im[2] + im[3], b2r = re[2] - re[3], b2i = im[2] - im[3];
    const double r1r = re[0] + c1 * a1r + c2 * a2r, r1i = im[0] + c1 * a1i + c2 * a2i;
    const double r2r = re[0] + c2 * a1r + c1 * a2r, r2i = im[0] + c2 * a1i + c1 * a2i;
    const double u1r = s1 * b1r + s2 * b2r, u1i = s1 * b1i + s2 * b2i;  // times i
    const double u2r = s2 * b1r - s1 * b2r, u2i = s2 * b1i - s1 * b2i;
    re[0] += a1r + a2r;
    im[0] += a1i + a2i;
    re[1] = r1r - u1i;
    im[1] = r1i + u1r;
    re[4] = r1r + u1i;
    im[4] = r1i - u1r;
    re[2] = r2r - u2i;
    im[2] = r2i + u2r;
    re[3] = r2r + u2i;
    im[3] = r2i - u2r;
}
template <>
inline void dft_fixed<8>(double* re, double* im, double sg) {
    // two radix-4 halves (even / odd samples), twiddles exp(sg i pi k / 4)
    double er[4] = {re[0], re[2], re[4], re[6]}, ei[4] = {im[0], im[2], im[4], im[6]};
    double orr[4] = {re[1], re[3], re[5], re[7]}, oi[4] = {im[1], im[3], im[5], im[7]};
    dft_fixed<4>(er, ei, sg);
    dft_fixed<4>(orr, oi, sg);
    const double h = 0.70710678118654752440;
    // o_k *= w^k, w = exp(sg i pi / 4)
    const double w1r = h, w1i = sg * h, w3r = -h, w3i = sg * h;
    double t;
    t = orr[1] * w1r - oi[1] * w1i;
    oi[1] = orr[1] * w1i + oi[1] * w1r;
    orr[1] = t;
    t = -sg * oi[2];  // times i sg
    oi[2] = sg * orr[2];
    orr[2] = t;
    t = orr[3] * w3r - oi[3] * w3i;
    oi[3] = orr[3] * w3i + oi[3] * w3r;
    orr[3] = t;
    for (int k = 0; k < 4; ++k) {
        re[k] = er[k] + orr[k];
        im[k] = ei[k] + oi[k];
        re[k + 4] = er[k] - orr[k];
        im[k + 4] = ei[k] - oi[k];
    }
}

template <>
inline void dft_fixed<7>(double* re, double* im, double sg) {
    const double c1 = 0.62348980185873353053, c2 = -0.22252093395631440429, c3 = -0.90096886790241912624;
    const double s1 = 0.78183148246802980871 * sg, s2 = 0.97492791218182360702 * sg,
                 s3 = 0.43388373911755812048 * sg;
    const double a1r = re[1] + re[6], a1i = im[1] + im[6], b1r = re[1] - re[6], b1i = im[1] - im[6];
    const double a2r = re[2] + re[5], a2i = im[2] + im[5], b2r = re[2] - re[5], b2i = im[2] - im[5];
    const double a3r = re[3] + re[4], a3i = im[3] + im[4], b3r = re[3] - re[4], b3i = im[3] - im[4];
    const double r1r = re[0] + c1 * a1r + c2 * a2r + c3 * a3r, r1i = im[0] + c1 * a1i + c2 * a2i + c3 * a3i;
    const double r2r = re[0] + c2 * a1r + c3 * a2r + c1 * a3r, r2i = im[0] + c2 * a1i + c3 * a2i + c1 * a3i;
    const double r3r = re[0] + c3 * a1r + c1 * a2r + c2 * a3r, r3i = im[0] + c3 * a1i + c1 * a2i + c2 * a3i;
    // u_q = sum_k b_k sin(2 pi k q / 7) sg, the odd part times i
    const double u1r = s1 * b1r + s2 * b2r + s3 * b3r, u1i = s1 * b1i + s2 * b2i + s3 * b3i;
    const double u2r = s2 * b1r - s3 * b2r - s1 * b3r, u2i = s2 * b1i - s3 * b2i - s1 * b3i;
    const double u3r = s3 * b1r - s1 * b2r + s2 * b3r, u3i = s3 * b1i - s1 * b2i + s2 * b3i;
    re[0] += a1r + a2r + a3r;
    im[0] += a1i + a2i + a3i;
    re[1] = r1r - u1i;
    im[1] = r1i + u1r;
    re[6] = r1r + u1i;
    im[6] = r1i - u1r;
    re[2] = r2r - u2i;
    im[2] = r2i + u2r;
    re[5] = r2r + u2i;
    im[5] = r2i - u2r;
    re[3] = r3r - u3i;
    im[3] = r3i + u3r;
    re[4] = r3r + u3i;
    im[4] = r3i - u3r;
}

// odd p > 7: the symmetric-pair direct DFT
inline void dft_odd_generic(double* re, double* im, int p, double sg, const std::vector<double>& co,
                            const std::vector<double>& si, double* tmp) {
    const int h = (p - 1) / 2;
    double* ar = tmp;
    double* ai = tmp + h;
    double* br = tmp + 2 * h;
    double* bi = tmp + 3 * h;
    double* yr = tmp + 4 * h;
    double* yi = tmp + 4 * h + p;
    double y0r = re[0], y0i = im[0];
    for (int k = 1; k <= h; ++k) {
        ar[k - 1] = re[k] + re[p - k];
        ai[k - 1] = im[k] + im[p - k];
        br[k - 1] = re[k] - re[p - k];
        bi[k - 1] = im[k] - im[p - k];
        y0r += ar[k - 1];
        y0i += ai[k - 1];
    }
    for (int q = 1; q <= h; ++q) {
        double rr = re[0], ri = im[0], ir = 0.0, ii = 0.0;
        int idx = 0;
        for (int k = 0; k < h; ++k) {
            idx += q;
            if (idx >= p) idx -= p;
            rr += ar[k] * co[idx];
            ri += ai[k] * co[idx];
            ir += br[k] * si[idx];
            ii += bi[k] * si[idx];
        }
        // sum b_k (i sg sin) = i sg (ir + i ii) = (-sg ii, sg ir)
        yr[q] = rr - sg * ii;
        yi[q] = ri + sg * ir;
        yr[p - q] = rr + sg * ii;
        yi[p - q] = ri - sg * ir;
    }
    re[0] = y0r;
    im[0] = y0i;
    for (int q = 1; q < p; ++q) {
        re[q] = yr[q];
        im[q] = yi[q];
    }
}

template <int P>
inline void stockham_stage(const double* xr, const double* xi, double* yr, double* yi, int m, long ns,
                           const double* twr, const double* twi, double sg, int pg, const std::vector<double>& co,
                           const std::vector<double>& si, double* tmp) {
    const int p = P > 0 ? P : pg;
    const long stride = m / p;
    double fr[P > 0 ? P : 1], fi[P > 0 ? P : 1];
    thread_local std::vector<double> vr_, vi_;
    if (P == 0 && static_cast<int>(vr_.size()) < p) {
        vr_.resize(p);
        vi_.resize(p);
    }
    double* ar = P > 0 ? fr : vr_.data();
    double* ai = P > 0 ? fi : vi_.data();
    for (long jb = 0, j = 0; jb < stride / ns; ++jb)
    for (long k = 0; k < ns; ++k, ++j) {  // j = jb ns + k: no integer division
        const double* wr = twr + k * p;
        const double* wi = twi + k * p;
        for (int r = 0; r < p; ++r) {
            const double vr = xr[j + r * stride], vi = xi[j + r * stride];
            const double tr = wr[r], ti = sg < 0 ? wi[r] : -wi[r];  // inverse: conjugate twiddles
            ar[r] = vr * tr - vi * ti;
            ai[r] = vr * ti + vi * tr;
        }
        if constexpr (P > 0) dft_fixed<P>(ar, ai, sg);
        else dft_odd_generic(ar, ai, p, sg, co, si, tmp);
        const long base = jb * ns * p + k;
        for (int r = 0; r < p; ++r) {
            yr[base + r * ns] = ar[r];
            yi[base + r * ns] = ai[r];
        }
    }
}

inline std::vector<double>& scratch(int which, size_t n) {
    thread_local std::vector<double> s[6];
    if (s[which].size() < n) s[which].resize(n);
    return s[which];
}

// out = DFT_m(in) (inv: the unnormalised inverse); in and out may not alias
inline void cfft(const CPlan& c, const cd* in, cd* out, bool inv) {
    const int m = c.m;
    auto& ar = scratch(2, m);
    auto& ai = scratch(3, m);
    auto& br = scratch(4, m);
    auto& bi = scratch(5, m);
    thread_local std::vector<double> tmp;
    if (tmp.size() < 8 * static_cast<size_t>(m) + 16) tmp.resize(8 * static_cast<size_t>(m) + 16);
    for (int j = 0; j < m; ++j) {
        ar[j] = in[j].real();
        ai[j] = in[j].imag();
    }
    const double sg = inv ? 1.0 : -1.0;
    double *xr = ar.data(), *xi = ai.data(), *yr = br.data(), *yi = bi.data();
    long ns = 1;
    for (size_t s = 0; s < c.factors.size(); ++s) {
        const int p = c.factors[s];
        const double* twr = c.twr[s].data();
        const double* twi = c.twi[s].data();
        switch (p) {
            case 2: stockham_stage<2>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
            case 3: stockham_stage<3>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
            case 4: stockham_stage<4>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
            case 5: stockham_stage<5>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
            case 7: stockham_stage<7>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
            case 8: stockham_stage<8>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
            default: stockham_stage<0>(xr, xi, yr, yi, m, ns, twr, twi, sg, p, c.pc[s], c.ps[s], tmp.data()); break;
        }
        std::swap(xr, yr);
        std::swap(xi, yi);
        ns *= p;
    }
    for (int j = 0; j < m; ++j) out[j] = cd(xr[j], xi[j]);
}

}  // namespace oracle_fftw

namespace oracle_fftw {
inline std::vector<cd>& cscratch(int which, size_t n) {
    thread_local std::vector<cd> s[2];
    if (s[which].size() < n) s[which].resize(n);
    return s[which];
}
}  // namespace oracle_fftw

struct oracle_fftw_plan_s {
    int n = 0;
    bool half = false;               // even n: half-length packing
    oracle_fftw::CPlan c;            // complex plan of length n/2 (half) or n
    std::vector<oracle_fftw::cd> w;  // exp(-2 pi i k / n), k < n/2 (half packing split)
};
typedef oracle_fftw_plan_s* fftw_plan;

namespace oracle_fftw {
inline fftw_plan make_plan(int n) {
    auto* p = new oracle_fftw_plan_s;
    p->n = n;
    p->half = (n % 2 == 0) && n >= 4;
    make_cplan(p->c, p->half ? n / 2 : n);
    if (p->half) {
        const long double two_pi = 6.283185307179586476925286766559005768L;
        p->w.resize(n / 2 + 1);
        for (int k = 0; k <= n / 2; ++k) {
            const long double a = two_pi * k / n;
            p->w[k] = cd(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
        }
    }
    return p;
}
}  // namespace oracle_fftw

inline fftw_plan fftw_plan_dft_r2c_1d(int n, double*, fftw_complex*, unsigned) { return oracle_fftw::make_plan(n); }
inline fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex*, double*, unsigned) { return oracle_fftw::make_plan(n); }
inline void fftw_destroy_plan(fftw_plan p) { delete p; }

inline void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
    using oracle_fftw::cd;
    const int n = p->n;
    if (!p->half) {
        auto& a = oracle_fftw::cscratch(0, n);
        auto& b = oracle_fftw::cscratch(1, n);
        for (int j = 0; j < n; ++j) a[j] = cd(in[j], 0.0);
        oracle_fftw::cfft(p->c, a.data(), b.data(), false);
        for (int k = 0; k <= n / 2; ++k) {
            out[k][0] = b[k].real();
            out[k][1] = b[k].imag();
        }
        out[0][1] = 0.0;
        return;
    }
    const int h = n / 2;
    auto& a = oracle_fftw::cscratch(0, h);
    auto& Z = oracle_fftw::cscratch(1, h);
    for (int j = 0; j < h; ++j) a[j] = cd(in[2 * j], in[2 * j + 1]);
    oracle_fftw::cfft(p->c, a.data(), Z.data(), false);
    // X_k = (Z_k + conj Z_{h-k})/2 - i w^k (Z_k - conj Z_{h-k})/2
    for (int k = 0; k <= h; ++k) {
        const cd zk = Z[k == h ? 0 : k], zc = std::conj(Z[k == 0 ? 0 : h - k]);
        const cd e = 0.5 * (zk + zc), o = 0.5 * (zk - zc);
        const cd x = e + oracle_fftw::mul_i(oracle_fftw::cmul(p->w[k], o), -1.0);
        out[k][0] = x.real();
        out[k][1] = x.imag();
    }
    out[0][1] = 0.0;
    out[h][1] = 0.0;
}

inline void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
    using oracle_fftw::cd;
    const int n = p->n;
    if (!p->half) {
        auto& a = oracle_fftw::cscratch(0, n);
        auto& b = oracle_fftw::cscratch(1, n);
        a[0] = cd(in[0][0], 0.0);
        for (int k = 1; k <= n / 2; ++k) {
            a[k] = cd(in[k][0], in[k][1]);
            a[n - k] = std::conj(a[k]);
        }
        oracle_fftw::cfft(p->c, a.data(), b.data(), true);
        for (int j = 0; j < n; ++j) out[j] = b[j].real();
        return;
    }
    const int h = n / 2;
    auto& a = oracle_fftw::cscratch(0, h);
    auto& z = oracle_fftw::cscratch(1, h);
    // inverse of the split: Z_k = E_k + i conj(w^k) O_k with
    // E_k = X_k + conj X_{h-k}, O_k = X_k - conj X_{h-k} (DC/Nyquist imag ignored)
    auto X = [&](int k) {
        cd v(in[k][0], in[k][1]);
        if (k == 0 || k == h) v = cd(v.real(), 0.0);
        return v;
    };
    for (int k = 0; k < h; ++k) {
        const cd xk = X(k), xc = std::conj(X(h - k));
        const cd e = xk + xc, o = xk - xc;
        a[k] = e + oracle_fftw::mul_i(oracle_fftw::cmul(std::conj(p->w[k]), o), 1.0);
    }
    oracle_fftw::cfft(p->c, a.data(), z.data(), true);
    for (int j = 0; j < h; ++j) {
        out[2 * j] = z[j].real();
        out[2 * j + 1] = z[j].imag();
    }
}

#endif
