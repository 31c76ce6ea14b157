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
 * Algorithm (chosen so the CPU baseline is not handicapped by the shim):
 * even n uses the standard half-length packing (z_k = x_2k + i x_2k+1, one
 * complex FFT of n/2 and an O(n) split); the complex FFT is a recursive
 * mixed-radix decimation in time with precomputed twiddles (no modular
 * arithmetic in the inner loops), hand-written radix 2/3/4/5 butterflies and
 * a symmetric-pair direct DFT for larger odd factors. Twiddles are computed in
 * long double. Plans are immutable; execution uses thread_local scratch, so
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

struct CPlan {  // complex FFT of length m
    int m = 0;
    std::vector<int> factors;
    std::vector<cd> tw;  // exp(-2 pi i k / m), k < m
    // per odd radix p > 5: cos/sin(2 pi k / p), k = 0..p-1
    std::vector<std::vector<double>> pc, ps;
    std::vector<int> pidx;  // radix -> index into pc/ps (or -1)
};

inline void make_cplan(CPlan& c, int m) {
    c.m = m;
    const long double two_pi = 6.283185307179586476925286766559005768L;
    c.tw.resize(m);
    for (int k = 0; k < m; ++k) {
        const long double a = two_pi * k / m;
        c.tw[k] = cd(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    int r = m;
    while (r % 4 == 0) { c.factors.push_back(4); r /= 4; }
    while (r % 2 == 0) { c.factors.push_back(2); r /= 2; }
    for (int f = 3; f * f <= r; f += 2)
        while (r % f == 0) { c.factors.push_back(f); r /= f; }
    if (r > 1) c.factors.push_back(r);
    c.pidx.assign(m + 1, -1);
    for (int p : c.factors)
        if (p > 5 && c.pidx[p] < 0) {
            c.pidx[p] = static_cast<int>(c.pc.size());
            std::vector<double> co(p), si(p);
            for (int k = 0; k < p; ++k) {
                const long double a = two_pi * k / p;
                co[k] = static_cast<double>(cosl(a));
                si[k] = static_cast<double>(sinl(a));
            }
            c.pc.push_back(co);
            c.ps.push_back(si);
        }
}

// y_q = sum_r t_r exp(sgn 2 pi i r q / p), in place on t[0..p)
inline void small_dft(cd* t, int p, bool inv, const CPlan& c, cd* tmp) {
    const double s = inv ? 1.0 : -1.0;
    if (p == 2) {
        const cd a = t[0], b = t[1];
        t[0] = a + b;
        t[1] = a - b;
    } else if (p == 4) {
        const cd a = t[0] + t[2], b = t[0] - t[2], d = t[1] + t[3];
        const cd e = (t[1] - t[3]) * cd(0, s);
        t[0] = a + d;
        t[2] = a - d;
        t[1] = b + e;
        t[3] = b - e;
    } else if (p == 3) {
        const double c3 = -0.5, s3 = 0.86602540378443864676 * s;
        const cd a = t[1] + t[2], b = (t[1] - t[2]) * cd(0, s3);
        const cd m0 = t[0] + c3 * a;
        t[0] = t[0] + a;
        t[1] = m0 + b;
        t[2] = m0 - b;
    } else if (p == 5) {
        const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
        const double s1 = 0.95105651629515357212 * s, s2 = 0.58778525229247312917 * s;
        const cd a1 = t[1] + t[4], b1 = t[1] - t[4], a2 = t[2] + t[3], b2 = t[2] - t[3];
        const cd r1 = t[0] + c1 * a1 + c2 * a2, r2 = t[0] + c2 * a1 + c1 * a2;
        const cd i1 = (s1 * b1 + s2 * b2) * cd(0, 1), i2 = (s2 * b1 - s1 * b2) * cd(0, 1);
        t[0] = t[0] + a1 + a2;
        t[1] = r1 + i1;
        t[4] = r1 - i1;
        t[2] = r2 + i2;
        t[3] = r2 - i2;
    } else {  // odd p: symmetric pairs
        const int h = (p - 1) / 2;
        const std::vector<double>& co = c.pc[c.pidx[p]];
        const std::vector<double>& si = c.ps[c.pidx[p]];
        cd* a = tmp;
        cd* b = tmp + h;
        cd y0 = t[0];
        for (int k = 1; k <= h; ++k) {
            a[k - 1] = t[k] + t[p - k];
            b[k - 1] = t[k] - t[p - k];
            y0 += a[k - 1];
        }
        cd* y = tmp + 2 * h;
        for (int q = 1; q <= h; ++q) {
            double rr = t[0].real(), ri = t[0].imag(), ir = 0.0, ii = 0.0;
            int idx = 0;
            for (int k = 0; k < h; ++k) {
                idx += q;
                if (idx >= p) idx -= p;
                const double cw = co[idx], sw = si[idx];
                rr += a[k].real() * cw;
                ri += a[k].imag() * cw;
                ir += b[k].real() * sw;
                ii += b[k].imag() * sw;
            }
            // sum_k b_k * (i s sin) = i s (ir + i ii)
            const cd im = cd(-s * ii, s * ir);
            y[q] = cd(rr, ri) + im;
            y[p - q] = cd(rr, ri) - im;
        }
        t[0] = y0;
        for (int q = 1; q < p; ++q) t[q] = y[q];
    }
}

// out[0..n) = DFT_n of in[0], in[stride], ...; this level's twiddle base is
// exp(-2 pi i / n) = c.tw[tw_step]
inline void fft_rec(const cd* in, long stride, cd* out, int n, const CPlan& c, int tw_step, int fi, bool inv,
                    cd* tmp) {
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    const int p = c.factors[fi];
    const int m = n / p;
    for (int r = 0; r < p; ++r) fft_rec(in + r * stride, stride * p, out + static_cast<long>(r) * m, m, c, tw_step * p, fi + 1, inv, tmp);
    cd* t = tmp;
    cd* scratch = tmp + p;
    for (int k = 0; k < m; ++k) {
        t[0] = out[k];
        for (int r = 1; r < p; ++r) {
            cd w = c.tw[static_cast<long>(r) * k * tw_step];
            if (inv) w = std::conj(w);
            t[r] = w * out[k + r * m];
        }
        small_dft(t, p, inv, c, scratch);
        for (int q = 0; q < p; ++q) out[k + q * m] = t[q];
    }
}

inline std::vector<cd>& scratch(int which, size_t n) {
    thread_local std::vector<cd> s[3];
    if (s[which].size() < n) s[which].resize(n);
    return s[which];
}

inline void cfft(const CPlan& c, const cd* in, cd* out, bool inv) {
    auto& tmp = scratch(2, 4 * static_cast<size_t>(c.m) + 16);
    fft_rec(in, 1, out, c.m, c, 1, 0, inv, tmp.data());
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
        auto& a = oracle_fftw::scratch(0, n);
        auto& b = oracle_fftw::scratch(1, n);
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
    auto& a = oracle_fftw::scratch(0, h);
    auto& Z = oracle_fftw::scratch(1, h);
    for (int j = 0; j < h; ++j) a[j] = cd(in[2 * j], in[2 * j + 1]);
    oracle_fftw::cfft(p->c, a.data(), Z.data(), false);
    // X_k = (Z_k + conj Z_{h-k})/2 - i w^k (Z_k - conj Z_{h-k})/2
    for (int k = 0; k <= h; ++k) {
        const cd zk = Z[k % h], zc = std::conj(Z[(h - k) % h]);
        const cd e = 0.5 * (zk + zc), o = 0.5 * (zk - zc);
        const cd x = e + cd(0, -1) * p->w[k] * o;
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
        auto& a = oracle_fftw::scratch(0, n);
        auto& b = oracle_fftw::scratch(1, n);
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
    auto& a = oracle_fftw::scratch(0, h);
    auto& z = oracle_fftw::scratch(1, h);
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
        a[k] = e + cd(0, 1) * std::conj(p->w[k]) * o;
    }
    oracle_fftw::cfft(p->c, a.data(), z.data(), true);
    for (int j = 0; j < h; ++j) {
        out[2 * j] = z[j].real();
        out[2 * j + 1] = z[j].imag();
    }
}

#endif
