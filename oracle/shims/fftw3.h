/*
 * TEST INFRASTRUCTURE ONLY (oracle build shim) -- never linked into the product.
 *
 * Minimal stand-in for the five FFTW3 entry points the reference's
 * src/fc_core.cpp uses (fc_core.cpp:3,185-186,211-216,263,282,291,295,312,327):
 *   fftw_plan_dft_r2c_1d / fftw_plan_dft_c2r_1d (FFTW_ESTIMATE|FFTW_UNALIGNED),
 *   fftw_execute_dft_r2c / fftw_execute_dft_c2r (new-array execute),
 *   fftw_destroy_plan.
 * FFTW is absent from this image and the reference pins no version, so this
 * header restates FFTW's published transform definitions:
 *   r2c: Y[k] = sum_j x[j] exp(-2 pi i j k / n), k = 0..n/2 (unnormalised)
 *   c2r: y[j] = sum_{k=0}^{n-1} Y[k] exp(+2 pi i j k / n) over the Hermitian
 *        extension of the n/2+1 input bins; the imaginary parts of the DC and
 *        (even n) Nyquist bins are ignored, as FFTW does (unnormalised).
 * Implementation: recursive mixed-radix decimation-in-time over the prime
 * factors of n, twiddles evaluated in long double. Plans are immutable;
 * execute uses thread_local scratch, so concurrent execution of one plan
 * from several threads is safe (the reference relies on that, fc_core.cpp:174).
 */
#ifndef ORACLE_SHIM_FFTW3_H
#define ORACLE_SHIM_FFTW3_H

#include <cmath>
#include <complex>
#include <vector>

typedef double fftw_complex[2];

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

struct oracle_fftw_plan_s {
    int n = 0;
    bool r2c = true;
    std::vector<std::complex<double>> tw;  // exp(-2 pi i k / n), k = 0..n-1
    std::vector<int> factors;              // prime factors, ascending
};
typedef oracle_fftw_plan_s* fftw_plan;

namespace oracle_fftw {

inline void fft_rec(const std::complex<double>* in, int stride, std::complex<double>* out, int n,
                    const oracle_fftw_plan_s& pl, int tw_step, int fidx, bool inverse,
                    std::complex<double>* tmp) {
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    const int p = pl.factors[fidx];
    const int m = n / p;
    for (int r = 0; r < p; ++r)
        fft_rec(in + static_cast<long>(r) * stride, stride * p, out + static_cast<long>(r) * m, m,
                pl, tw_step * p, fidx + 1, inverse, tmp);
    // combine: X[k + q m] = sum_r w_n^{r (k + q m)} S_r[k]
    const int N = pl.n;
    for (int k = 0; k < m; ++k) {
        for (int r = 0; r < p; ++r) tmp[r] = out[k + r * m];
        for (int q = 0; q < p; ++q) {
            std::complex<double> acc = 0.0;
            const long kk = k + static_cast<long>(q) * m;
            for (int r = 0; r < p; ++r) {
                const long e = (static_cast<long>(r) * kk * tw_step) % N;
                std::complex<double> w = pl.tw[e];
                if (inverse) w = std::conj(w);
                acc += w * tmp[r];
            }
            out[kk] = acc;
        }
    }
}

inline std::vector<std::complex<double>>& scratch_a(int n) {
    thread_local std::vector<std::complex<double>> s;
    if (static_cast<int>(s.size()) < n) s.resize(n);
    return s;
}
inline std::vector<std::complex<double>>& scratch_b(int n) {
    thread_local std::vector<std::complex<double>> s;
    if (static_cast<int>(s.size()) < n) s.resize(n);
    return s;
}
inline std::vector<std::complex<double>>& scratch_t(int n) {
    thread_local std::vector<std::complex<double>> s;
    if (static_cast<int>(s.size()) < n) s.resize(n);
    return s;
}

inline fftw_plan make_plan(int n, bool r2c) {
    auto* p = new oracle_fftw_plan_s;
    p->n = n;
    p->r2c = r2c;
    p->tw.resize(n);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int k = 0; k < n; ++k) {
        const long double a = two_pi * k / n;
        p->tw[k] = std::complex<double>(static_cast<double>(cosl(a)), static_cast<double>(-sinl(a)));
    }
    int m = n;
    for (int f = 2; f * f <= m; ++f)
        while (m % f == 0) {
            p->factors.push_back(f);
            m /= f;
        }
    if (m > 1) p->factors.push_back(m);
    return p;
}

}  // namespace oracle_fftw

inline fftw_plan fftw_plan_dft_r2c_1d(int n, double*, fftw_complex*, unsigned) {
    return oracle_fftw::make_plan(n, true);
}
inline fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex*, double*, unsigned) {
    return oracle_fftw::make_plan(n, false);
}
inline void fftw_destroy_plan(fftw_plan p) { delete p; }

inline void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
    const int n = p->n;
    auto& a = oracle_fftw::scratch_a(n);
    auto& b = oracle_fftw::scratch_b(n);
    auto& t = oracle_fftw::scratch_t(n);
    for (int j = 0; j < n; ++j) a[j] = std::complex<double>(in[j], 0.0);
    oracle_fftw::fft_rec(a.data(), 1, b.data(), n, *p, 1, 0, false, t.data());
    for (int k = 0; k <= n / 2; ++k) {
        out[k][0] = b[k].real();
        out[k][1] = b[k].imag();
    }
    out[0][1] = 0.0;
    if (n % 2 == 0) out[n / 2][1] = 0.0;
}

inline void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
    const int n = p->n;
    auto& a = oracle_fftw::scratch_a(n);
    auto& b = oracle_fftw::scratch_b(n);
    auto& t = oracle_fftw::scratch_t(n);
    a[0] = std::complex<double>(in[0][0], 0.0);
    for (int k = 1; k <= n / 2; ++k) {
        a[k] = std::complex<double>(in[k][0], in[k][1]);
        a[n - k] = std::conj(a[k]);
    }
    if (n % 2 == 0) a[n / 2] = std::complex<double>(in[n / 2][0], 0.0);
    oracle_fftw::fft_rec(a.data(), 1, b.data(), n, *p, 1, 0, true, t.data());
    for (int j = 0; j < n; ++j) out[j] = b[j].real();
}

#endif
