// FC operator tables, built once per (N, n_cont, degree, filter) on the host.
//
// Blend matrix: the reference (src/fc_core.cpp:55-152) fits, for each
// orthonormal Gram polynomial on the d+1 boundary points, a 31-term
// trigonometric series of period 2(d+n_cont+3) that matches the polynomial on
// [0,d] and zero on [d+n_cont, d+n_cont+2] (10x oversampled), by normal
// equations at 120 decimal digits, and samples it on the n_cont-1 gap points.
// Here the same least-squares problem is solved by Householder QR in IEEE
// binary128 (__float128): QR works on B itself (condition ~1e10 instead of
// the normal equations' ~1e20), so 113-bit arithmetic leaves ~1e-24 error in
// the fitted values, far below the double rounding of the table. The Gram
// basis is computed in double exactly as the reference does (fc_core.cpp:88-112),
// generalised from d=2 to any degree; the 1e-13 residual guard is kept.
#include "fc_tables.h"

#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <functional>

namespace fcsg {

namespace {

constexpr int kOversample = 10;  // src/fc_core.cpp:27-29
constexpr int kZeroWidth = 3;
constexpr int kModes = 15;

using q128 = __float128;

void gram_basis(int d, std::vector<std::vector<double>>& pv, std::vector<std::vector<double>>& coef) {
    const int n = d + 1;
    std::vector<std::vector<double>> q(n, std::vector<double>(n)), cf(n, std::vector<double>(n, 0.0));
    for (int m = 0; m < n; ++m) {
        for (int i = 0; i < n; ++i) q[m][i] = std::pow(static_cast<double>(i), m);
        cf[m][m] = 1.0;
    }
    for (int k = 0; k < n; ++k) {
        for (int p = 0; p < k; ++p) {
            double dot = 0;
            for (int i = 0; i < n; ++i) dot += q[p][i] * q[k][i];
            for (int i = 0; i < n; ++i) q[k][i] -= dot * q[p][i];
            for (int m = 0; m < n; ++m) cf[k][m] -= dot * cf[p][m];
        }
        double nrm = 0;
        for (int i = 0; i < n; ++i) nrm += q[k][i] * q[k][i];
        nrm = std::sqrt(nrm);
        for (int i = 0; i < n; ++i) q[k][i] /= nrm;
        for (int m = 0; m < n; ++m) cf[k][m] /= nrm;
    }
    pv = q;
    coef = cf;
}

// least squares min |B x - Y| for several right-hand sides (columns of Y),
// Householder QR; B is rows x cols row-major, Y is rows x nrhs. Returns x
// (cols x nrhs).
std::vector<q128> lsq_householder(std::vector<q128> B, std::vector<q128> Y, int rows, int cols,
                                  int nrhs) {
    for (int k = 0; k < cols; ++k) {
        q128 nrm = 0;
        for (int i = k; i < rows; ++i) nrm += B[i * cols + k] * B[i * cols + k];
        nrm = sqrtq(nrm);
        if (nrm == 0) throw Error(kConfig, "blend matrix solve: singular system");
        const q128 alpha = B[k * cols + k] > 0 ? -nrm : nrm;
        std::vector<q128> v(rows - k);
        for (int i = k; i < rows; ++i) v[i - k] = B[i * cols + k];
        v[0] -= alpha;
        q128 vn = 0;
        for (auto x : v) vn += x * x;
        for (int j = k; j < cols; ++j) {
            q128 s = 0;
            for (int i = k; i < rows; ++i) s += v[i - k] * B[i * cols + j];
            s = 2 * s / vn;
            for (int i = k; i < rows; ++i) B[i * cols + j] -= s * v[i - k];
        }
        for (int j = 0; j < nrhs; ++j) {
            q128 s = 0;
            for (int i = k; i < rows; ++i) s += v[i - k] * Y[i * nrhs + j];
            s = 2 * s / vn;
            for (int i = k; i < rows; ++i) Y[i * nrhs + j] -= s * v[i - k];
        }
    }
    std::vector<q128> x(static_cast<size_t>(cols) * nrhs);
    for (int j = 0; j < nrhs; ++j)
        for (int k = cols - 1; k >= 0; --k) {
            q128 s = Y[k * nrhs + j];
            for (int c = k + 1; c < cols; ++c) s -= B[k * cols + c] * x[c * nrhs + j];
            x[k * nrhs + j] = s / B[k * cols + k];
        }
    return x;
}

}  // namespace

std::vector<double> build_blend_matrix(int n_cont, int d) {
    if (d < 1 || d + 1 > kMaxDeg + 1) throw Error(kConfig, "blend matrix: unsupported degree");
    if (n_cont - 1 > kMaxGap) throw Error(kConfig, "blend matrix: n_cont too large");
    const q128 lam = q128(2) * (d + n_cont + kZeroWidth);
    const q128 twopi = 2 * acosq(q128(-1));
    const int n_match = kOversample * d + 1;
    const int n_zero = kOversample * (kZeroWidth - 1) + 1;
    const int rows = n_match + n_zero;
    const int cols = 2 * kModes + 1;
    std::vector<q128> zs(rows);
    for (int i = 0; i < n_match; ++i) zs[i] = q128(d) * i / (n_match - 1);
    for (int i = 0; i < n_zero; ++i) zs[n_match + i] = q128(d + n_cont) + q128(kZeroWidth - 1) * i / (n_zero - 1);
    std::vector<q128> B(static_cast<size_t>(rows) * cols);
    for (int r = 0; r < rows; ++r) {
        B[r * cols] = 1;
        for (int m = 1; m <= kModes; ++m) {
            const q128 arg = twopi * m * zs[r] / lam;
            B[r * cols + 2 * m - 1] = cosq(arg);
            B[r * cols + 2 * m] = sinq(arg);
        }
    }
    std::vector<std::vector<double>> pv, coef;
    gram_basis(d, pv, coef);
    const int nrhs = d + 1;
    std::vector<q128> Y(static_cast<size_t>(rows) * nrhs, 0);
    for (int k = 0; k <= d; ++k)
        for (int r = 0; r < n_match; ++r) {
            q128 v = 0, zp = 1;
            for (int m = 0; m <= d; ++m) {
                v += q128(coef[k][m]) * zp;
                zp *= zs[r];
            }
            Y[r * nrhs + k] = v;
        }
    const auto X = lsq_householder(B, Y, rows, cols, nrhs);
    // residual guard (src/fc_core.cpp:130-138)
    for (int k = 0; k <= d; ++k) {
        q128 resid = 0;
        for (int r = 0; r < rows; ++r) {
            q128 v = 0;
            for (int i = 0; i < cols; ++i) v += B[r * cols + i] * X[i * nrhs + k];
            resid = std::max(resid, fabsq(v - Y[r * nrhs + k]));
        }
        if (resid > q128(1e-13)) throw Error(kConfig, "blend matrix fit residual too large");
    }
    const int n_gap = n_cont - 1;
    std::vector<double> A(static_cast<size_t>(n_gap) * (d + 1), 0.0);
    for (int k = 0; k <= d; ++k)
        for (int j = 0; j < n_gap; ++j) {
            const q128 z = q128(d + 1 + j);
            q128 val = X[0 * nrhs + k];
            for (int m = 1; m <= kModes; ++m) {
                const q128 arg = twopi * m * z / lam;
                val += X[(2 * m - 1) * nrhs + k] * cosq(arg) + X[(2 * m) * nrhs + k] * sinq(arg);
            }
            for (int i = 0; i <= d; ++i) A[static_cast<size_t>(j) * (d + 1) + i] += static_cast<double>(val) * pv[k][i];
        }
    return A;
}



FcTables build_fc_tables(int n_points, int n_cont, int degree, FilterSpec f) {
    // FcOperator ctor checks (src/fc_core.cpp:192-193)
    if (n_points < 10) throw Error(kConfig, "FcOperator: n_points must be >= 10");
    if (n_cont < 4) throw Error(kConfig, "FcOperator: n_cont must be >= 4");
    if (n_points < 2 * (degree + 1)) throw Error(kConfig, "FcOperator: line too short for the degree");
    FcTables t;
    t.n = n_points;
    t.n_cont = n_cont;
    t.degree = degree;
    t.filter = f;
    t.n_ext = n_points + n_cont - 1;
    t.period = static_cast<double>(t.n_ext) / (n_points - 1);
    t.n_modes = t.n_ext / 2 + 1;
    t.blend = build_blend_matrix(n_cont, degree);
    const int n = t.n_ext;
    const int kmax = n / 2;
    t.filter_profile.resize(t.n_modes);
    t.smear_profile.resize(t.n_modes);
    for (int k = 0; k < t.n_modes; ++k) {  // src/fc_core.cpp:199-206
        const double r = kmax > 0 ? static_cast<double>(k) / kmax : 0.0;
        t.filter_profile[k] = std::exp(-f.alpha * std::pow(r, 2.0 * f.p));
        t.smear_profile[k] = std::exp(-f.alpha * std::pow(r, 2.0 * f.p_smear));
    }
    // FFT plan: DIF stages, span L_0 = n, L_{s+1} = L_s / p_s
    const Factors fs = factor_stages(n);
    for (int s = 0; s < fs.n; ++s) {
        t.radix.push_back(fs.r[s]);
        t.span.push_back(fs.span[s]);
    }
    t.tw.resize(n);
    for (int k = 0; k < n; ++k) {
        const q128 a = 2 * acosq(q128(-1)) * k / n;
        t.tw[k].x = static_cast<double>(cosq(a));
        t.tw[k].y = static_cast<double>(-sinq(a));
    }
    // digit reversal of the in-place DIF: position pos = q0*m0 + rest holds
    // frequency q0 + p0 * (frequency of rest in the length-m0 sub-transform)
    t.freq_of_pos.resize(n);
    std::function<int(int, int)> freq = [&](int pos, int s) -> int {
        if (s == static_cast<int>(t.radix.size())) return 0;
        const int p = t.radix[s];
        const int m = t.span[s] / p;
        const int q0 = pos / m;
        return q0 + p * freq(pos % m, s + 1);
    };
    for (int pos = 0; pos < n; ++pos) t.freq_of_pos[pos] = freq(pos, 0);
    // spectral multipliers, same double expressions as src/fc_core.cpp:265-281,294
    t.mult.assign(4 * static_cast<size_t>(n), double2{0.0, 0.0});
    const double beta = t.period;
    const double w0 = 2.0 * M_PI / beta;
    const double inv_n = 1.0 / n;
    for (int pos = 0; pos < n; ++pos) {
        const int k = t.freq_of_pos[pos];
        const int kk = (k <= n / 2) ? k : n - k;  // |signed frequency|
        const double sgn = (k <= n / 2) ? 1.0 : -1.0;
        // d1: i * w0 * k * inv_n, conjugate-symmetric; even-n Nyquist zeroed
        double2 m1{0.0, 0.0};
        if (!(n % 2 == 0 && kk == n / 2)) m1.y = sgn * (w0 * kk * inv_n);
        t.mult[0 * n + pos] = m1;
        const double w = w0 * kk;
        t.mult[1 * n + pos] = double2{-w * w * inv_n, 0.0};
        t.mult[2 * n + pos] = double2{t.filter_profile[kk] * inv_n, 0.0};
        t.mult[3 * n + pos] = double2{t.smear_profile[kk] * inv_n, 0.0};
    }
    // the prime-factor order of the warp transform (wline.h): entry
    // (k1 * 5 + k2) * 7 + k3 holds frequency (105 k1 + 56 k2 + 120 k3) mod 280
    if (n == 280) {
        std::vector<int> pos_of_freq(n);
        for (int pos = 0; pos < n; ++pos) pos_of_freq[t.freq_of_pos[pos]] = pos;
        t.mult_pfa.assign(4 * static_cast<size_t>(n), double2{0.0, 0.0});
        for (int k1 = 0; k1 < 8; ++k1)
            for (int k2 = 0; k2 < 5; ++k2)
                for (int k3 = 0; k3 < 7; ++k3) {
                    const int idx = (k1 * 5 + k2) * 7 + k3;
                    const int pos = pos_of_freq[(105 * k1 + 56 * k2 + 120 * k3) % n];
                    for (int m = 0; m < 4; ++m) t.mult_pfa[m * n + idx] = t.mult[m * n + pos];
                }
    }
    // operand fragments of the tensor-core prime DFT (fft_line.h
    // middle_dmma_ct): lane (g, t) = (lane / 4, lane % 4) of m-tile mt and
    // k-step ks holds (cos, sin)(2 pi q r / P), q = 8 mt + g, r = 1 + 4 ks + t,
    // zero outside q, r <= (P - 1) / 2 -- the values of the twiddle table, so
    // that the kernel neither reduces q r mod P nor gathers from it
    if (!t.radix.empty() && t.radix.back() >= 17) {
        const int P = t.radix.back(), H = (P - 1) / 2, pstep = n / P;
        const int MT = (H + 1 + 7) / 8, KS = (H + 3) / 4;
        t.prime_frag.assign(static_cast<size_t>(MT) * KS * 32, double2{0.0, 0.0});
        for (int mt = 0; mt < MT; ++mt)
            for (int ks = 0; ks < KS; ++ks)
                for (int lane = 0; lane < 32; ++lane) {
                    const int q = 8 * mt + (lane >> 2), r = 1 + 4 * ks + (lane & 3);
                    if (q > H || r > H) continue;
                    const double2 w = t.tw[static_cast<size_t>((q * r) % P) * pstep];  // (cos, -sin)
                    t.prime_frag[(static_cast<size_t>(mt) * KS + ks) * 32 + lane] = double2{w.x, -w.y};
                }
    }
    return t;
}

SpectrumTail build_spectrum_tail(int w, int n_cont) {
    if (w < kFbMinWindow || w > kFbMaxWindow) throw Error(kConfig, "fallback classifier: window out of range");
    constexpr int d = 2;  // FcOperator::degree
    const std::vector<double> A = build_blend_matrix(n_cont, d);
    const int g = n_cont - 1;
    SpectrumTail t;
    t.w = w;
    t.n_ext = w + g;
    t.nb = t.n_ext / 2 + 1;
    t.k_lo = (3 * (t.nb - 1)) / 4;  // src/viscosity.cpp:177
    t.nk = t.nb - t.k_lo;
    // ext = E x: x itself, then the gap (FcOperator::continuation,
    // src/fc_core.cpp:221-238): right blend of x[w-1-d .. w-1] plus the
    // reflected left blend of x[d .. 0]
    std::vector<q128> E(static_cast<size_t>(t.n_ext) * w, q128(0));
    for (int i = 0; i < w; ++i) E[static_cast<size_t>(i) * w + i] = 1;
    for (int j = 0; j < g; ++j) {
        q128* row = E.data() + static_cast<size_t>(w + j) * w;
        for (int i = 0; i <= d; ++i) row[w - 1 - d + i] += A[static_cast<size_t>(j) * (d + 1) + i];
        const int jr = g - 1 - j;
        for (int i = 0; i <= d; ++i) row[d - i] += A[static_cast<size_t>(jr) * (d + 1) + i];
    }
    const q128 twopi = 2 * acosq(q128(-1));
    const int nk2 = 2 * t.nk;
    t.table.assign(static_cast<size_t>(w) * nk2 + t.nk + 2, 0.0);
    for (int kk = 0; kk < t.nk; ++kk) {
        const int k = t.k_lo + kk;
        for (int i = 0; i < w; ++i) {
            q128 re = 0, im = 0;
            for (int j = 0; j < t.n_ext; ++j) {
                const q128 e = E[static_cast<size_t>(j) * w + i];
                if (e == 0) continue;
                const q128 a = twopi * ((static_cast<long>(j) * k) % t.n_ext) / t.n_ext;
                re += e * cosq(a);
                im -= e * sinq(a);
            }
            t.table[static_cast<size_t>(i) * nk2 + 2 * kk] = static_cast<double>(re);
            t.table[static_cast<size_t>(i) * nk2 + 2 * kk + 1] = static_cast<double>(im);
        }
    }
    double sx = 0.0, sxx = 0.0;
    double* lx = t.table.data() + static_cast<size_t>(w) * nk2;
    for (int kk = 0; kk < t.nk; ++kk) {
        lx[kk] = std::log(static_cast<double>(t.k_lo + kk));
        sx += lx[kk];
        sxx += lx[kk] * lx[kk];
    }
    lx[t.nk] = sx;
    lx[t.nk + 1] = sxx;
    return t;
}

}  // namespace fcsg
