// The reference-side binding of the OPERATOR SEAM, compiled: a replacement
// for the reference's src/fc_core.cpp (fcs::fc, include/fcs/fc_core.hpp:33-110)
// whose FcOperator / OperatorCache / fc_derivative / apply_filter /
// smear_initial_data / build_fc_operator run on the B200 through the fcsg C
// ABI (include/fcsg.h) instead of FFTW + MPFR. It is what a maintainer would
// add to the reference's fcsolver library; here it
// is built by oracle/Makefile (target `dropin`) against the reference's own
// headers and linked with the reference's OTHER sources unmodified, and the
// reference's own tests/test_fc_core.cpp runs against it on the GPU box
// (`make -C oracle check-dropin`). TEST INFRASTRUCTURE: the product is
// libfcsg.so; nothing in the package uses this file.
//
// Mapping:
//   FcOperator(n, n_cont, filter)          -> fcsg_operator (tables built by
//                                              fcsg's binary128 QR; sizes and
//                                              profiles from fcsg_operator_info)
//   derivative / filter / strong_filter    -> fcsg_fc_lines_host (modes 1-2 / 3 / 4)
//   continuation                           -> the blend matrix applied on the host
//                                              (24 x 3 + 24 x 3 multiply-adds)
//   spectrum / evaluate (validation paths) -> the extension's DFT on the host,
//                                              summed in long double
// Errors: fcsg's kinds are rethrown as the reference's ConfigError /
// UsageError (include/fcs/errors.hpp). A process-wide fcsg context on device
// FCSG_DEVICE (default 0) serves every operator; calls are serialised by a
// mutex, since the reference promises thread-safe const methods
// (include/fcs/fc_core.hpp:27-29) and an fcsg context is used from one thread
// at a time.
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "fcs/errors.hpp"
#include "fcs/fc_core.hpp"
#include "fcsg.h"

namespace fcs::fc {

namespace {

std::mutex& gpu_mutex() {
    static std::mutex m;
    return m;
}

void raise(fcsg_ctx* c, int rc) {
    if (rc == FCSG_OK) return;
    char msg[512] = {0};
    int kind = rc;
    if (c) fcsg_last_error(c, msg, sizeof msg, &kind, nullptr, nullptr, nullptr, nullptr, nullptr);
    const std::string m = msg[0] ? msg : ("fcsg error " + std::to_string(rc));
    if (kind == FCSG_CONFIG) throw ConfigError(m);
    if (kind == FCSG_USAGE) throw UsageError(m);
    throw std::runtime_error(m);
}

fcsg_ctx* context() {
    static fcsg_ctx* ctx = [] {
        const char* d = std::getenv("FCSG_DEVICE");
        fcsg_ctx* c = nullptr;
        const int rc = fcsg_create(d ? std::atoi(d) : 0, &c);
        if (rc != FCSG_OK) throw std::runtime_error("fcsg_create failed (no CUDA device?)");
        return c;
    }();
    return ctx;
}

// the extended line [f; gap] of an operator (n_ext values)
std::vector<double> extension(const FcOperator& op, const double* in, int stride) {
    std::vector<double> ext(op.n_ext());
    for (int i = 0; i < op.n_points(); ++i) ext[i] = in[static_cast<long>(i) * stride];
    op.continuation(ext.data(), ext.data() + op.n_points());
    return ext;
}

// unnormalised forward DFT bins 0..n_ext/2 of a real sequence (FFTW's r2c
// convention), summed in long double over a cached root table per length
std::vector<std::pair<long double, long double>> dft_half(const std::vector<double>& x) {
    static std::mutex m;
    static std::map<int, std::vector<std::pair<long double, long double>>> roots;
    const int n = static_cast<int>(x.size());
    const std::vector<std::pair<long double, long double>>* r;
    {
        std::lock_guard<std::mutex> lock(m);
        auto& t = roots[n];
        if (t.empty()) {
            const long double w = 2.0L * 3.14159265358979323846264338327950288L / n;
            t.resize(n);
            for (int j = 0; j < n; ++j) t[j] = {std::cos(w * j), std::sin(w * j)};
        }
        r = &t;
    }
    std::vector<std::pair<long double, long double>> out(n / 2 + 1);
    for (int k = 0; k <= n / 2; ++k) {
        long double re = 0.0L, im = 0.0L;
        for (int j = 0, kj = 0; j < n; ++j, kj = (kj + k) % n) {
            re += x[j] * (*r)[kj].first;
            im -= x[j] * (*r)[kj].second;
        }
        out[k] = {re, im};
    }
    return out;
}

}  // namespace

struct FcOperator::Impl {
    int op_id = -1;
};

FcOperator::FcOperator(int n_points, int n_cont, FilterSpec filter) : n_(n_points), n_cont_(n_cont) {
    // the reference's argument checks come first (ConfigError, src/fc_core.cpp:192-193)
    if (n_points < 10) throw ConfigError("FcOperator: n_points must be >= 10");
    if (n_cont < 4) throw ConfigError("FcOperator: n_cont must be >= 4");
    impl_ = std::make_unique<Impl>();
    blend_ = &blend_matrix(n_cont_);  // takes the GPU lock itself (not held here: std::mutex is not recursive)
    std::lock_guard<std::mutex> lock(gpu_mutex());
    fcsg_ctx* c = context();
    raise(c, fcsg_operator(c, n_points, n_cont, degree, filter.alpha, filter.p, filter.p_smear, &impl_->op_id));
    raise(c, fcsg_operator_info(c, impl_->op_id, &n_ext_, &n_modes_, &period_, nullptr, nullptr, nullptr));
    filter_profile_.resize(n_modes_);
    smear_profile_.resize(n_modes_);
    raise(c, fcsg_operator_info(c, impl_->op_id, nullptr, nullptr, nullptr, nullptr, filter_profile_.data(),
                                smear_profile_.data()));
}

FcOperator::~FcOperator() = default;

const std::vector<double>& FcOperator::blend_matrix(int n_cont) {
    static std::mutex m;
    static std::map<int, std::vector<double>> cache;
    std::lock_guard<std::mutex> lock(m);
    auto it = cache.find(n_cont);
    if (it != cache.end()) return it->second;
    if (n_cont < 4) throw ConfigError("FcOperator: n_cont must be >= 4");
    std::vector<double> A(static_cast<size_t>(n_cont - 1) * (degree + 1));
    {
        std::lock_guard<std::mutex> g(gpu_mutex());
        fcsg_ctx* c = context();
        int op = -1;
        // the blend matrix depends on (degree, n_cont) only; any line length builds it
        raise(c, fcsg_operator(c, 64, n_cont, degree, FilterSpec{}.alpha, FilterSpec{}.p, FilterSpec{}.p_smear, &op));
        raise(c, fcsg_operator_info(c, op, nullptr, nullptr, nullptr, A.data(), nullptr, nullptr));
    }
    return cache.emplace(n_cont, std::move(A)).first->second;
}

// gap_j = sum_i A[j][i] f[N-1-d+i] + sum_i A[g-1-j][i] f[d-i] (the right blend
// plus the reflected left blend, g = n_cont - 1)
void FcOperator::continuation(const double* in, double* gap_out) const {
    const int d1 = degree + 1, g = n_cont_ - 1;
    const std::vector<double>& A = *blend_;
    for (int j = 0; j < g; ++j) {
        double r = 0.0, l = 0.0;
        for (int i = 0; i < d1; ++i) {
            r += A[static_cast<size_t>(j) * d1 + i] * in[n_ - d1 + i];
            l += A[static_cast<size_t>(g - 1 - j) * d1 + i] * in[degree - i];
        }
        gap_out[j] = r + l;
    }
}

void FcOperator::derivative(const double* in, int in_stride, double* out, int out_stride, int order) const {
    if (order != 1 && order != 2) throw UsageError("derivative: order must be 1 or 2");
    std::lock_guard<std::mutex> lock(gpu_mutex());
    fcsg_ctx* c = context();
    raise(c, fcsg_fc_lines_host(c, impl_->op_id, order, in, 0, in_stride, out, 0, out_stride, 1, 1.0));
}

void FcOperator::apply_profile(const double* in, int in_stride, double* out, int out_stride,
                               const std::vector<double>& profile) const {
    const int mode = (&profile == &smear_profile_) ? FCSG_SMEAR : FCSG_FILTER;
    std::lock_guard<std::mutex> lock(gpu_mutex());
    fcsg_ctx* c = context();
    raise(c, fcsg_fc_lines_host(c, impl_->op_id, mode, in, 0, in_stride, out, 0, out_stride, 1, 1.0));
}

void FcOperator::filter(const double* in, int in_stride, double* out, int out_stride) const {
    apply_profile(in, in_stride, out, out_stride, filter_profile_);
}

void FcOperator::strong_filter(const double* in, int in_stride, double* out, int out_stride) const {
    apply_profile(in, in_stride, out, out_stride, smear_profile_);
}

void FcOperator::spectrum(const double* in, int in_stride, std::vector<double>& mag) const {
    const auto bins = dft_half(extension(*this, in, in_stride));
    mag.resize(bins.size());
    for (size_t k = 0; k < bins.size(); ++k)
        mag[k] = static_cast<double>(std::hypot(bins[k].first, bins[k].second) / n_ext_);
}

// the trigonometric interpolant of the extension at x (unit-span
// coordinates, period = period()): c_0 + sum_k w_k Re(c_k e^{2 pi i k x / period}),
// w_k = 2 except the even-n_ext Nyquist bin (1)
double FcOperator::evaluate(const std::vector<double>& in, double x) const {
    if (static_cast<int>(in.size()) != n_) throw UsageError("evaluate: length mismatch");
    const auto bins = dft_half(extension(*this, in.data(), 1));
    const int nb = static_cast<int>(bins.size());
    long double v = bins[0].first / n_ext_;
    const long double two_pi = 2.0L * 3.14159265358979323846264338327950288L;
    for (int k = 1; k < nb; ++k) {
        const long double wk = (n_ext_ % 2 == 0 && k == nb - 1) ? 1.0L : 2.0L;
        const long double a = two_pi * k * x / period_;
        v += wk / n_ext_ * (bins[k].first * std::cos(a) - bins[k].second * std::sin(a));
    }
    return static_cast<double>(v);
}

GridLine smear_initial_data(const FcOperator& op, const GridLine& line, const std::vector<double>& mask) {
    if (mask.size() != line.values.size()) throw UsageError("smear_initial_data: mask length mismatch");
    GridLine out = line;
    bool blend = false;
    for (double m : mask) blend = blend || m != 0.0;
    if (!blend) return out;  // all-zero mask: the line unchanged, bit for bit
    std::vector<double> s(line.values.size());
    op.strong_filter(line.values.data(), 1, s.data(), 1);
    for (size_t i = 0; i < s.size(); ++i) out.values[i] = mask[i] * s[i] + (1.0 - mask[i]) * line.values[i];
    return out;
}

GridLine fc_derivative(const FcOperator& op, const GridLine& line, int order) {
    if (static_cast<int>(line.values.size()) != op.n_points()) throw UsageError("fc_derivative: length mismatch");
    if (order != 1 && order != 2) throw UsageError("derivative: order must be 1 or 2");
    GridLine out = line;
    op.derivative(line.values.data(), 1, out.values.data(), 1, order);
    // unit-span derivative -> physical spacing: (1 / ((N-1) h))^order
    const double s = std::pow(1.0 / (line.h * (op.n_points() - 1)), order);
    for (double& v : out.values) v *= s;
    return out;
}

GridLine apply_filter(const FcOperator& op, const GridLine& line) {
    if (static_cast<int>(line.values.size()) != op.n_points()) throw UsageError("apply_filter: length mismatch");
    GridLine out = line;
    op.filter(line.values.data(), 1, out.values.data(), 1);
    return out;
}

struct OperatorCache::Impl {
    std::mutex mu;
    std::map<std::tuple<int, int, double, int, int>, std::shared_ptr<const FcOperator>> ops;
};

OperatorCache& OperatorCache::instance() {
    static OperatorCache c;
    return c;
}

std::shared_ptr<const FcOperator> OperatorCache::get(int n_points, int n_cont, FilterSpec filter) {
    static Impl impl;
    std::lock_guard<std::mutex> lock(impl.mu);
    const auto key = std::make_tuple(n_points, n_cont, filter.alpha, filter.p, filter.p_smear);
    auto& slot = impl.ops[key];
    if (!slot) slot = std::make_shared<FcOperator>(n_points, n_cont, filter);
    return slot;
}

std::shared_ptr<const FcOperator> OperatorCache::get(int n_points) { return get(n_points, 25, FilterSpec{}); }

std::shared_ptr<const FcOperator> build_fc_operator(int n_points, int n_cont, int filter_order, double filter_alpha) {
    if (filter_order % 2 != 0) throw ConfigError("filter_order must be even (2p)");
    FilterSpec f;
    f.alpha = filter_alpha;
    f.p = filter_order / 2;
    return OperatorCache::instance().get(n_points, n_cont, f);
}

}  // namespace fcs::fc
