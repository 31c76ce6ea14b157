/*
 * TEST INFRASTRUCTURE ONLY -- C-ABI exporter around the UNMODIFIED reference
 * (compiled from /root/reference/proj/src by oracle/Makefile into
 * oracle/_ref/libfcsref.so). Used by tests/ as the parity oracle, by
 * tests/golden/make_golden.py to write the committed fixtures, and by
 * bench.py --impl reference / cpu_baseline to time the reference's own CPU
 * step. Never linked into the product.
 *
 * Entry points mirror the reference API they call:
 *   ref_blend_matrix  -> fc::FcOperator::blend_matrix      (fc_core.cpp:156-163)
 *   ref_fc_*          -> fc::OperatorCache::get + FcOperator (fc_core.cpp:190-306,391-402)
 *   ref_engine_*      -> run::Engine init/step_phase/run    (runtime.cpp:293-530)
 *   ref_train_classifier -> visc::train_classifier + MlpClassifier::save
 *                                                           (viscosity.cpp:91-106,364-513)
 */
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <functional>
#include <limits>

#include "fcs/bc.hpp"
#include "fcs/errors.hpp"
#include "fcs/euler.hpp"
#include "fcs/fc_core.hpp"
#include "fcs/geometry.hpp"
#include "fcs/subpatch_data.hpp"
#include "fcs/viscosity.hpp"
// Engine::step_phase / dt_ / step_ are private; the phase-level parity hooks
// below need them (test-only access, the reference source is not modified).
// Every other header is included first so only class Engine is affected.
#define private public
#include "fcs/runtime.hpp"
#undef private

using namespace fcs;

namespace {
thread_local std::string g_err;
thread_local int g_err_kind = 0;

// error kinds shared with include/fcsg.h
enum { kOk = 0, kConfig = 1, kUsage = 2, kGeometry = 3, kDecomposition = 4, kInvalidState = 5, kOther = 9 };

template <class F>
int guard(F&& f) {
    try {
        f();
        return kOk;
    } catch (const InvalidStateError& e) {
        g_err = e.what();
        g_err += " at patch " + std::to_string(e.patch) + " subpatch " + std::to_string(e.subpatch) +
                 " (" + std::to_string(e.i) + "," + std::to_string(e.j) + ")";
        g_err_kind = kInvalidState;
    } catch (const ConfigError& e) {
        g_err = e.what();
        g_err_kind = kConfig;
    } catch (const UsageError& e) {
        g_err = e.what();
        g_err_kind = kUsage;
    } catch (const GeometryError& e) {
        g_err = e.what();
        g_err_kind = kGeometry;
    } catch (const DecompositionError& e) {
        g_err = e.what();
        g_err_kind = kDecomposition;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_err_kind = kOther;
    }
    return g_err_kind;
}

struct RefEngine {
    std::unique_ptr<run::Engine> eng;
};

BcKind bc_kind(int k) {
    switch (k) {
        case 0: return BcKind::inflow;
        case 1: return BcKind::outflow_pressure;
        case 2: return BcKind::slip_wall;
        case 3: return BcKind::noslip_adiabatic;
        case 4: return BcKind::supersonic_outflow;
        case 5: return BcKind::zero_normal_all;
    }
    throw UsageError("bad bc kind");
}

const Field* field_by_name(const SubpatchData& d, const std::string& w, int c) {
    if (w == "x") return &d.x;
    if (w == "y") return &d.y;
    if (w == "iq1x") return &d.iq1x;
    if (w == "iq2x") return &d.iq2x;
    if (w == "iq1y") return &d.iq1y;
    if (w == "iq2y") return &d.iq2y;
    if (w == "h_min") return &d.h_min;
    if (w == "h_max") return &d.h_max;
    if (w == "w_norm") return &d.w_norm;
    if (w == "mu_hat") return &d.mu_hat;
    if (w == "mu") return &d.mu;
    if (w == "tau") return &d.tau;
    if (w == "speed") return &d.speed;
    if (w == "e") return &d.e[c];
    if (w == "e0") return &d.e0[c];
    if (w == "e2") return &d.e2[c];
    if (w == "e3") return &d.e3[c];
    if (w == "rhs") return &d.rhs[c];
    if (w == "rhs3") return &d.rhs3[c];
    if (w == "theta") return &d.s6;
    if (w == "m01") return &d.s5;
    if (w == "tau_rho") return &d.s4;
    throw UsageError("unknown field " + w);
}

}  // namespace

extern "C" {

const char* ref_last_error(int* kind) {
    if (kind) *kind = g_err_kind;
    return g_err.c_str();
}

int ref_blend_matrix(int n_cont, double* out) {
    return guard([&] {
        const auto& A = fc::FcOperator::blend_matrix(n_cont);
        std::memcpy(out, A.data(), A.size() * sizeof(double));
    });
}

int ref_fc_info(int n, int n_cont, int* n_ext, double* period, double* filter_profile,
                double* smear_profile) {
    return guard([&] {
        auto op = fc::OperatorCache::instance().get(n, n_cont, fc::FilterSpec{});
        *n_ext = op->n_ext();
        *period = op->period();
        if (filter_profile)
            std::memcpy(filter_profile, op->filter_profile().data(),
                        op->filter_profile().size() * sizeof(double));
        if (smear_profile)
            std::memcpy(smear_profile, op->smear_profile().data(),
                        op->smear_profile().size() * sizeof(double));
    });
}

/* mode: 1/2 = derivative order (unit span), 3 = filter, 4 = strong filter,
 * 5 = continuation (writes n_cont-1 gap values per line into out).
 * Line l element i lives at in[l*line_stride + i*stride]. */
int ref_fc_apply(int n, int n_cont, int mode, const double* in, long line_stride, int stride,
                 int n_lines, double* out, int n_threads) {
    return guard([&] {
        auto op = fc::OperatorCache::instance().get(n, n_cont, fc::FilterSpec{});
        if (mode < 1 || mode > 5) throw UsageError("bad mode");
        auto work = [&](int l0, int l1) {
            std::vector<double> tmp(n);
            for (int l = l0; l < l1; ++l) {
                const double* src = in + static_cast<long>(l) * line_stride;
                double* dst = out + static_cast<long>(l) * line_stride;
                if (mode <= 2) op->derivative(src, stride, dst, stride, mode);
                else if (mode == 3) op->filter(src, stride, dst, stride);
                else if (mode == 4) op->strong_filter(src, stride, dst, stride);
                else {
                    for (int i = 0; i < n; ++i) tmp[i] = src[static_cast<long>(i) * stride];
                    op->continuation(tmp.data(), out + static_cast<long>(l) * (n_cont - 1));
                }
            }
        };
        if (n_threads <= 1) {
            work(0, n_lines);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < n_threads; ++t) {
                const int a = static_cast<int>(static_cast<long>(n_lines) * t / n_threads);
                const int b = static_cast<int>(static_cast<long>(n_lines) * (t + 1) / n_threads);
                th.emplace_back(work, a, b);
            }
            for (auto& t : th) t.join();
        }
    });
}

/* FcOperator::evaluate (fc_core.cpp:318-340), for the continuation KATs. */
int ref_fc_evaluate(int n, int n_cont, const double* in, int n_x, const double* xs, double* out) {
    return guard([&] {
        auto op = fc::OperatorCache::instance().get(n, n_cont, fc::FilterSpec{});
        std::vector<double> v(in, in + n);
        for (int k = 0; k < n_x; ++k) out[k] = op->evaluate(v, xs[k]);
    });
}

int ref_train_classifier(const char* path, double* holdout_accuracy) {
    return guard([&] {
        visc::MlpClassifier m;
        auto rep = visc::train_classifier(visc::TrainConfig{}, &m);
        m.save(path);
        if (holdout_accuracy) *holdout_accuracy = rep.holdout_accuracy;
    });
}

/* MlpClassifier::forward/classify_stencil on already-normalised stencils. */
int ref_mlp_forward(const char* path, int n, const double* x7, double* logits4, int* cls) {
    return guard([&] {
        auto m = visc::MlpClassifier::load(path);
        for (int k = 0; k < n; ++k) {
            m.forward(x7 + 7L * k, logits4 + 4L * k);
            cls[k] = m.classify_stencil(x7 + 7L * k);
        }
    });
}

/* Classifier::classify_line (ann variant) on raw lines. */
int ref_classify_line(const char* path, int n, const double* values, int* tau) {
    return guard([&] {
        visc::ClassifierConfig cc;
        cc.variant = visc::ClassifierConfig::Variant::ann;
        cc.weight_path = path;
        visc::Classifier c(cc);
        std::vector<uint8_t> t(n);
        c.classify_line(values, n, t.data());
        for (int i = 0; i < n; ++i) tau[i] = t[i];
    });
}

/* One rectangular I patch [x0,x0+lx]x[y0,y0+ly] split by subdivide_Q(r,s,n0,nv)
 * (geometry.cpp:213-255), sides W,E,S,N with BC kind codes (0 inflow,
 * 1 outflow_pressure, 2 slip_wall, 3 noslip_adiabatic, 4 supersonic_outflow,
 * 5 zero_normal_all; -1 = interior side). The engine is initialised with a
 * zero state; call ref_engine_set_state for every subpatch and then
 * ref_engine_finish_ic (== Engine::apply_ic with that state, runtime.cpp:276-287). */
void* ref_engine_affine(double x0, double y0, double e1x, double e1y, double e2x, double e2y, int r, int s, int n0,
                        int nv, const int* side_kinds, const double* side_states, const double* side_pressure,
                        double cfl, double T, int workers, const char* weight_path, long max_steps) {
    RefEngine* out = nullptr;
    guard([&] {
        geom::Patch p;
        p.kind = geom::PatchKind::I;
        p.map = std::make_shared<geom::AffineMap>(Vec2{x0, y0}, Vec2{e1x, e1y}, Vec2{e2x, e2y});
        BcTable bcs;
        const char* names[4] = {"w", "e", "s", "n"};
        for (int k = 0; k < 4; ++k) {
            if (side_kinds[k] < 0) {
                p.sides[k] = geom::SideInfo{false, ""};
            } else {
                p.sides[k] = geom::SideInfo{true, names[k]};
                BcSpec b;
                b.kind = bc_kind(side_kinds[k]);
                for (int c = 0; c < 4; ++c) b.state[c] = side_states[4 * k + c];
                b.pressure = side_pressure[k];
                bcs[names[k]] = b;
            }
        }
        p.index = 0;
        geom::subdivide_Q(p, r, s, n0, nv);
        geom::DomainDecomposition dec;
        dec.nv = nv;
        dec.n0 = n0;
        dec.patches.push_back(std::move(p));
        dec.assign_global_ids();
        run::EngineConfig cfg;
        cfg.cfl = cfl;
        cfg.T = T;
        cfg.workers = workers;
        cfg.max_steps = max_steps;
        if (weight_path && weight_path[0]) {
            cfg.classifier.variant = visc::ClassifierConfig::Variant::ann;
            cfg.classifier.weight_path = weight_path;
        }
        auto ic = [](double, double) { return std::array<double, 4>{0, 0, 0, 0}; };
        auto re = std::make_unique<RefEngine>();
        re->eng = std::make_unique<run::Engine>(std::move(dec), std::move(bcs), ic, cfg);
        re->eng->init();
        out = re.release();
    });
    return out;
}

void* ref_engine_rect(double x0, double y0, double lx, double ly, int r, int s, int n0, int nv,
                      const int* side_kinds, const double* side_states, const double* side_pressure,
                      double cfl, double T, int workers, const char* weight_path, long max_steps) {
    return ref_engine_affine(x0, y0, lx, 0.0, 0.0, ly, r, s, n0, nv, side_kinds, side_states, side_pressure, cfl, T,
                             workers, weight_path, max_steps);
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_engine_nsubs(void* h) { return static_cast<int>(static_cast<RefEngine*>(h)->eng->subs().size()); }

int ref_engine_dims(void* h, int id, int* ni, int* nj) {
    return guard([&] {
        const auto& d = static_cast<RefEngine*>(h)->eng->subs().at(id);
        *ni = d.ni;
        *nj = d.nj;
    });
}

int ref_engine_get(void* h, int id, const char* what, int comp, double* out) {
    return guard([&] {
        const auto& d = static_cast<RefEngine*>(h)->eng->subs().at(id);
        if (std::string(what) == "mask") {
            for (size_t k = 0; k < d.mask.size(); ++k) out[k] = d.mask[k];
            return;
        }
        const Field* f = field_by_name(d, what, comp);
        std::memcpy(out, f->v.data(), f->v.size() * sizeof(double));
    });
}

int ref_engine_set(void* h, int id, const char* what, int comp, const double* in) {
    return guard([&] {
        auto& d = static_cast<RefEngine*>(h)->eng->subs().at(id);
        Field* f = const_cast<Field*>(field_by_name(d, what, comp));
        std::memcpy(f->v.data(), in, f->v.size() * sizeof(double));
    });
}

int ref_engine_finish_ic(void* h) {
    return guard([&] {
        auto& eng = *static_cast<RefEngine*>(h)->eng;
        for (auto& d : eng.subs()) euler::enforce_bc(d, 0.0);
        eng.exchange_solution();
    });
}

/* Engine::step_phase(worker=0, phase, stage); requires workers == 1. */
int ref_engine_phase(void* h, int phase, int stage) {
    return guard([&] { static_cast<RefEngine*>(h)->eng->step_phase(0, phase, stage); });
}

/* The worker-0 dt block of Engine::run (runtime.cpp:492-497). */
int ref_engine_dt(void* h, double* dt) {
    return guard([&] {
        auto& eng = *static_cast<RefEngine*>(h)->eng;
        double b = std::numeric_limits<double>::infinity();
        for (double v : eng.dt_local_) b = std::min(b, v);
        eng.dt_ = eng.cfg_.cfl * b;
        if (eng.t_ + eng.dt_ > eng.cfg_.T) eng.dt_ = eng.cfg_.T - eng.t_;
        *dt = eng.dt_;
    });
}

int ref_engine_set_dt(void* h, double dt) {
    return guard([&] { static_cast<RefEngine*>(h)->eng->dt_ = dt; });
}

/* The worker-0 advance block of Engine::run (runtime.cpp:505-511). */
int ref_engine_advance(void* h) {
    return guard([&] {
        auto& eng = *static_cast<RefEngine*>(h)->eng;
        eng.t_ += eng.dt_;
        ++eng.step_;
    });
}

int ref_engine_time(void* h, double* t, long* step) {
    auto& eng = *static_cast<RefEngine*>(h)->eng;
    *t = eng.t_;
    *step = eng.step_;
    return 0;
}

/* Engine::run (runtime.cpp:460-530) with the configured worker threads. */
int ref_engine_run(void* h, double* wall_seconds, long* steps, double* t) {
    return guard([&] {
        auto rs = static_cast<RefEngine*>(h)->eng->run();
        *wall_seconds = rs.wall_seconds;
        *steps = rs.steps;
        *t = rs.t;
    });
}

int ref_engine_set_max_steps(void* h, long max_steps) {
    static_cast<RefEngine*>(h)->eng->cfg_.max_steps = max_steps;
    return 0;
}

}  // extern "C"
