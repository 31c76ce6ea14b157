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
 *   ref_engine_problem -> wb::get_problem (problems.cpp:379-388), and the
 *                        SubpatchData / CommPlan exporters (sub_info, lines,
 *                        plan) that feed the same geometry and plan to the product
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
#include "fcs/workbench.hpp"  // after runtime.hpp, which it includes

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
    if (w == "det") return &d.det;
    if (w == "grad") return &d.s1;  // |grad rho| after density_gradient_raster
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

/* Classifier::classify_line (fallback variant: FC-spectrum decay). */
int ref_classify_line_fallback(int window, double abs_floor, int n, const double* values, int* tau) {
    return guard([&] {
        visc::ClassifierConfig cc;
        cc.variant = visc::ClassifierConfig::Variant::fallback;
        cc.window = window;
        cc.abs_floor = abs_floor;
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

/* A named problem of the reference's workbench (flow-cylinder, wedge, prism,
 * riemann4, sod, ...) with its own initial condition applied by
 * Engine::init; cfl / T <= 0 keep the problem's values. */
void* ref_engine_problem(const char* name, double target_h, double cfl, double T, int workers,
                         const char* weight_path, long max_steps) {
    RefEngine* out = nullptr;
    guard([&] {
        wb::ProblemSpec ps = wb::get_problem(name, target_h);
        run::EngineConfig cfg;
        cfg.cfl = cfl > 0 ? cfl : ps.cfl;
        cfg.T = T > 0 ? T : ps.T;
        cfg.workers = workers;
        cfg.max_steps = max_steps;
        if (weight_path && weight_path[0]) {
            cfg.classifier.variant = visc::ClassifierConfig::Variant::ann;
            cfg.classifier.weight_path = weight_path;
        }
        auto re = std::make_unique<RefEngine>();
        re->eng = std::make_unique<run::Engine>(std::move(ps.dec), std::move(ps.bcs), ps.ic, cfg);
        re->eng->init();
        out = re.release();
    });
    return out;
}

/* Test geometries built through the reference's own geometry API (its named
 * multi-patch problems -- flow-cylinder, wedge, prism, shock-cylinder-matrix
 * -- fail their own minimum-overlap / window checks):
 *   0  annulus: one periodic S patch (AnnulusMap, r 0.5..1), 3 subpatches,
 *      curved no-slip wall inside, zero_normal_all outside
 *   1  two patches with non-coincident lattices: a Cartesian I patch and a
 *      bilinear S patch overlapping it (6x6 Lagrange interpolation both ways),
 *      slip walls, inflow, supersonic outflow
 *   3  the config-3 cylinder layout of problems.cylinder_flow(full=False):
 *      periodic annulus r in [1, 2.2] (subdivide_Q(8, 1, 65, 9)) and four
 *      Cartesian I patches (n0 = 120) over [-4, 12] x [-6, 6], Mach 3 free
 *      stream, slip walls, inflow / supersonic outflow (n0 ignored)
 *   5  the config-4 forward-facing step layout of problems.step_flow(1): C1
 *      corner patch at the step's top (0.6, 0.2) (one L-shaped subpatch),
 *      S patches along the step top and face, two I patches (256 x 256
 *      subpatches); Mach 3 inflow, supersonic outflow, slip walls (n0 ignored)
 *   6  the same at scale 2 (problems.step_flow(2): 3.22M points, the C1
 *      patch's L-shaped subpatch 139 x 139 with rows of 139 and 70 points)
 *   4  the same at full size (problems.cylinder_flow(full=True): annulus
 *      subdivide_Q(16, 1, 129, 9), Cartesian n0 = 238; 2.57M points)
 *   2  a C1 corner patch alone (CurveSumMap of two non-orthogonal segments,
 *      subdivide_L: one L-shaped subpatch), slip walls at the reentrant
 *      corner; the overlap validation that asks for an S patch at the corner
 *      is skipped (every fringe point of the lone patch is intra-patch)
 * n0: points per preliminary cell (n1 for the C1 patch); IC: uniform flow
 * plus a Gaussian density bump, applied by Engine::init. */
void* ref_engine_testgeom(int which, int n0, int nv, double cfl, int workers, const char* weight_path) {
    RefEngine* out = nullptr;
    guard([&] {
        using geom::Patch;
        using geom::PatchKind;
        using geom::SideInfo;
        const SideInfo interior{false, ""};
        geom::DomainDecomposition dec;
        dec.nv = nv;
        dec.n0 = n0;
        BcTable bcs;
        BcSpec slip;
        slip.kind = BcKind::slip_wall;
        BcSpec noslip;
        noslip.kind = BcKind::noslip_adiabatic;
        BcSpec zn;
        zn.kind = BcKind::zero_normal_all;
        BcSpec sup;
        sup.kind = BcKind::supersonic_outflow;
        BcSpec in;
        in.kind = BcKind::inflow;
        in.state = euler::conservative(1.0, 0.5, 0.0, 0.7);
        bcs["wall"] = slip;
        bcs["cyl"] = noslip;
        bcs["outer"] = zn;
        bcs["out"] = sup;
        bcs["in"] = in;
        Vec2 bump{0.0, 0.0};
        double u0 = 0.5, v0 = 0.0;
        bool free_stream = false;
        if (which == 0) {
            Patch ring;
            ring.kind = PatchKind::S;
            ring.map = std::make_shared<geom::AnnulusMap>(Vec2{0.0, 0.0}, 0.5, 1.0, -M_PI, 2 * M_PI);
            ring.periodic1 = true;
            ring.sides = {interior, interior, SideInfo{true, "cyl"}, SideInfo{true, "outer"}};
            dec.patches.push_back(std::move(ring));
            bump = {0.75, 0.0};
            u0 = 0.2;
            v0 = 0.1;
        } else if (which == 1) {
            Patch a;
            a.kind = PatchKind::I;
            a.map = std::make_shared<geom::AffineMap>(Vec2{0.0, 0.0}, Vec2{1.0, 0.0}, Vec2{0.0, 1.05});
            a.sides = {SideInfo{true, "in"}, interior, SideInfo{true, "wall"}, SideInfo{true, "wall"}};
            dec.patches.push_back(std::move(a));
            Patch b;
            b.kind = PatchKind::S;
            // a trapezoid: walls continue A's walls through the overlap, the
            // outflow side is slanted (non-constant Jacobian)
            b.map = std::make_shared<geom::BilinearMap>(Vec2{0.5, 0.0}, Vec2{1.8, 0.0}, Vec2{0.5, 1.05},
                                                        Vec2{1.5, 1.05});
            b.sides = {interior, SideInfo{true, "out"}, SideInfo{true, "wall"}, SideInfo{true, "wall"}};
            dec.patches.push_back(std::move(b));
            bump = {0.85, 0.5};
        } else if (which == 2) {
            const Vec2 c{0.5, 0.5};
            const double arm = 0.3, ang = 70.0 * M_PI / 180.0;
            const Vec2 da{1.0, 0.0}, db{std::cos(ang), std::sin(ang)};
            auto ellA = std::make_shared<geom::Segment>(c + arm * da, c - arm * da);
            auto ellB = std::make_shared<geom::Segment>(c + arm * db, c - arm * db);
            Patch p = geom::build_c1_patch(ellA, ellB, c, "wall");
            for (auto& sd : p.sides) sd = SideInfo{true, "outer"};
            dec.patches.push_back(std::move(p));
            bump = {0.6, 0.6};
            u0 = 0.3;
            v0 = 0.2;
        } else if (which == 3 || which == 4) {
            Patch ring;
            ring.kind = PatchKind::S;
            ring.map = std::make_shared<geom::AnnulusMap>(Vec2{0.0, 0.0}, 1.0, 2.2, -M_PI, 2 * M_PI);
            ring.periodic1 = true;
            ring.sides = {interior, interior, SideInfo{true, "wall"}, interior};
            dec.patches.push_back(std::move(ring));
            auto rect = [&](Vec2 o, Vec2 e1, Vec2 e2, std::array<SideInfo, 4> sd) {
                Patch p;
                p.kind = PatchKind::I;
                p.map = std::make_shared<geom::AffineMap>(o, e1, e2);
                p.sides = sd;
                dec.patches.push_back(std::move(p));
            };
            rect({-4.0, -6.0}, {2.8, 0.0}, {0.0, 12.0},
                 {SideInfo{true, "in"}, interior, SideInfo{true, "wall"}, SideInfo{true, "wall"}});
            rect({1.2, -6.0}, {10.8, 0.0}, {0.0, 12.0},
                 {interior, SideInfo{true, "out"}, SideInfo{true, "wall"}, SideInfo{true, "wall"}});
            rect({-1.7, 1.2}, {3.4, 0.0}, {0.0, 4.8}, {interior, interior, interior, SideInfo{true, "wall"}});
            rect({-1.7, -6.0}, {3.4, 0.0}, {0.0, 4.8}, {interior, interior, SideInfo{true, "wall"}, interior});
            bcs["in"].state = euler::conservative(1.4, 3.0, 0.0, 1.0);
            free_stream = true;
        } else if (which == 5 || which == 6) {
            const Vec2 c{0.6, 0.2};
            const double a = 0.15;
            auto ellA = std::make_shared<geom::Segment>(Vec2{c.x + a, c.y}, Vec2{c.x - a, c.y});
            auto ellB = std::make_shared<geom::Segment>(Vec2{c.x, c.y - a}, Vec2{c.x, c.y + a});
            Patch p = geom::build_c1_patch(ellA, ellB, c, "wall");
            dec.patches.push_back(std::move(p));
            auto rect = [&](PatchKind kind, Vec2 o, Vec2 e1, Vec2 e2, std::array<SideInfo, 4> sd) {
                Patch q;
                q.kind = kind;
                q.map = std::make_shared<geom::AffineMap>(o, e1, e2);
                q.sides = sd;
                dec.patches.push_back(std::move(q));
            };
            rect(PatchKind::I, {0.0, 0.0}, {0.57, 0.0}, {0.0, 1.0},
                 {SideInfo{true, "in"}, interior, SideInfo{true, "wall"}, SideInfo{true, "wall"}});
            rect(PatchKind::I, {0.4, 0.26}, {2.6, 0.0}, {0.0, 0.74},
                 {interior, SideInfo{true, "out"}, interior, SideInfo{true, "wall"}});
            rect(PatchKind::S, {0.6, 0.2}, {2.4, 0.0}, {0.0, 0.25},
                 {interior, SideInfo{true, "out"}, SideInfo{true, "wall"}, interior});
            // concave corner at the step's foot: C2 between the floor and the face
            dec.patches.push_back(geom::build_c2_patch(std::make_shared<geom::Segment>(Vec2{0.3, 0.0}, Vec2{0.6, 0.0}),
                                                       std::make_shared<geom::Segment>(Vec2{0.6, 0.2}, Vec2{0.6, 0.0}),
                                                       Vec2{0.6, 0.0}, "wall"));
            bcs["in"].state = euler::conservative(1.4, 3.0, 0.0, 1.0);
            free_stream = true;
        } else {
            throw UsageError("unknown test geometry");
        }
        for (size_t k = 0; k < dec.patches.size(); ++k) dec.patches[k].index = static_cast<int>(k);
        if (which == 5 || which == 6) {
            const int k = which == 5 ? 1 : 2;  // problems.step_flow(k)
            const int rs[5][2] = {{2, 0}, {1, 2}, {5, 1}, {4, 1}, {1, 1}};
            for (auto& p : dec.patches) {
                if (p.kind == PatchKind::C1)
                    geom::subdivide_L(p, 2 * k, 59, nv);
                else
                    geom::subdivide_Q(p, k * rs[p.index][0], k * rs[p.index][1], 238, nv);
            }
        } else if (which == 3 || which == 4) {
            const bool full = which == 4;
            const int rs[5][2] = {{full ? 16 : 8, 1}, {1, 5}, {5, 5}, {1, 2}, {1, 2}};
            for (auto& p : dec.patches)
                geom::subdivide_Q(p, rs[p.index][0], rs[p.index][1], p.index ? (full ? 238 : 120) : (full ? 129 : 65),
                                  nv);
        } else {
            for (auto& p : dec.patches) {
                if (p.kind == PatchKind::C1)
                    geom::subdivide_L(p, 2, n0, nv);
                else if (p.periodic1)
                    geom::subdivide_Q(p, 3, 1, n0, nv);
                else if (p.index == 1)
                    geom::subdivide_Q(p, 2, 1, n0 + 6, nv);  // a different lattice and subpatch shape
                else
                    geom::subdivide_Q(p, 1, 1, n0, nv);
            }
        }
        dec.assign_global_ids();
        run::EngineConfig cfg;
        cfg.cfl = cfl;
        cfg.T = 1e300;
        cfg.workers = workers;
        // a lone C1 patch has no S patch at its corner; its plan is complete
        // without one (every fringe point is intra-patch)
        if (which == 2) cfg.validate_overlap = false;
        if (weight_path && weight_path[0]) {
            cfg.classifier.variant = visc::ClassifierConfig::Variant::ann;
            cfg.classifier.weight_path = weight_path;
        }
        auto ic = [bump, u0, v0, free_stream](double x, double y) {
            if (free_stream) return euler::conservative(1.4, 3.0, 0.0, 1.0);
            const double r2 = (x - bump.x) * (x - bump.x) + (y - bump.y) * (y - bump.y);
            const double rho = 1.0 + 0.2 * std::exp(-r2 / 0.02);
            return euler::conservative(rho, u0, v0, 0.7);
        };
        auto re = std::make_unique<RefEngine>();
        re->eng = std::make_unique<run::Engine>(std::move(dec), std::move(bcs), ic, cfg);
        re->eng->init();
        out = re.release();
    });
    return out;
}

/* info[9] = patch index, i0, j0, ni, nj, cut_i, cut_j (local; 0 = rectangle),
 * periodic1, patch kind; hh[2] = h1, h2 (geom::Patch / Subpatch) */
int ref_engine_sub_info(void* h, int id, int* info, double* hh) {
    return guard([&] {
        const auto& d = static_cast<RefEngine*>(h)->eng->subs().at(id);
        const auto& sp = *d.sp;
        const auto& p = *d.patch;
        info[0] = p.index;
        info[1] = sp.i0;
        info[2] = sp.j0;
        info[3] = d.ni;
        info[4] = d.nj;
        const bool l = sp.i_cut > sp.i0 && sp.j_cut > sp.j0;
        info[5] = l ? sp.i_cut - sp.i0 : 0;
        info[6] = l ? sp.j_cut - sp.j0 : 0;
        info[7] = p.periodic1 ? 1 : 0;
        info[8] = static_cast<int>(p.kind);
        hh[0] = p.h1;
        hh[1] = p.h2;
    });
}

/* LineInfo tables (include/fcs/subpatch_data.hpp:34-43): per line (rows then
 * columns) begin, n, inv_len, and the resolved BC of both ends: kind (-1 none,
 * else the BcKind order), state[4], pressure. Arrays sized nj + ni. */
int ref_engine_lines(void* h, int id, int* begin, int* n, double* inv_len, int* kind_lo, double* bc_lo, int* kind_hi,
                     double* bc_hi) {
    return guard([&] {
        const auto& d = static_cast<RefEngine*>(h)->eng->subs().at(id);
        int k = 0;
        auto put = [&](const SubpatchData::LineInfo& li) {
            begin[k] = li.begin;
            n[k] = li.n;
            inv_len[k] = li.inv_len;
            const BcSpec* b[2] = {li.bc_lo, li.bc_hi};
            int* kk[2] = {kind_lo, kind_hi};
            double* bb[2] = {bc_lo, bc_hi};
            for (int e = 0; e < 2; ++e) {
                kk[e][k] = b[e] ? static_cast<int>(b[e]->kind) : -1;
                for (int c = 0; c < 4; ++c) bb[e][5 * k + c] = b[e] ? b[e]->state[c] : 0.0;
                bb[e][5 * k + 4] = b[e] ? b[e]->pressure : 1.0;
            }
            ++k;
        };
        for (const auto& li : d.rows) put(li);
        for (const auto& li : d.cols) put(li);
    });
}

/* CommPlan entries of recipient `id` (include/fcs/runtime.hpp:16-49); which
 * 0 = solution, 1 = viscosity. counts[2] = copies, interps. With non-null
 * arrays: copies (dst, src_sub, src) + copy_w; interps (dst, src_sub, si0,
 * sj0) + interp_w (wx[6], wy[6], w). */
int ref_engine_plan(void* h, int id, int which, int* counts, int* copies, double* copy_w, int* interps,
                    double* interp_w) {
    return guard([&] {
        const auto& plan = static_cast<RefEngine*>(h)->eng->plan();
        const auto& pe = (which == 0 ? plan.solution : plan.visc).at(id);
        counts[0] = static_cast<int>(pe.copies.size());
        counts[1] = static_cast<int>(pe.interps.size());
        if (copies) {
            for (size_t k = 0; k < pe.copies.size(); ++k) {
                copies[3 * k] = pe.copies[k].dst;
                copies[3 * k + 1] = pe.copies[k].src_sub;
                copies[3 * k + 2] = pe.copies[k].src;
                copy_w[k] = pe.copies[k].w;
            }
        }
        if (interps) {
            for (size_t k = 0; k < pe.interps.size(); ++k) {
                const auto& e = pe.interps[k];
                interps[4 * k] = e.dst;
                interps[4 * k + 1] = e.src_sub;
                interps[4 * k + 2] = e.si0;
                interps[4 * k + 3] = e.sj0;
                for (int a = 0; a < 6; ++a) {
                    interp_w[13 * k + a] = e.wx[a];
                    interp_w[13 * k + 6 + a] = e.wy[a];
                }
                interp_w[13 * k + 12] = e.w;
            }
        }
    });
}

/* DomainDecomposition::to_json (src/geometry.cpp:573-594) of the engine's
 * decomposition, dumped; *len = full length (truncated to cap - 1). */
int ref_engine_mesh_json(void* h, char* buf, long cap, long* len) {
    return guard([&] {
        const std::string t = static_cast<RefEngine*>(h)->eng->dec().to_json().dump();
        *len = static_cast<long>(t.size());
        if (cap > 0) {
            const size_t n = std::min<size_t>(t.size(), static_cast<size_t>(cap - 1));
            std::memcpy(buf, t.data(), n);
            buf[n] = 0;
        }
    });
}

/* DomainDecomposition::from_json (src/geometry.cpp:596-629) of a mesh file's
 * text, written back with to_json: what the reference makes of a mesh file. */
int ref_mesh_roundtrip(const char* in, char* buf, long cap, long* len) {
    return guard([&] {
        const auto dec = geom::DomainDecomposition::from_json(nlohmann::json::parse(in));
        const std::string t = dec.to_json().dump();
        *len = static_cast<long>(t.size());
        if (cap > 0) {
            const size_t n = std::min<size_t>(t.size(), static_cast<size_t>(cap - 1));
            std::memcpy(buf, t.data(), n);
            buf[n] = 0;
        }
    });
}

/* energy_integral / area_integral (src/workbench.cpp:212-220) */
int ref_engine_integrals(void* h, double* energy, double* area) {
    return guard([&] {
        const auto& eng = *static_cast<RefEngine*>(h)->eng;
        *energy = wb::energy_integral(eng);
        *area = wb::area_integral(eng);
    });
}

/* density_gradient_raster (src/workbench.cpp:222-305): v[ny][nx], meta = x0, y0, dx, dy */
int ref_engine_raster(void* h, int nx, int ny, double* v, double* meta) {
    return guard([&] {
        const wb::Raster r = wb::density_gradient_raster(*static_cast<RefEngine*>(h)->eng, nx, ny);
        std::copy(r.v.begin(), r.v.end(), v);
        meta[0] = r.x0;
        meta[1] = r.y0;
        meta[2] = r.dx;
        meta[3] = r.dy;
    });
}

namespace {
wb::Raster raster_of(int nx, int ny, const double* meta, const double* v) {
    wb::Raster r;
    r.nx = nx;
    r.ny = ny;
    r.x0 = meta[0];
    r.y0 = meta[1];
    r.dx = meta[2];
    r.dy = meta[3];
    r.v.assign(v, v + static_cast<size_t>(nx) * ny);
    return r;
}
}  // namespace

/* write_pgm(schlieren(raster, beta)) (src/workbench.cpp:307-333) */
int ref_write_schlieren_pgm(int nx, int ny, const double* meta, const double* v, double beta, const char* path) {
    return guard([&] { wb::write_pgm(wb::schlieren(raster_of(nx, ny, meta, v), beta), path); });
}

/* fit_shock_angle (src/workbench.cpp:335-366) */
int ref_fit_shock_angle(int nx, int ny, const double* meta, const double* v, double x_lo, double x_hi, double y_lo,
                        double y_hi, double* deg) {
    return guard([&] { *deg = wb::fit_shock_angle(raster_of(nx, ny, meta, v), x_lo, x_hi, y_lo, y_hi); });
}

/* write_subpatch_csv (src/workbench.cpp:368-386) */
int ref_engine_write_csv(void* h, const char* dir) {
    return guard([&] { wb::write_subpatch_csv(*static_cast<RefEngine*>(h)->eng, dir); });
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
