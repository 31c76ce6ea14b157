// Step-seam binding (see run_fcsg.hpp). TEST INFRASTRUCTURE.
#include "run_fcsg.hpp"

#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "fcs/errors.hpp"
#include "fcsg.h"

namespace fcs::run {

namespace {

struct Ctx {
    fcsg_ctx* c = nullptr;
    fcsg_engine* e = nullptr;
    ~Ctx() {
        if (e) fcsg_engine_destroy(e);
        if (c) fcsg_destroy(c);
    }
    void check(int rc) const {
        if (rc == FCSG_OK) return;
        char msg[512] = {0};
        int kind = rc, patch = -1, sub = -1, i = -1, j = -1;
        double t = 0.0;
        fcsg_last_error(c, msg, sizeof msg, &kind, &patch, &sub, &i, &j, &t);
        switch (kind) {
            case FCSG_CONFIG: throw ConfigError(msg);
            case FCSG_USAGE: throw UsageError(msg);
            case FCSG_GEOMETRY: throw GeometryError(msg);
            case FCSG_DECOMPOSITION: throw DecompositionError(msg);
            case FCSG_INVALID_STATE: throw InvalidStateError(msg, patch, sub, i, j, t);
            default: throw std::runtime_error(msg);
        }
    }
};

// one line end's resolved BC: kind (-1 none), conservative state, pressure
void push_bc(const BcSpec* b, std::vector<int>& kind, std::vector<double>& st, std::vector<double>& pr) {
    kind.push_back(b ? static_cast<int>(b->kind) : -1);
    for (int c = 0; c < 4; ++c) st.push_back(b ? b->state[c] : 0.0);
    pr.push_back(b ? b->pressure : 1.0);
}

}  // namespace

Engine::RunStats run_fcsg(Engine& eng, const EngineConfig& cfg, long max_steps, int device) {
    Ctx g;
    g.check(fcsg_create(device, &g.c));
    const bool ann = cfg.classifier.variant == visc::ClassifierConfig::Variant::ann;
    fcsg_engine_config ec{};
    ec.cfl = cfg.cfl;
    ec.T = cfg.T;
    ec.n_cont = cfg.n_cont;
    ec.filter_alpha = cfg.filter.alpha;
    ec.filter_p = cfg.filter.p;
    ec.filter_p_smear = cfg.filter.p_smear;
    for (int k = 0; k < 4; ++k) ec.visc_c[k] = cfg.visc_weights.c[k];
    ec.abs_floor = cfg.classifier.abs_floor;
    ec.smear_radius = cfg.smear_radius;
    ec.classifier = ann ? 0 : 1;
    ec.classifier_window = cfg.classifier.window;
    g.check(fcsg_engine_create(g.c, &ec, &g.e));

    auto& subs = eng.subs();
    // SubpatchData -> device (init_subpatch_data's output, src/subpatch_data.cpp:69-154)
    for (const SubpatchData& d : subs) {
        std::vector<int> kind;
        std::vector<double> st, pr;
        for (const auto& li : d.rows) push_bc(li.bc_lo, kind, st, pr);
        for (const auto& li : d.rows) push_bc(li.bc_hi, kind, st, pr);
        for (const auto& li : d.cols) push_bc(li.bc_lo, kind, st, pr);
        for (const auto& li : d.cols) push_bc(li.bc_hi, kind, st, pr);
        const auto& sp = *d.sp;
        const bool l = sp.i_cut > sp.i0 && sp.j_cut > sp.j0;  // L-shaped (C1) subpatch
        int id = -1;
        g.check(fcsg_engine_add_subpatch(g.e, d.patch->index, sp.i0, sp.j0, d.ni, d.nj, l ? sp.i_cut - sp.i0 : 0,
                                         l ? sp.j_cut - sp.j0 : 0, d.patch->h1, d.patch->h2, d.mask.data(),
                                         d.iq1x.v.data(), d.iq2x.v.data(), d.iq1y.v.data(), d.iq2y.v.data(),
                                         d.h_min.v.data(), d.h_max.v.data(), d.w_norm.v.data(), kind.data(), st.data(),
                                         pr.data(), &id));
        if (id != d.id) throw UsageError("run_fcsg: subpatch ids must be 0..n-1 in order");
    }
    // CommPlan (include/fcs/runtime.hpp:16-49), flattened by recipient in the
    // reference's order: copies, then interpolations
    const CommPlan& plan = eng.plan();
    struct Flat {
        std::vector<int> dst_sub, dst, src_sub, src;
        std::vector<double> w;
        std::vector<int> idst_sub, idst, isrc_sub, si0, sj0;
        std::vector<double> wx, wy, iw;
    } fl[2];
    for (int which = 0; which < 2; ++which) {
        const auto& sets = which == 0 ? plan.solution : plan.visc;
        Flat& f = fl[which];
        for (size_t r = 0; r < sets.size(); ++r) {
            for (const CopyEntry& c : sets[r].copies) {
                f.dst_sub.push_back(static_cast<int>(r));
                f.dst.push_back(c.dst);
                f.src_sub.push_back(c.src_sub);
                f.src.push_back(c.src);
                f.w.push_back(c.w);
            }
            for (const InterpEntry& it : sets[r].interps) {
                f.idst_sub.push_back(static_cast<int>(r));
                f.idst.push_back(it.dst);
                f.isrc_sub.push_back(it.src_sub);
                f.si0.push_back(it.si0);
                f.sj0.push_back(it.sj0);
                f.wx.insert(f.wx.end(), it.wx.begin(), it.wx.end());
                f.wy.insert(f.wy.end(), it.wy.begin(), it.wy.end());
                f.iw.push_back(it.w);
            }
        }
    }
    g.check(fcsg_engine_set_plan(g.e, static_cast<long>(fl[0].dst.size()), fl[0].dst_sub.data(), fl[0].dst.data(),
                                 fl[0].src_sub.data(), fl[0].src.data(), static_cast<long>(fl[1].dst.size()),
                                 fl[1].dst_sub.data(), fl[1].dst.data(), fl[1].src_sub.data(), fl[1].src.data(),
                                 fl[1].w.data()));
    for (int which = 0; which < 2; ++which) {
        const Flat& f = fl[which];
        if (f.idst.empty()) continue;
        g.check(fcsg_engine_set_plan_interps(g.e, which, static_cast<long>(f.idst.size()), f.idst_sub.data(),
                                             f.idst.data(), f.isrc_sub.data(), f.si0.data(), f.sj0.data(),
                                             f.wx.data(), f.wy.data(), which == 1 ? f.iw.data() : nullptr));
    }
    if (ann) g.check(fcsg_engine_load_mlp(g.e, cfg.classifier.weight_path.c_str()));
    g.check(fcsg_engine_finalize(g.e));
    // State after init() (apply_ic: IC, enforce_bc, one exchange), [4][nj][ni]
    for (const SubpatchData& d : subs) {
        std::vector<double> e4;
        for (const Field& f : d.e) e4.insert(e4.end(), f.v.begin(), f.v.end());
        g.check(fcsg_engine_set_state(g.e, d.id, e4.data()));
    }
    const auto t0 = std::chrono::steady_clock::now();
    long done = 0;
    g.check(fcsg_engine_run(g.e, max_steps, 1, &done));
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (SubpatchData& d : subs)
        for (int c = 0; c < 4; ++c) g.check(fcsg_engine_get_field(g.e, d.id, "e", c, d.e[c].v.data()));
    Engine::RunStats rs;
    long steps = 0;
    g.check(fcsg_engine_time(g.e, &rs.t, &steps));
    rs.steps = steps;
    rs.wall_seconds = wall;
    rs.seconds_per_step = steps > 0 ? wall / steps : 0.0;
    return rs;
}

}  // namespace fcs::run
