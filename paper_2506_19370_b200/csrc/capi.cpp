// extern "C" boundary (include/fcsg.h). Every entry point catches and maps
// exceptions to the reference's error kinds; nothing throws across the ABI.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/fcsg.h"
#include "context.h"
#include "engine.h"
#include "fc_lines.h"

using namespace fcsg;

namespace fcsg {

int Ctx::get_op(int n, int n_cont, int degree, FilterSpec f) {
    auto key = std::make_tuple(n, n_cont, degree, f.alpha, f.p, f.p_smear);
    auto it = op_index.find(key);
    if (it != op_index.end()) return it->second;
    auto op = std::make_unique<DevOp>();
    op->t = build_fc_tables(n, n_cont, degree, f);
    const auto& t = op->t;
    if (static_cast<int>(t.radix.size()) > kMaxStages) throw Error(kConfig, "FFT plan too deep");
    op->d_tw = dev::alloc_n<double2>(t.tw.size());
    op->d_blend = dev::alloc_n<double>(t.blend.size());
    op->d_mult = dev::alloc_n<double2>(t.mult.size());
    dev::h2d(op->d_tw, t.tw.data(), t.tw.size() * sizeof(double2), stream);
    dev::h2d(op->d_blend, t.blend.data(), t.blend.size() * sizeof(double), stream);
    dev::h2d(op->d_mult, t.mult.data(), t.mult.size() * sizeof(double2), stream);
    FcPlanDev& p = op->plan;
    p.n = t.n;
    p.n_ext = t.n_ext;
    p.n_gap = t.n_cont - 1;
    p.dp1 = t.degree + 1;
    p.nstages = static_cast<int>(t.radix.size());
    for (int s = 0; s < p.nstages; ++s) {
        p.radix[s] = t.radix[s];
        p.span[s] = t.span[s];
    }
    p.tw = op->d_tw;
    p.blend = op->d_blend;
    p.mult = op->d_mult;
    p.mult_pfa = nullptr;
    if (!t.mult_pfa.empty()) {
        op->d_mult_pfa = dev::alloc_n<double2>(t.mult_pfa.size());
        dev::h2d(op->d_mult_pfa, t.mult_pfa.data(), t.mult_pfa.size() * sizeof(double2), stream);
        p.mult_pfa = op->d_mult_pfa;
    }
    p.prime_frag = nullptr;
    if (!t.prime_frag.empty()) {
        op->d_prime_frag = dev::alloc_n<double2>(t.prime_frag.size());
        dev::h2d(op->d_prime_frag, t.prime_frag.data(), t.prime_frag.size() * sizeof(double2), stream);
        p.prime_frag = op->d_prime_frag;
    }
    const int id = static_cast<int>(ops.size());
    ops.push_back(std::move(op));
    op_index[key] = id;
    return id;
}

const DevOp& Ctx::op(int id) const {
    if (id < 0 || id >= static_cast<int>(ops.size())) throw Error(kUsage, "bad operator id");
    return *ops[id];
}

}  // namespace fcsg

namespace {

template <class F>
int guard(Ctx* c, F&& f) {
    if (!c) return FCSG_USAGE;
    try {
        // every entry runs on the context's device, whatever the calling
        // thread's current device is (contexts on several devices in one process)
        dev::set_device(c->device);
        f();
        return FCSG_OK;
    } catch (const StateError& e) {
        c->err = e.what();
        c->err_kind = FCSG_INVALID_STATE;
        c->err_patch = e.patch;
        c->err_sub = e.sub;
        c->err_i = e.i;
        c->err_j = e.j;
        c->err_t = e.t;
    } catch (const Error& e) {
        c->err = e.what();
        c->err_kind = e.kind;
    } catch (const std::exception& e) {
        c->err = e.what();
        c->err_kind = FCSG_OTHER;
    }
    return c->err_kind;
}

int pick_lb(long n_lines, int n_ext) {
    static const int forced = [] {  // A/B runs: FCSG_FC_LB = complex lines per CTA (4, 5, 6, 8, 16)
        const char* v = std::getenv("FCSG_FC_LB");
        return v ? std::atoi(v) : 0;
    }();
    if (forced == 4 || forced == 5 || forced == 6 || forced == 8 || forced == 16) return forced;
    // Complex lines per CTA. The compile-time plans (n_ext 280, 536) run three
    // 256-thread CTAs per SM: pick the LB whose grid fills its last wave of
    // 3 x 148 CTAs best (a 1.15-wave grid costs two CTA lifetimes), the
    // smaller LB on ties. Runtime plans: enough CTAs for two per SM,
    // shared memory permitting.
    if (n_ext == 280 || n_ext == 536 || n_ext == 282 || n_ext == 171) {  // fft_line.h has_ct_plan
        const long slots = 3L * 148;
        int best = 4;
        double best_fill = -1.0;
        for (int lb : {4, 5, 6, 8}) {
            const long nblk = (n_lines + 2 * lb - 1) / (2 * lb);
            const long waves = (nblk + slots - 1) / slots;
            const double fill = waves > 0 ? static_cast<double>(nblk) / (waves * slots) : 0.0;
            if (fill > best_fill + 1e-9) {
                best_fill = fill;
                best = lb;
            }
        }
        return best;
    }
    int lb = 16;
    while (lb > 4 && (n_lines + 2 * lb - 1) / (2 * lb) < 296) lb /= 2;
    while (lb > 4 && static_cast<long>(n_ext) * (lb + 1) * 16 > 96 * 1024) lb /= 2;
    return lb;
}

}  // namespace

struct fcsg_ctx : Ctx {};

extern "C" {

int fcsg_is_cuda_build(void) { return dev::is_cuda() ? 1 : 0; }

int fcsg_create(int device, fcsg_ctx** out) {
    if (!out) return FCSG_USAGE;
    auto* c = new fcsg_ctx();
    int rc = guard(c, [&] {
        c->device = device;
        dev::set_device(device);
        c->stream = dev::create_stream();
    });
    if (rc != FCSG_OK) {
        delete c;
        *out = nullptr;
        return rc;
    }
    *out = c;
    return FCSG_OK;
}

int fcsg_destroy(fcsg_ctx* ctx) {
    if (!ctx) return FCSG_OK;
    try {
        dev::sync(ctx->stream);
    } catch (...) {
    }
    ctx->ops.clear();
    dev::destroy_stream(ctx->stream);
    delete ctx;
    return FCSG_OK;
}

int fcsg_last_error(fcsg_ctx* ctx, char* msg, int msg_len, int* kind, int* patch, int* subpatch, int* i,
                    int* j, double* t) {
    if (!ctx) return FCSG_USAGE;
    if (msg && msg_len > 0) {
        std::strncpy(msg, ctx->err.c_str(), msg_len - 1);
        msg[msg_len - 1] = 0;
    }
    if (kind) *kind = ctx->err_kind;
    if (patch) *patch = ctx->err_patch;
    if (subpatch) *subpatch = ctx->err_sub;
    if (i) *i = ctx->err_i;
    if (j) *j = ctx->err_j;
    if (t) *t = ctx->err_t;
    return FCSG_OK;
}

int fcsg_synchronize(fcsg_ctx* ctx) {
    return guard(ctx, [&] { dev::sync(ctx->stream); });
}

int fcsg_device_alloc(fcsg_ctx* ctx, size_t bytes, void** ptr) {
    return guard(ctx, [&] { *ptr = dev::alloc(bytes); });
}
int fcsg_device_free(fcsg_ctx* ctx, void* ptr) {
    return guard(ctx, [&] { dev::free(ptr); });
}
int fcsg_memcpy_h2d(fcsg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guard(ctx, [&] { dev::h2d(dst, src, bytes, ctx->stream); });
}
int fcsg_memcpy_d2h(fcsg_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guard(ctx, [&] { dev::d2h(dst, src, bytes, ctx->stream); });
}

int fcsg_operator(fcsg_ctx* ctx, int n_points, int n_cont, int degree, double alpha, int p, int p_smear,
                  int* op_id) {
    return guard(ctx, [&] {
        FilterSpec f;
        f.alpha = alpha;
        f.p = p;
        f.p_smear = p_smear;
        *op_id = ctx->get_op(n_points, n_cont, degree, f);
    });
}

int fcsg_operator_info(fcsg_ctx* ctx, int op_id, int* n_ext, int* n_modes, double* period, double* blend,
                       double* filter_profile, double* smear_profile) {
    return guard(ctx, [&] {
        const auto& t = ctx->op(op_id).t;
        if (n_ext) *n_ext = t.n_ext;
        if (n_modes) *n_modes = t.n_modes;
        if (period) *period = t.period;
        if (blend) std::memcpy(blend, t.blend.data(), t.blend.size() * sizeof(double));
        if (filter_profile) std::memcpy(filter_profile, t.filter_profile.data(), t.n_modes * sizeof(double));
        if (smear_profile) std::memcpy(smear_profile, t.smear_profile.data(), t.n_modes * sizeof(double));
    });
}

int fcsg_fc_lines(fcsg_ctx* ctx, int op_id, int mode, const double* d_in, long in_line_stride, long in_stride,
                  double* d_out, long out_line_stride, long out_stride, long n_lines, double scale,
                  void* stream) {
    return guard(ctx, [&] {
        if (mode < FCSG_D1 || mode > FCSG_SMEAR) throw Error(kUsage, "fc_derivative: order must be 1 or 2");
        if (n_lines < 0) throw Error(kUsage, "negative line count");
        const auto& op = ctx->op(op_id);
        FcLinesArgs a{};
        a.pl = op.plan;
        a.mode = mode;
        a.in = d_in;
        a.out = d_out;
        a.line_stride = in_line_stride;
        a.stride = in_stride;
        a.out_line_stride = out_line_stride;
        a.out_stride = out_stride;
        a.n_lines = n_lines;
        a.scale = scale;
        launch_fc_lines(a, pick_lb(n_lines, op.t.n_ext), stream);
        dev::check("fc_lines launch");
    });
}

int fcsg_fc_lines_host(fcsg_ctx* ctx, int op_id, int mode, const double* h_in, long in_line_stride,
                       long in_stride, double* h_out, long out_line_stride, long out_stride, long n_lines,
                       double scale) {
    return guard(ctx, [&] {
        const auto& op = ctx->op(op_id);
        const long n = op.t.n;
        const size_t in_elems = n_lines > 0 ? (n_lines - 1) * in_line_stride + (n - 1) * in_stride + 1 : 0;
        const size_t out_elems = n_lines > 0 ? (n_lines - 1) * out_line_stride + (n - 1) * out_stride + 1 : 0;
        double* din = dev::alloc_n<double>(in_elems);
        double* dout = dev::alloc_n<double>(out_elems);
        try {
            dev::h2d(din, h_in, in_elems * sizeof(double), ctx->stream);
            if (h_out != h_in) dev::h2d(dout, h_out, out_elems * sizeof(double), ctx->stream);
            else dev::d2d(dout, din, out_elems * sizeof(double), ctx->stream);
            int rc = fcsg_fc_lines(ctx, op_id, mode, din, in_line_stride, in_stride, dout, out_line_stride,
                                   out_stride, n_lines, scale, ctx->stream);
            if (rc != FCSG_OK) throw Error(ctx->err_kind, ctx->err);
            dev::d2h(h_out, dout, out_elems * sizeof(double), ctx->stream);
        } catch (...) {
            dev::free(din);
            dev::free(dout);
            throw;
        }
        dev::free(din);
        dev::free(dout);
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Engine

struct fcsg_engine {
    Ctx* ctx;
    std::unique_ptr<Engine> eng;
};

extern "C" {

int fcsg_engine_create(fcsg_ctx* ctx, const fcsg_engine_config* cfg, fcsg_engine** out) {
    return guard(ctx, [&] {
        if (!cfg || !out) throw Error(kUsage, "null argument");
        EngineConfig c;
        c.cfl = cfg->cfl;
        c.T = cfg->T;
        c.n_cont = cfg->n_cont;
        c.filter.alpha = cfg->filter_alpha;
        c.filter.p = cfg->filter_p;
        c.filter.p_smear = cfg->filter_p_smear;
        for (int k = 0; k < 4; ++k) c.visc_c[k] = cfg->visc_c[k];
        c.abs_floor = cfg->abs_floor;
        c.smear_radius = cfg->smear_radius;
        c.debug_rhs = cfg->debug_rhs != 0;
        c.allow_cartesian = cfg->force_general == 0;
        c.reference_order = cfg->reference_order != 0;
        c.classifier = cfg->classifier;
        c.classifier_window = cfg->classifier_window;
        auto* e = new fcsg_engine{ctx, std::make_unique<Engine>(*ctx, c)};
        *out = e;
    });
}

int fcsg_engine_destroy(fcsg_engine* eng) {
    if (!eng) return FCSG_OK;
    try {
        dev::sync(eng->ctx->stream);
    } catch (...) {
    }
    delete eng;
    return FCSG_OK;
}

int fcsg_engine_add_subpatch(fcsg_engine* e, int patch, int i0, int j0, int ni, int nj, int cut_i, int cut_j,
                             double h1, double h2, const uint8_t* mask, const double* iq1x, const double* iq2x, const double* iq1y,
                             const double* iq2y, const double* h_min, const double* h_max, const double* w_norm,
                             const int* bc_kind, const double* bc_state, const double* bc_pressure, int* sub_id) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (ni <= 0 || nj <= 0) throw Error(kUsage, "bad subpatch shape");
        SubSpec s;
        s.patch = patch;
        s.i0 = i0;
        s.j0 = j0;
        s.ni = ni;
        s.nj = nj;
        s.cut_i = cut_i;
        s.cut_j = cut_j;
        s.h1 = h1;
        s.h2 = h2;
        const size_t n = static_cast<size_t>(ni) * nj;
        s.mask.assign(mask, mask + n);
        auto cp = [&](const double* p) { return std::vector<double>(p, p + n); };
        s.iq1x = cp(iq1x);
        s.iq2x = cp(iq2x);
        s.iq1y = cp(iq1y);
        s.iq2y = cp(iq2y);
        s.h_min = cp(h_min);
        s.h_max = cp(h_max);
        s.w_norm = cp(w_norm);
        auto bc = [&](int k) {
            BcDev b{};
            b.kind = bc_kind[k];
            if (b.kind < -1 || b.kind > 5) throw Error(kConfig, "bad boundary condition kind");
            for (int c = 0; c < 4; ++c) b.state[c] = bc_state[4 * k + c];
            b.pressure = bc_pressure[k];
            return b;
        };
        int k = 0;
        for (int j = 0; j < nj; ++j) s.row_lo.push_back(bc(k++));
        for (int j = 0; j < nj; ++j) s.row_hi.push_back(bc(k++));
        for (int i = 0; i < ni; ++i) s.col_lo.push_back(bc(k++));
        for (int i = 0; i < ni; ++i) s.col_hi.push_back(bc(k++));
        const int id = e->eng->add_subpatch(std::move(s));
        if (sub_id) *sub_id = id;
    });
}

int fcsg_engine_set_plan_interps(fcsg_engine* e, int which, long n, const int* dst_sub, const int* dst,
                                 const int* src_sub, const int* si0, const int* sj0, const double* wx, const double* wy,
                                 const double* w) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (n < 0) throw Error(kUsage, "bad interpolation count");
        auto vi = [&](const int* p) { return std::vector<int>(p, p + n); };
        std::vector<double> vw = (which == 1 && n > 0) ? std::vector<double>(w, w + n) : std::vector<double>();
        e->eng->set_plan_interps(which, vi(dst_sub), vi(dst), vi(src_sub), vi(si0), vi(sj0),
                                 std::vector<double>(wx, wx + 6 * n), std::vector<double>(wy, wy + 6 * n), vw);
    });
}

int fcsg_engine_set_plan(fcsg_engine* e, long n_sol, const int* sol_dst_sub, const int* sol_dst,
                         const int* sol_src_sub, const int* sol_src, long n_visc, const int* v_dst_sub,
                         const int* v_dst, const int* v_src_sub, const int* v_src, const double* v_w) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        auto vi = [](const int* p, long n) { return p ? std::vector<int>(p, p + n) : std::vector<int>(); };
        e->eng->set_plan(vi(sol_dst_sub, n_sol), vi(sol_dst, n_sol), vi(sol_src_sub, n_sol), vi(sol_src, n_sol),
                         vi(v_dst_sub, n_visc), vi(v_dst, n_visc), vi(v_src_sub, n_visc), vi(v_src, n_visc),
                         v_w ? std::vector<double>(v_w, v_w + n_visc) : std::vector<double>());
    });
}

int fcsg_engine_load_mlp(fcsg_engine* e, const char* path) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->load_mlp_file(path ? path : ""); });
}

int fcsg_engine_finalize(fcsg_engine* e) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->finalize(); });
}

int fcsg_engine_set_state(fcsg_engine* e, int sub, const double* e4) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->set_state(sub, e4); });
}

int fcsg_engine_get_field(fcsg_engine* e, int sub, const char* name, int comp, double* out) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->get_field(sub, name, comp, out); });
}

int fcsg_engine_gradient(fcsg_engine* e, int comp) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->gradient(comp); });
}

int fcsg_engine_set_quadrature(fcsg_engine* e, int sub, const double* wq) {
    if (!e || !wq) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->set_quadrature(sub, wq); });
}

int fcsg_engine_integrals(fcsg_engine* e, int comp, double* per_sub) {
    if (!e || !per_sub) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->integrals(comp, per_sub); });
}

int fcsg_engine_sample(fcsg_engine* e, long n, const int* sub, const int* il, const int* jl, const double* fu,
                       const double* fv, double* out) {
    if (!e || (n > 0 && (!sub || !il || !jl || !fu || !fv || !out))) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->sample(n, sub, il, jl, fu, fv, out); });
}

int fcsg_engine_set_field(fcsg_engine* e, int sub, const char* name, int comp, const double* in) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->set_field(sub, name, comp, in); });
}

int fcsg_engine_finish_ic(fcsg_engine* e) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->finish_ic(); });
}

int fcsg_engine_phase(fcsg_engine* e, int phase, int stage) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->phase(phase, stage); });
}

int fcsg_engine_reduce_dt(fcsg_engine* e, double* dt) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *dt = e->eng->reduce_dt(); });
}

int fcsg_engine_advance(fcsg_engine* e) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->advance(); });
}

int fcsg_engine_run(fcsg_engine* e, long n, int use_graph, long* done) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        const long d = e->eng->run_steps(n, use_graph != 0);
        if (done) *done = d;
    });
}

int fcsg_engine_enqueue(fcsg_engine* e, long n) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->enqueue_steps(n); });
}

int fcsg_engine_time(fcsg_engine* e, double* t, long* steps) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (t) *t = e->eng->time();
        if (steps) *steps = e->eng->steps();
    });
}

int fcsg_engine_total_points(fcsg_engine* e, long* n) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *n = e->eng->total_points(); });
}

int fcsg_engine_is_cartesian(fcsg_engine* e, int* yes) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *yes = e->eng->cartesian() ? 1 : 0; });
}

int fcsg_engine_stream(fcsg_engine* e, void** stream) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *stream = e->eng->stream(); });
}

}  // extern "C"

extern "C" {

int fcsg_engine_time_group(fcsg_engine* e, int which, int reps, double* ms) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *ms = e->eng->time_pass(which, reps); });
}

int fcsg_engine_launches_per_step(fcsg_engine* e, int* n) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *n = e->eng->launches_per_step(); });
}

}  // extern "C"

extern "C" {

int fcsg_engine_run_host(fcsg_engine* e, long n, const double* in, long in_stride, double* out, long out_stride,
                         long* done) {
    if (!e || !in || !out) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        const long d = e->eng->run_host(n, in, in_stride, out, out_stride);
        if (done) *done = d;
    });
}

int fcsg_engine_set_state_bulk(fcsg_engine* e, const double* e4s) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->set_state_bulk(e4s); });
}

int fcsg_engine_get_state_bulk(fcsg_engine* e, double* out) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->get_state_bulk(out); });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// multi-rank halo exchange and the part-wise superstep

extern "C" {

int fcsg_engine_set_halo_interps(fcsg_engine* e, int which, long n, const int* sub, const int* si0, const int* sj0,
                                 const double* wx, const double* wy) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (n < 0) throw Error(kUsage, "bad interpolation count");
        auto vi = [&](const int* p) { return std::vector<int>(p, p + n); };
        e->eng->set_halo_interps(which, vi(sub), vi(si0), vi(sj0), std::vector<double>(wx, wx + 6 * n),
                                 std::vector<double>(wy, wy + 6 * n));
    });
}

int fcsg_engine_set_halo(fcsg_engine* e, long n_send_e, const int* e_sub, const int* e_loc, long n_recv_e,
                         long n_send_mu, const int* mu_sub, const int* mu_loc, long n_recv_mu) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        auto vi = [](const int* p, long n) { return (p && n > 0) ? std::vector<int>(p, p + n) : std::vector<int>(); };
        e->eng->set_halo(vi(e_sub, n_send_e), vi(e_loc, n_send_e), n_recv_e, vi(mu_sub, n_send_mu),
                         vi(mu_loc, n_send_mu), n_recv_mu);
    });
}

int fcsg_engine_halo_size(fcsg_engine* e, int which, long* n) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *n = e->eng->halo_size(which); });
}

int fcsg_engine_pack(fcsg_engine* e, int which, void* d_buf) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (which == 0) e->eng->pack_e(static_cast<double*>(d_buf));
        else if (which == 1) e->eng->pack_mu(static_cast<double*>(d_buf));
        else throw Error(kUsage, "bad halo selector");
        dev::check("pack");
    });
}

int fcsg_engine_unpack(fcsg_engine* e, int which, const void* d_buf) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (which == 0) e->eng->unpack_e(static_cast<const double*>(d_buf));
        else if (which == 1) e->eng->unpack_mu(static_cast<const double*>(d_buf));
        else throw Error(kUsage, "bad halo selector");
        dev::check("unpack");
    });
}

int fcsg_engine_enqueue_part(fcsg_engine* e, int part, int stage) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { e->eng->enqueue_part(part, stage); });
}

int fcsg_engine_dtmin_ptr(fcsg_engine* e, void** dptr) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] { *dptr = e->eng->dtmin_device_ptr(); });
}

int fcsg_comm_unique_id(char* id) {
    if (!id) return FCSG_USAGE;
    try {  // no context (and no device switch): rank 0 calls this before any engine exists
        comm_unique_id(id);
        return FCSG_OK;
    } catch (const Error& e) {
        return e.kind;
    } catch (...) {
        return FCSG_OTHER;
    }
}

int fcsg_engine_attach_comm(fcsg_engine* e, int nranks, int rank, const char* id, int n_peers, const int* peers,
                            const long* e_send, const long* e_recv, const long* mu_send, const long* mu_recv) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        if (!id || n_peers < 0 || (n_peers > 0 && !(peers && e_send && e_recv && mu_send && mu_recv)))
            throw Error(kUsage, "bad transport arguments");
        auto vl = [n_peers](const long* p) { return std::vector<long>(p, p + n_peers); };
        std::vector<int> pv(peers, peers + n_peers);
        dev::set_device(e->ctx->device);
        auto comm = comm_create(nranks, rank, id);
        e->eng->attach_comm(std::move(comm), pv, vl(e_send), vl(e_recv), vl(mu_send), vl(mu_recv));
    });
}

int fcsg_engine_check_error(fcsg_engine* e) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        dev::sync(e->ctx->stream);
        e->eng->check_error();
    });
}

}  // extern "C"

extern "C" {

int fcsg_engine_copy_dtmin(fcsg_engine* e, void* d_buf, int to_engine) {
    if (!e) return FCSG_USAGE;
    return guard(e->ctx, [&] {
        void* p = e->eng->dtmin_device_ptr();
        if (to_engine) dev::d2d(p, d_buf, 8, e->ctx->stream);
        else dev::d2d(d_buf, p, 8, e->ctx->stream);
    });
}

}  // extern "C"
