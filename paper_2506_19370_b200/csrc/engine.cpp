// Host Engine (see engine.h). Device layout: every per-point field is one
// contiguous array over all subpatches, [sub][j][i] (the reference's Field
// order, include/fcs/field.hpp:9-23), so a subpatch is a (nj, ni) slab and a
// point has the global index sub*ni*nj + j*ni + i. All subpatches of one
// engine share one rectangular shape (every configuration measured here);
// the FC operators for rows (n = ni) and columns (n = nj) are shared too.
#include "engine.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <numeric>

namespace fcsg {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();
}

Engine::Engine(Ctx& ctx, const EngineConfig& cfg) : ctx_(ctx), cfg_(cfg) {}

Engine::~Engine() {
    if (graph_exec_) dev::graph_destroy(graph_exec_, graph_);
    for (void* p : allocs_) dev::free(p);
}

int Engine::add_subpatch(SubSpec s) {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    const size_t n = static_cast<size_t>(s.ni) * s.nj;
    if (s.ni < 10 || s.nj < 10) throw Error(kConfig, "FcOperator: n_points must be >= 10");
    if (!subs_.empty() && (s.ni != subs_[0].ni || s.nj != subs_[0].nj))
        throw Error(kUsage, "all subpatches of one engine must share one shape");
    auto chk = [&](const std::vector<double>& v, const char* nm) {
        if (v.size() != n) throw Error(kUsage, std::string("subpatch field size mismatch: ") + nm);
    };
    if (s.mask.size() != n) throw Error(kUsage, "subpatch mask size mismatch");
    chk(s.iq1x, "iq1x");
    chk(s.iq2x, "iq2x");
    chk(s.iq1y, "iq1y");
    chk(s.iq2y, "iq2y");
    chk(s.h_min, "h_min");
    chk(s.h_max, "h_max");
    chk(s.w_norm, "w_norm");
    for (auto m : s.mask)
        if (m == 0) throw Error(kUsage, "L-shaped subpatches are not supported by this engine");
    subs_.push_back(std::move(s));
    return static_cast<int>(subs_.size()) - 1;
}

void Engine::set_plan(std::vector<int> sol_dst_sub, std::vector<int> sol_dst, std::vector<int> sol_src_sub,
                      std::vector<int> sol_src, std::vector<int> v_dst_sub, std::vector<int> v_dst,
                      std::vector<int> v_src_sub, std::vector<int> v_src, std::vector<double> v_w) {
    if (subs_.empty()) throw Error(kUsage, "add subpatches before the plan");
    const long sz = static_cast<long>(subs_[0].ni) * subs_[0].nj;
    const int S = static_cast<int>(subs_.size());
    const long np = sz * S;
    auto gidx = [&](int sub, int loc) -> long {
        if (sub < 0 || sub >= S || loc < 0 || loc >= sz) throw Error(kUsage, "plan entry out of range");
        return sub * sz + loc;
    };
    // donors on other ranks (src_sub == -1) live in the halo slots after the local points
    auto sidx = [&](int sub, int loc, long n_halo) -> long {
        if (sub == -1) {
            if (loc < 0 || loc >= n_halo) throw Error(kUsage, "halo slot out of range");
            return np + loc;
        }
        return gidx(sub, loc);
    };
    x_dst_.clear();
    x_src_.clear();
    for (size_t k = 0; k < sol_dst.size(); ++k) {
        x_dst_.push_back(gidx(sol_dst_sub[k], sol_dst[k]));
        x_src_.push_back(sidx(sol_src_sub[k], sol_src[k], n_recv_e_));
    }
    // CSR by recipient point, keeping the given (reference) order per point
    std::vector<long> dsts(v_dst.size());
    for (size_t k = 0; k < v_dst.size(); ++k) dsts[k] = gidx(v_dst_sub[k], v_dst[k]);
    std::vector<size_t> order(v_dst.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return dsts[a] < dsts[b]; });
    visc_off_.assign(np + 1, 0);
    visc_src_.clear();
    visc_w_.clear();
    for (size_t k : order) {
        visc_off_[dsts[k] + 1]++;
        visc_src_.push_back(sidx(v_src_sub[k], v_src[k], n_recv_mu_));
        visc_w_.push_back(v_w[k]);
    }
    for (long p = 0; p < np; ++p) visc_off_[p + 1] += visc_off_[p];
    have_plan_ = true;
}

void Engine::set_halo(std::vector<int> e_sub, std::vector<int> e_loc, long n_recv_e, std::vector<int> mu_sub,
                      std::vector<int> mu_loc, long n_recv_mu) {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    if (have_plan_) throw Error(kUsage, "set the halo before the plan");
    if (e_sub.size() != e_loc.size() || mu_sub.size() != mu_loc.size() || n_recv_e < 0 || n_recv_mu < 0)
        throw Error(kUsage, "bad halo lists");
    halo_e_src_.clear();
    halo_mu_src_.clear();
    for (size_t k = 0; k < e_sub.size(); ++k) halo_e_src_.emplace_back(e_sub[k], e_loc[k]);
    for (size_t k = 0; k < mu_sub.size(); ++k) halo_mu_src_.emplace_back(mu_sub[k], mu_loc[k]);
    n_recv_e_ = n_recv_e;
    n_recv_mu_ = n_recv_mu;
}

long Engine::halo_size(int which) const {
    switch (which) {
        case 0: return static_cast<long>(halo_e_src_.size());
        case 1: return n_recv_e_;
        case 2: return static_cast<long>(halo_mu_src_.size());
        case 3: return n_recv_mu_;
    }
    throw Error(kUsage, "bad halo selector");
}

void Engine::pack_e(double* d_buf) { launch_pack(E_, 0, d_halo_e_, static_cast<long>(halo_e_.size()), d_buf, ctx_.stream); }
void Engine::unpack_e(const double* d_buf) { launch_unpack(E_, 0, n_recv_e_, d_buf, ctx_.stream); }
void Engine::pack_mu(double* d_buf) { launch_pack(E_, 1, d_halo_mu_, static_cast<long>(halo_mu_.size()), d_buf, ctx_.stream); }
void Engine::unpack_mu(const double* d_buf) { launch_unpack(E_, 1, n_recv_mu_, d_buf, ctx_.stream); }

void Engine::enqueue_part(int part, int stage) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    void* s = ctx_.stream;
    switch (part) {
        case -1: launch_bc(E_, s); break;
        case 0: launch_phase0(E_, host_step_ == 0, s); break;
        case 1: launch_phase1(E_, s); break;
        case 2:
            launch_phase2(E_, plans_, host_step_ == 0, s);
            launch_bc(E_, s);
            launch_finalize_dt(E_, s);
            break;
        case 3:
            if (stage < 0 || stage > 4) throw Error(kUsage, "bad stage");
            launch_stage(E_, plans_, stage, s);
            launch_bc(E_, s);
            break;
        case 4: launch_exchange(E_, s); break;
        case 5:
            launch_advance(E_, s);
            ++host_step_;
            break;
        default: throw Error(kUsage, "bad step part");
    }
    dev::check("enqueue_part");
}

void Engine::set_mlp_packed(const std::vector<double>& w) {
    if (static_cast<int>(w.size()) != kMlpWeights) throw Error(kConfig, "weight file has wrong input/output dimensions");
    mlp_ = w;
    if (finalized_) {
        dev::h2d(const_cast<double*>(E_.mlp), mlp_.data(), mlp_.size() * sizeof(double), ctx_.stream);
        const std::vector<double> fr = mlp_mma_fragments(mlp_);
        dev::h2d(const_cast<double*>(E_.mlp_frag), fr.data(), fr.size() * sizeof(double), ctx_.stream);
    }
}

void Engine::load_mlp_file(const std::string& path) {
    // MlpClassifier::load (src/viscosity.cpp:63-89)
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Error(kConfig, "classifier weights not found: " + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "FCNN", 4) != 0) throw Error(kConfig, "bad weight file magic");
    auto rd = [&]() {
        uint32_t v = 0;
        is.read(reinterpret_cast<char*>(&v), 4);
        return v;
    };
    if (rd() != 1) throw Error(kConfig, "unsupported weight file version");
    const uint32_t act = rd();
    const uint32_t nl = rd();
    const int want_r[kMlpLayers] = {16, 16, 16, 16, 4}, want_c[kMlpLayers] = {7, 16, 16, 16, 16};
    if (act != 1 || nl != kMlpLayers) throw Error(kConfig, "weight file has wrong input/output dimensions");
    std::vector<double> packed;
    for (uint32_t l = 0; l < nl; ++l) {
        const int r = static_cast<int>(rd()), c = static_cast<int>(rd());
        if (r != want_r[l] || c != want_c[l]) throw Error(kConfig, "weight file has wrong input/output dimensions");
        std::vector<double> w(static_cast<size_t>(r) * c), b(r);
        is.read(reinterpret_cast<char*>(w.data()), w.size() * sizeof(double));
        is.read(reinterpret_cast<char*>(b.data()), b.size() * sizeof(double));
        packed.insert(packed.end(), w.begin(), w.end());
        packed.insert(packed.end(), b.begin(), b.end());
    }
    if (!is) throw Error(kConfig, "truncated weight file: " + path);
    set_mlp_packed(packed);
}

void Engine::finalize() {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    if (subs_.empty()) throw Error(kUsage, "engine has no subpatches");
    if (mlp_.empty()) throw Error(kConfig, "ann classifier requires a weight file path");
    const int S = static_cast<int>(subs_.size());
    ni_ = subs_[0].ni;
    nj_ = subs_[0].nj;
    const long sz = static_cast<long>(ni_) * nj_;
    npts_ = sz * S;
    op_row_ = ctx_.get_op(ni_, cfg_.n_cont, 2, cfg_.filter);
    op_col_ = ctx_.get_op(nj_, cfg_.n_cont, 2, cfg_.filter);
    plans_.row = ctx_.op(op_row_).plan;
    plans_.col = ctx_.op(op_col_).plan;
    plans_.scr_row = step_scr_cap(plans_.row);
    plans_.scr_col = step_scr_cap(plans_.col);

    auto up = [&](const void* h, size_t bytes) {
        void* d = dev::alloc(bytes);
        allocs_.push_back(d);
        dev::h2d(d, h, bytes, ctx_.stream);
        return d;
    };
    EngineDev& E = E_;
    E.S = S;
    E.ni = ni_;
    E.nj = nj_;
    E.npts = npts_;
    if (npts_ >= (1L << 31)) throw Error(kConfig, "more than 2^31 points on one device");
    E.div_ni = make_fastdiv(static_cast<unsigned>(ni_));
    E.div_sz = make_fastdiv(static_cast<unsigned>(sz));
    E.cfl = cfg_.cfl;
    E.T = cfg_.T;
    for (int k = 0; k < 4; ++k) E.visc_c[k] = cfg_.visc_c[k];
    E.abs_floor = cfg_.abs_floor;
    E.smear_radius = cfg_.smear_radius;
    E.cartesian = cfg_.allow_cartesian ? 1 : 0;
    E.reference_order = cfg_.reference_order ? 1 : 0;
    for (const auto& sp : subs_)
        for (size_t k = 0; k < sp.iq2x.size(); ++k)
            if (sp.iq2x[k] != 0.0 || sp.iq1y[k] != 0.0) E.cartesian = 0;
    std::vector<double> il1(S), il2(S);
    std::vector<int> i0(S), j0(S), pt(S);
    std::vector<BcDev> rlo, rhi, clo, chi;
    std::vector<uint8_t> mask;
    std::vector<double> geo[7];
    for (int s = 0; s < S; ++s) {
        const auto& sp = subs_[s];
        // SubpatchData::LineInfo::inv_len (src/subpatch_data.cpp:134,147)
        il1[s] = 1.0 / ((sp.ni - 1) * sp.h1);
        il2[s] = 1.0 / ((sp.nj - 1) * sp.h2);
        i0[s] = sp.i0;
        j0[s] = sp.j0;
        pt[s] = sp.patch;
        auto pad = [](const std::vector<BcDev>& v, size_t n) {
            std::vector<BcDev> o = v;
            BcDev none{};
            none.kind = -1;
            o.resize(n, none);
            return o;
        };
        auto a = pad(sp.row_lo, nj_), b = pad(sp.row_hi, nj_), c = pad(sp.col_lo, ni_), d = pad(sp.col_hi, ni_);
        rlo.insert(rlo.end(), a.begin(), a.end());
        rhi.insert(rhi.end(), b.begin(), b.end());
        clo.insert(clo.end(), c.begin(), c.end());
        chi.insert(chi.end(), d.begin(), d.end());
        mask.insert(mask.end(), sp.mask.begin(), sp.mask.end());
        const std::vector<double>* src[7] = {&sp.iq1x, &sp.iq2x, &sp.iq1y, &sp.iq2y, &sp.h_min, &sp.h_max, &sp.w_norm};
        for (int k = 0; k < 7; ++k) geo[k].insert(geo[k].end(), src[k]->begin(), src[k]->end());
    }
    E.inv_len1 = static_cast<const double*>(up(il1.data(), S * sizeof(double)));
    E.inv_len2 = static_cast<const double*>(up(il2.data(), S * sizeof(double)));
    E.sub_i0 = static_cast<const int*>(up(i0.data(), S * sizeof(int)));
    E.sub_j0 = static_cast<const int*>(up(j0.data(), S * sizeof(int)));
    E.sub_patch = static_cast<const int*>(up(pt.data(), S * sizeof(int)));
    E.bc_row_lo = static_cast<const BcDev*>(up(rlo.data(), rlo.size() * sizeof(BcDev)));
    E.bc_row_hi = static_cast<const BcDev*>(up(rhi.data(), rhi.size() * sizeof(BcDev)));
    E.bc_col_lo = static_cast<const BcDev*>(up(clo.data(), clo.size() * sizeof(BcDev)));
    E.bc_col_hi = static_cast<const BcDev*>(up(chi.data(), chi.size() * sizeof(BcDev)));
    E.mask = static_cast<const uint8_t*>(up(mask.data(), mask.size()));
    const double** gp[7] = {&E.iq1x, &E.iq2x, &E.iq1y, &E.iq2y, &E.h_min, &E.h_max, &E.w_norm};
    for (int k = 0; k < 7; ++k) *gp[k] = static_cast<const double*>(up(geo[k].data(), geo[k].size() * sizeof(double)));

    // state + temporaries in one pool; every field has room for the halo
    // slots after its npts local points
    const int n_fields = 4 * 5 + (cfg_.debug_rhs ? 4 : 0) + 7 + 4 * 4;
    const size_t fstride = npts_ + std::max(n_recv_e_, n_recv_mu_);
    pool_ = dev::alloc_n<double>(static_cast<size_t>(n_fields) * fstride);
    allocs_.push_back(pool_);
    dev::memset0(pool_, static_cast<size_t>(n_fields) * fstride * sizeof(double), ctx_.stream);
    int f = 0;
    auto nextf = [&]() { return pool_ + static_cast<size_t>(f++) * fstride; };
    for (int c = 0; c < 4; ++c) E.e[c] = nextf();
    for (int c = 0; c < 4; ++c) E.e0[c] = nextf();
    for (int c = 0; c < 4; ++c) E.e2[c] = nextf();
    for (int c = 0; c < 4; ++c) E.e3[c] = nextf();
    for (int c = 0; c < 4; ++c) E.rhs3[c] = nextf();
    for (int c = 0; c < 4; ++c) E.rhs[c] = cfg_.debug_rhs ? nextf() : nullptr;
    E.mu_hat = nextf();
    E.mu = nextf();
    E.tau = nextf();
    E.speed = nextf();
    E.proxy = nextf();
    E.seed = nextf();
    E.m01 = nextf();
    for (int c = 0; c < 4; ++c) E.tA[c] = nextf();
    for (int c = 0; c < 4; ++c) E.tW[c] = nextf();
    for (int c = 0; c < 4; ++c) E.tS4[c] = nextf();
    for (int c = 0; c < 4; ++c) E.tS5[c] = nextf();
    for (int c = 0; c < 4; ++c) E.tF[c] = E.tA[c];  // phase 2 and the stage passes never overlap
    // tau starts at 4 everywhere (Classifier::classify fills 4, src/viscosity.cpp:212)
    {
        std::vector<double> four(npts_, 4.0), one(npts_, 1.0);
        dev::h2d(E.tau, four.data(), npts_ * sizeof(double), ctx_.stream);
        dev::h2d(E.speed, one.data(), npts_ * sizeof(double), ctx_.stream);
    }
    if (have_plan_) {
        if (!x_dst_.empty()) {
            E.x_dst = static_cast<const long*>(up(x_dst_.data(), x_dst_.size() * sizeof(long)));
            E.x_src = static_cast<const long*>(up(x_src_.data(), x_src_.size() * sizeof(long)));
        }
        E.n_x = static_cast<long>(x_dst_.size());
        if (!visc_src_.empty()) {
            E.visc_off = static_cast<const int*>(up(visc_off_.data(), visc_off_.size() * sizeof(int)));
            E.visc_src = static_cast<const long*>(up(visc_src_.data(), visc_src_.size() * sizeof(long)));
            E.visc_w = static_cast<const double*>(up(visc_w_.data(), visc_w_.size() * sizeof(double)));
        }
    }
    E.mlp = static_cast<const double*>(up(mlp_.data(), mlp_.size() * sizeof(double)));
    {
        const std::vector<double> fr = mlp_mma_fragments(mlp_);
        E.mlp_frag = static_cast<const double*>(up(fr.data(), fr.size() * sizeof(double)));
    }
    {
        std::vector<double> tt(kTanhTable);
        for (int k = 0; k < kTanhTable; ++k) tt[k] = static_cast<double>(tanhl(static_cast<long double>(k) / 64.0L));
        E.tanh_tab = static_cast<const double*>(up(tt.data(), tt.size() * sizeof(double)));
    }
    halo_e_.clear();
    halo_mu_.clear();
    for (auto [sb, lc] : halo_e_src_) {
        if (sb < 0 || sb >= S || lc < 0 || lc >= sz) throw Error(kUsage, "halo donor out of range");
        halo_e_.push_back(sb * sz + lc);
    }
    for (auto [sb, lc] : halo_mu_src_) {
        if (sb < 0 || sb >= S || lc < 0 || lc >= sz) throw Error(kUsage, "halo donor out of range");
        halo_mu_.push_back(sb * sz + lc);
    }
    if (!halo_e_.empty()) d_halo_e_ = static_cast<long*>(up(halo_e_.data(), halo_e_.size() * sizeof(long)));
    if (!halo_mu_.empty()) d_halo_mu_ = static_cast<long*>(up(halo_mu_.data(), halo_mu_.size() * sizeof(long)));
    StepScalars sc{};
    double inf = kInf;
    std::memcpy(&sc.dtmin_bits, &inf, 8);
    E.sc = static_cast<StepScalars*>(up(&sc, sizeof(sc)));
    finalized_ = true;
}

double* Engine::field_ptr(const std::string& w, int c) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (c < 0 || c > 3) throw Error(kUsage, "bad component");
    const EngineDev& E = E_;
    if (w == "e") return E.e[c];
    if (w == "e0") return E.e0[c];
    if (w == "e2") return E.e2[c];
    if (w == "e3") return E.e3[c];
    if (w == "rhs3") return E.rhs3[c];
    if (w == "rhs") {
        if (!E.rhs[0]) throw Error(kUsage, "rhs is kept only with debug_rhs");
        return E.rhs[c];
    }
    if (w == "mu_hat") return E.mu_hat;
    if (w == "mu") return E.mu;
    if (w == "tau") return E.tau;
    if (w == "speed") return E.speed;
    if (w == "proxy") return E.proxy;
    if (w == "m01") return E.m01;
    if (w == "iq1x") return const_cast<double*>(E.iq1x);
    if (w == "iq2x") return const_cast<double*>(E.iq2x);
    if (w == "iq1y") return const_cast<double*>(E.iq1y);
    if (w == "iq2y") return const_cast<double*>(E.iq2y);
    if (w == "h_min") return const_cast<double*>(E.h_min);
    if (w == "h_max") return const_cast<double*>(E.h_max);
    if (w == "w_norm") return const_cast<double*>(E.w_norm);
    throw Error(kUsage, "unknown field " + w);
}

void Engine::set_state(int sub, const double* e4) {
    if (sub < 0 || sub >= E_.S) throw Error(kUsage, "bad subpatch id");
    const long sz = static_cast<long>(ni_) * nj_;
    for (int c = 0; c < 4; ++c) dev::h2d(E_.e[c] + sub * sz, e4 + c * sz, sz * sizeof(double), ctx_.stream);
}

void Engine::set_state_bulk(const double* e) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    for (int c = 0; c < 4; ++c) dev::h2d_async(E_.e[c], e + c * npts_, npts_ * sizeof(double), ctx_.stream);
    dev::sync(ctx_.stream);
}

void Engine::get_state_bulk(double* e) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    for (int c = 0; c < 4; ++c) dev::d2h_async(e + c * npts_, E_.e[c], npts_ * sizeof(double), ctx_.stream);
    dev::sync(ctx_.stream);
}

void Engine::get_field(int sub, const std::string& name, int comp, double* out) {
    if (sub < 0 || sub >= E_.S) throw Error(kUsage, "bad subpatch id");
    const long sz = static_cast<long>(ni_) * nj_;
    dev::d2h(out, field_ptr(name, comp) + sub * sz, sz * sizeof(double), ctx_.stream);
}

void Engine::set_field(int sub, const std::string& name, int comp, const double* in) {
    if (sub < 0 || sub >= E_.S) throw Error(kUsage, "bad subpatch id");
    const long sz = static_cast<long>(ni_) * nj_;
    dev::h2d(field_ptr(name, comp) + sub * sz, in, sz * sizeof(double), ctx_.stream);
}

void Engine::check_error() {
    StepScalars sc;
    dev::d2h(&sc, E_.sc, sizeof(sc), ctx_.stream);
    if (sc.err.code == 0) return;
    // clear so the engine can report the next failure
    StepScalars clr = sc;
    clr.err = DevError{0, 0, 0, 0};
    dev::h2d(E_.sc, &clr, sizeof(clr), ctx_.stream);
    const auto& sp = subs_.at(sc.err.sub);
    const char* msg = sc.err.code == 1   ? "nonpositive density or pressure"
                      : sc.err.code == 2 ? "nonpositive density or pressure (viscosity proxy)"
                                         : "nonfinite wave speed";
    throw StateError(msg, sp.patch, sc.err.sub, sp.i0 + sc.err.i, sp.j0 + sc.err.j, sc.t);
}

void Engine::finish_ic() {
    launch_bc(E_, ctx_.stream);
    launch_exchange(E_, ctx_.stream);
    dev::check("finish_ic");
    dev::sync(ctx_.stream);
}

void Engine::phase(int ph, int stage) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    switch (ph) {
        case 0: launch_phase0(E_, host_step_ == 0, ctx_.stream); break;
        case 1: launch_phase1(E_, ctx_.stream); break;
        case 2:
            launch_phase2(E_, plans_, host_step_ == 0, ctx_.stream);
            launch_bc(E_, ctx_.stream);
            break;
        case 3:
            if (stage < 0 || stage > 4) throw Error(kUsage, "bad stage");
            launch_stage(E_, plans_, stage, ctx_.stream);
            launch_bc(E_, ctx_.stream);
            break;
        case 6: launch_exchange(E_, ctx_.stream); break;
        default: throw Error(kUsage, "bad phase");
    }
    dev::check("phase");
    dev::sync(ctx_.stream);
    check_error();
}

double Engine::reduce_dt() {
    launch_finalize_dt(E_, ctx_.stream);
    dev::check("finalize_dt");
    StepScalars sc;
    dev::d2h(&sc, E_.sc, sizeof(sc), ctx_.stream);
    return sc.dt;
}

void Engine::advance() {
    launch_advance(E_, ctx_.stream);
    dev::check("advance");
    dev::sync(ctx_.stream);
    ++host_step_;
}

double Engine::time() {
    StepScalars sc;
    dev::d2h(&sc, E_.sc, sizeof(sc), ctx_.stream);
    return sc.t;
}

void Engine::enqueue_step(bool step0) {
    void* s = ctx_.stream;
    launch_phase0(E_, step0, s);
    launch_phase1(E_, s);
    launch_phase2(E_, plans_, step0, s);
    launch_bc(E_, s);
    launch_finalize_dt(E_, s);
    for (int st = 0; st < 5; ++st) {
        launch_stage(E_, plans_, st, s);
        launch_bc(E_, s);
        launch_exchange(E_, s);
    }
    launch_advance(E_, s);
}

void Engine::launch_group(int which) {
    void* s = ctx_.stream;
    switch (which) {
        case 0: launch_phase0(E_, false, s); break;
        case 1: launch_phase1(E_, s); break;
        case 2: launch_phase2(E_, plans_, false, s); break;
        case 3: launch_pass_a(E_, plans_, s); break;
        case 4: launch_pass_b(E_, plans_, 1, s); break;
        case 5: launch_pass_c(E_, plans_, 1, s); break;
        case 6: launch_bc(E_, s); break;
        case 7: launch_exchange(E_, s); break;
        default: throw Error(kUsage, "bad launch group");
    }
}

double Engine::time_pass(int which, int reps) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (reps < 1) reps = 1;
    launch_group(which);  // warm
    struct Arg {
        Engine* e;
        int which, reps;
    } a{this, which, reps};
    const double ms = dev::time_on_stream(
        ctx_.stream,
        [](void* p) {
            auto* q = static_cast<Arg*>(p);
            for (int r = 0; r < q->reps; ++r) q->e->launch_group(q->which);
        },
        &a);
    dev::check("time_pass");
    return ms / reps;
}

void Engine::enqueue_steps(long n) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    for (long k = 0; k < n; ++k) {
        if (host_step_ == 0 || !dev::is_cuda()) {
            enqueue_step(host_step_ == 0);
        } else {
            if (!graph_exec_) {
                dev::graph_begin(ctx_.stream);
                enqueue_step(false);
                dev::graph_end(ctx_.stream, &graph_, &graph_exec_);
            }
            dev::graph_launch(graph_exec_, ctx_.stream);
        }
        ++host_step_;
    }
    dev::check("enqueue");
}

long Engine::run_steps(long n, bool use_graph) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    const bool finite_T = std::isfinite(cfg_.T);
    long done = 0;
    for (; done < n; ++done) {
        if (finite_T && time() >= cfg_.T - 1e-15) break;
        const bool step0 = host_step_ == 0;
        if (step0 || !use_graph || !dev::is_cuda()) {
            enqueue_step(step0);
        } else {
            if (!graph_exec_) {
                dev::graph_begin(ctx_.stream);
                enqueue_step(false);
                dev::graph_end(ctx_.stream, &graph_, &graph_exec_);
            }
            dev::graph_launch(graph_exec_, ctx_.stream);
        }
        dev::check("step");
        ++host_step_;
        if (finite_T) {
            dev::sync(ctx_.stream);
            check_error();
        }
    }
    dev::sync(ctx_.stream);
    check_error();
    return done;
}

}  // namespace fcsg
