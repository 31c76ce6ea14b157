// Host Engine (see engine.h). Device layout: every per-point field is one
// contiguous array over all subpatches, [sub][j][i] (the reference's Field
// order, include/fcs/field.hpp:9-23), so a subpatch is a (nj, ni) slab and a
// point has the global index sub*ni*nj + j*ni + i. Subpatches of any shapes
// are stored grouped by shape (layout()); each group shares its row and
// column FC operators.
#include "engine.h"

#include "classify_f32.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>

#if !defined(FCSG_EMULATE)
#include <nvtx3/nvToolsExt.h>
#endif

namespace fcsg {

namespace {
constexpr double kInf = std::numeric_limits<double>::infinity();

// NVTX range around host-side enqueueing of a phase / stage (nsys, ncu
// --nvtx --nvtx-include "fcsg stage 1/"): the reference's RunStats timing
// (src/runtime.cpp:469,522-528) split by phase. Inside CUDA-graph capture the
// ranges mark the capture; eager steps (step 0, the phase hooks,
// FCSG_NO_GRAPH) carry them per launch.
struct Range {
    explicit Range(const char* name) {
#if !defined(FCSG_EMULATE)
        nvtxRangePushA(name);
#else
        (void)name;
#endif
    }
    ~Range() {
#if !defined(FCSG_EMULATE)
        nvtxRangePop();
#endif
    }
    Range(const Range&) = delete;
    Range& operator=(const Range&) = delete;
};
void range_push(const char* name) {
#if !defined(FCSG_EMULATE)
    nvtxRangePushA(name);
#else
    (void)name;
#endif
}
void range_pop() {
#if !defined(FCSG_EMULATE)
    nvtxRangePop();
#endif
}
const char* kStageRange[5] = {"fcsg stage 0", "fcsg stage 1", "fcsg stage 2", "fcsg stage 3", "fcsg stage 4"};
}

Engine::Engine(Ctx& ctx, const EngineConfig& cfg) : ctx_(ctx), cfg_(cfg) {
    if (const char* v = std::getenv("FCSG_STAGE_CHUNKS")) cfg_.stage_chunks = std::atoi(v);
}

Engine::~Engine() {
    if (graph_exec_) dev::graph_destroy(graph_exec_, graph_);
    if (ev_fork_) dev::destroy_event(ev_fork_);
    if (ev_join_) dev::destroy_event(ev_join_);
    if (side_) dev::destroy_stream(side_);
    for (int b = 0; b < 2; ++b)
        for (void* e : {ev_in_ready_[b], ev_in_used_[b], ev_out_ready_[b], ev_out_done_[b]})
            if (e) dev::destroy_event(e);
    if (cp_in_) dev::destroy_stream(cp_in_);
    if (cp_out_) dev::destroy_stream(cp_out_);
    for (void* e : cevents_) dev::destroy_event(e);
    for (void* st : cstreams_) dev::destroy_stream(st);
    if (ev_stage_) dev::destroy_event(ev_stage_);
    for (void* p : allocs_) dev::free(p);
}

int Engine::add_subpatch(SubSpec s) {
    if (finalized_ || laid_out_) throw Error(kUsage, "add every subpatch before the plan, halo and finalize");
    const size_t n = static_cast<size_t>(s.ni) * s.nj;
    if (s.cut_i < 0 || s.cut_j < 0 || s.cut_i >= s.ni || s.cut_j >= s.nj || ((s.cut_i == 0) != (s.cut_j == 0)))
        throw Error(kUsage, "bad L-cut");
    // FcOperator needs n >= 10 on every line (src/fc_core.cpp:192-193)
    if (s.ni - s.cut_i < 10 || s.nj - s.cut_j < 10) throw Error(kConfig, "FcOperator: n_points must be >= 10");
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
    for (int j = 0; j < s.nj; ++j)
        for (int i = 0; i < s.ni; ++i) {
            const bool in_set = !(i < s.cut_i && j < s.cut_j);
            if ((s.mask[static_cast<size_t>(j) * s.ni + i] != 0) != in_set)
                throw Error(kUsage, "mask must be 0 exactly outside the subpatch's point set");
        }
    subs_.push_back(std::move(s));
    return static_cast<int>(subs_.size()) - 1;
}

// Storage order: shape groups in order of first appearance, ids ascending
// within a group (a group view is then one contiguous slab).
void Engine::layout() {
    if (laid_out_) return;
    if (subs_.empty()) throw Error(kUsage, "engine has no subpatches");
    groups_.clear();
    std::vector<std::vector<int>> members;
    for (int id = 0; id < static_cast<int>(subs_.size()); ++id) {
        const auto& sp = subs_[id];
        size_t g = 0;
        while (g < groups_.size() && !(groups_[g].ni == sp.ni && groups_[g].nj == sp.nj)) ++g;
        if (g == groups_.size()) {
            groups_.push_back(Group{sp.ni, sp.nj, 0, 0, 0, 0});
            members.emplace_back();
        }
        members[g].push_back(id);
    }
    // multi-rank: inside each group the subpatches owning donors of the state
    // halo come first, so a stage's edge run can be passed, packed and sent
    // while the interior run is still being passed (enqueue_step)
    std::vector<char> edge(subs_.size(), 0);
    for (const auto& h : halo_e_src_)
        if (h.first >= 0 && h.first < static_cast<int>(subs_.size())) edge[h.first] = 1;
    for (size_t g = 0; g < groups_.size(); ++g) {
        auto& m = members[g];
        std::stable_partition(m.begin(), m.end(), [&](int id) { return edge[id] != 0; });
        groups_[g].n_edge = static_cast<int>(std::count_if(m.begin(), m.end(), [&](int id) { return edge[id] != 0; }));
    }
    slot_of_.assign(subs_.size(), -1);
    id_of_slot_.clear();
    off_of_slot_.clear();
    long off = 0;
    for (size_t g = 0; g < groups_.size(); ++g) {
        groups_[g].slot0 = static_cast<int>(id_of_slot_.size());
        groups_[g].n = static_cast<int>(members[g].size());
        groups_[g].p0 = off;
        for (int id : members[g]) {
            slot_of_[id] = static_cast<int>(id_of_slot_.size());
            id_of_slot_.push_back(id);
            off_of_slot_.push_back(off);
            off += sub_points(id);
        }
    }
    npts_ = off;
    if (npts_ >= (1L << 31)) throw Error(kConfig, "more than 2^31 points on one device");
    laid_out_ = true;
}

long Engine::gidx(int sub, int loc) const {
    if (sub < 0 || sub >= static_cast<int>(subs_.size()) || loc < 0 || loc >= sub_points(sub))
        throw Error(kUsage, "plan entry out of range");
    return off_of_slot_[slot_of_[sub]] + loc;
}

void Engine::set_plan(std::vector<int> sol_dst_sub, std::vector<int> sol_dst, std::vector<int> sol_src_sub,
                      std::vector<int> sol_src, std::vector<int> v_dst_sub, std::vector<int> v_dst,
                      std::vector<int> v_src_sub, std::vector<int> v_src, std::vector<double> v_w) {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    layout();
    const long np = npts_;
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

void Engine::set_plan_interps(int which, std::vector<int> dst_sub, std::vector<int> dst, std::vector<int> src_sub,
                              std::vector<int> si0, std::vector<int> sj0, std::vector<double> wx,
                              std::vector<double> wy, std::vector<double> w) {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    if (which != 0 && which != 1) throw Error(kUsage, "bad interpolation set");
    layout();
    const size_t n = dst.size();
    if (dst_sub.size() != n || src_sub.size() != n || si0.size() != n || sj0.size() != n || wx.size() != 6 * n ||
        wy.size() != 6 * n || (which == 1 && w.size() != n))
        throw Error(kUsage, "interpolation arrays of inconsistent length");
    std::vector<long> d(n), s0(n);
    std::vector<int> pitch(n);
    for (size_t k = 0; k < n; ++k) {
        d[k] = gidx(dst_sub[k], dst[k]);
        const int ss = src_sub[k];
        if (ss == -1 && which == 1) {  // evaluated by the donor's rank into halo slot si0
            if (si0[k] < 0 || si0[k] >= n_recv_mu_) throw Error(kUsage, "halo slot out of range");
            s0[k] = npts_ + si0[k];
            pitch[k] = 0;
            continue;
        }
        if (ss < 0 || ss >= static_cast<int>(subs_.size()))
            throw Error(kUsage, "interpolation donors must be local subpatches");
        const auto& sp = subs_[ss];
        if (si0[k] < 0 || sj0[k] < 0 || si0[k] + 6 > sp.ni || sj0[k] + 6 > sp.nj)
            throw Error(kUsage, "interpolation stencil outside the donor subpatch");
        s0[k] = gidx(ss, sj0[k] * sp.ni + si0[k]);
        pitch[k] = sp.ni;
    }
    if (which == 0) {
        xi_dst_ = d;
        xi_src_ = s0;
        xi_pitch_ = pitch;
        xi_w_.assign(12 * n, 0.0);
        for (size_t k = 0; k < n; ++k)
            for (int a = 0; a < 6; ++a) {
                xi_w_[12 * k + a] = wx[6 * k + a];
                xi_w_[12 * k + 6 + a] = wy[6 * k + a];
            }
    } else {
        std::vector<size_t> order(n);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return d[a] < d[b]; });
        vi_off_.assign(npts_ + 1, 0);
        vi_src_.clear();
        vi_pitch_.clear();
        vi_w_.clear();
        for (size_t k : order) {
            vi_off_[d[k] + 1]++;
            vi_src_.push_back(s0[k]);
            vi_pitch_.push_back(pitch[k]);
            for (int a = 0; a < 6; ++a) vi_w_.push_back(wx[6 * k + a]);
            for (int a = 0; a < 6; ++a) vi_w_.push_back(wy[6 * k + a]);
            vi_w_.push_back(w[k]);
        }
        for (long p = 0; p < npts_; ++p) vi_off_[p + 1] += vi_off_[p];
    }
    have_plan_ = true;
}

void Engine::set_halo(std::vector<int> e_sub, std::vector<int> e_loc, long n_recv_e, std::vector<int> mu_sub,
                      std::vector<int> mu_loc, long n_recv_mu) {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    if (laid_out_) throw Error(kUsage, "set the halo before the plan");  // the layout orders edge subpatches first
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

void Engine::set_halo_interps(int which, std::vector<int> sub, std::vector<int> si0, std::vector<int> sj0,
                              std::vector<double> wx, std::vector<double> wy) {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    if (which != 0 && which != 1) throw Error(kUsage, "bad halo list");
    const size_t n = sub.size();
    if (si0.size() != n || sj0.size() != n || wx.size() != 6 * n || wy.size() != 6 * n)
        throw Error(kUsage, "interpolation arrays of inconsistent length");
    HaloInterps& h = hi_[which];
    h.sub = std::move(sub);
    h.si0 = std::move(si0);
    h.sj0 = std::move(sj0);
    h.w.assign(12 * n, 0.0);
    for (size_t k = 0; k < n; ++k)
        for (int a = 0; a < 6; ++a) {
            h.w[12 * k + a] = wx[6 * k + a];
            h.w[12 * k + 6 + a] = wy[6 * k + a];
        }
}

void Engine::pack_e(double* d_buf) {
    launch_pack(E_, 0, d_halo_e_, static_cast<long>(halo_e_.size()), hp_[0], d_buf, ctx_.stream);
}
void Engine::unpack_e(const double* d_buf) { launch_unpack(E_, 0, n_recv_e_, d_buf, ctx_.stream); }
void Engine::pack_mu(double* d_buf) {
    launch_pack(E_, 1, d_halo_mu_, static_cast<long>(halo_mu_.size()), hp_[1], d_buf, ctx_.stream);
}
void Engine::unpack_mu(const double* d_buf) { launch_unpack(E_, 1, n_recv_mu_, d_buf, ctx_.stream); }

void Engine::attach_comm(std::unique_ptr<Comm> comm, std::vector<int> peers, std::vector<long> e_send,
                         std::vector<long> e_recv, std::vector<long> mu_send, std::vector<long> mu_recv) {
    if (!finalized_) throw Error(kUsage, "attach the transport after finalize");
    if (comm_) throw Error(kUsage, "transport already attached");
    const size_t np = peers.size();
    if (e_send.size() != np || e_recv.size() != np || mu_send.size() != np || mu_recv.size() != np)
        throw Error(kUsage, "per-peer count lists must match the peer list");
    for (size_t k = 0; k < np; ++k) {
        // (a rank may list itself: NCCL sends to self, which the self-exchange
        // GPU test uses to drive the transport on one device)
        if (peers[k] < 0 || peers[k] >= comm->size() || (k && peers[k] <= peers[k - 1]))
            throw Error(kUsage, "peers must be distinct ranks in ascending order");
        if (e_send[k] < 0 || e_recv[k] < 0 || mu_send[k] < 0 || mu_recv[k] < 0) throw Error(kUsage, "negative count");
    }
    const long want[4] = {static_cast<long>(halo_e_.size()), n_recv_e_, static_cast<long>(halo_mu_.size()),
                          n_recv_mu_};
    std::vector<long>* cnt[4] = {&e_send, &e_recv, &mu_send, &mu_recv};
    for (int w = 0; w < 4; ++w) {
        long sum = 0;
        for (long c : *cnt[w]) sum += c;
        if (sum != want[w]) throw Error(kUsage, "per-peer counts do not add up to the halo sizes");
        wire_cnt_[w] = *cnt[w];
        const long vals = (w < 2 ? 4 : 1) * std::max(sum, 1L);
        d_wire_[w] = dev::alloc_n<double>(vals);
        allocs_.push_back(d_wire_[w]);
    }
    peers_ = std::move(peers);
    comm_ = std::move(comm);
    if (graph_exec_) {  // a captured step without the transport
        dev::graph_destroy(graph_exec_, graph_);
        graph_exec_ = nullptr;
        graph_ = nullptr;
    }
}

// One halo of the multi-rank step, enqueued on `stream` (no host sync):
// pack the donor values this rank owes its peers (6x6 interpolations whose
// stencil lives here evaluated while packing), one grouped send / recv to the
// neighbour ranks, unpack into the halo slots the plan addresses with
// src_sub = -1. Buffers are per-peer slices in ascending peer order, the
// order both sides' plan split walked (distributed.split_plan).
void Engine::halo(int which, void* stream) {
    if (!comm_) return;
    const Range range(which == 0 ? "fcsg halo e" : "fcsg halo mu_hat");
    const int width = which == 0 ? 4 : 1;
    double* snd = d_wire_[which == 0 ? 0 : 2];
    double* rcv = d_wire_[which == 0 ? 1 : 3];
    const std::vector<long>& cs = wire_cnt_[which == 0 ? 0 : 2];
    const std::vector<long>& cr = wire_cnt_[which == 0 ? 1 : 3];
    if (which == 0) launch_pack(E_, 0, d_halo_e_, static_cast<long>(halo_e_.size()), hp_[0], snd, stream);
    else launch_pack(E_, 1, d_halo_mu_, static_cast<long>(halo_mu_.size()), hp_[1], snd, stream);
    comm_->group_start();
    long os = 0, orv = 0;
    for (size_t k = 0; k < peers_.size(); ++k) {
        if (cs[k]) comm_->send(snd + width * os, static_cast<size_t>(width * cs[k]), peers_[k]);
        if (cr[k]) comm_->recv(rcv + width * orv, static_cast<size_t>(width * cr[k]), peers_[k]);
        os += cs[k];
        orv += cr[k];
    }
    comm_->group_end(stream);
    launch_unpack(E_, which, which == 0 ? n_recv_e_ : n_recv_mu_, rcv, stream);
}

void Engine::reduce_dtmin(void* stream) {
    if (comm_) comm_->allreduce_min_u64(&E_.sc->dtmin_bits, stream);
}

void Engine::enqueue_part(int part, int stage) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    void* s = ctx_.stream;
    switch (part) {
        case -1: launch_bc(G_, s); break;
        case 0: launch_phase0(E_, G_, host_step_ == 0, s); break;
        case 1: launch_phase1(E_, s); break;
        case 2:
            launch_phase2(G_, host_step_ == 0, s);
            launch_bc(G_, s);
            launch_finalize_dt(E_, s);
            break;
        case 3:
            if (stage < 0 || stage > 4) throw Error(kUsage, "bad stage");
            launch_stage(G_, stage, s);
            launch_bc(G_, s);
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
        E_.cls_fast_margin = mlp_fast_margin(mlp_);
        E_.cls_margin32 = mlp_f32_margin(mlp_);
        *mlp32_ = mlp_f32_weights(mlp_);
        for (auto& g : G_) {
            g.E.cls_fast_margin = E_.cls_fast_margin;
            g.E.cls_margin32 = E_.cls_margin32;
        }
        for (auto& cv : chunks_)
            for (auto& c : cv) {
                c.E.cls_fast_margin = E_.cls_fast_margin;
                c.E.cls_margin32 = E_.cls_margin32;
            }
        if (graph_exec_) {  // the captured launches hold the old margin by value
            dev::graph_destroy(graph_exec_, graph_);
            graph_exec_ = nullptr;
            graph_ = nullptr;
        }
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

// Donor purity of the uploaded solution-exchange plan, the property the
// reference's phase 6 relies on (src/runtime.cpp:140-144,239-247: copies from
// the deepest-window interior donor, interpolation stencils entirely
// interior; the barriers at :482-512 order stage updates before the reads):
// every recipient is a fringe point (mask 2) and every donor point -- each
// copy source, each point of each 6x6 stencil -- an interior point (mask 1).
// exchange_kernel has no barrier between its reads and writes; with pure
// donors no point it writes is read by it. Donors on other ranks (halo slots)
// are checked by their own rank's plan.
void Engine::check_donor_purity(const std::vector<uint8_t>& mask) const {
    auto bad = [&](const char* what, long p) {
        const int slot = static_cast<int>(std::upper_bound(off_of_slot_.begin(), off_of_slot_.end(), p) -
                                          off_of_slot_.begin()) - 1;
        const auto& sp = subs_[id_of_slot_[slot]];
        const long loc = p - off_of_slot_[slot];
        throw Error(kDecomposition, std::string("exchange plan is not donor-pure: ") + what + " at subpatch " +
                                        std::to_string(id_of_slot_[slot]) + " (i=" + std::to_string(loc % sp.ni) +
                                        ", j=" + std::to_string(loc / sp.ni) + ")");
    };
    for (size_t k = 0; k < x_dst_.size(); ++k) {
        if (mask[x_dst_[k]] != 2) bad("copy recipient is not a fringe point", x_dst_[k]);
        if (x_src_[k] < npts_ && mask[x_src_[k]] != 1) bad("copy donor is not an interior point", x_src_[k]);
    }
    for (size_t k = 0; k < xi_dst_.size(); ++k) {
        if (mask[xi_dst_[k]] != 2) bad("interpolation recipient is not a fringe point", xi_dst_[k]);
        for (int b = 0; b < 6; ++b)
            for (int a = 0; a < 6; ++a) {
                const long p = xi_src_[k] + static_cast<long>(b) * xi_pitch_[k] + a;
                if (mask[p] != 1) bad("interpolation stencil point is not an interior point", p);
            }
    }
}

void Engine::finalize() {
    if (finalized_) throw Error(kUsage, "engine already finalized");
    if (subs_.empty()) throw Error(kUsage, "engine has no subpatches");
    // Classifier ctor (src/viscosity.cpp:134-141)
    if (cfg_.classifier == 0 && mlp_.empty()) throw Error(kConfig, "ann classifier requires a weight file path");
    layout();
    const int S = static_cast<int>(subs_.size());

    auto up = [&](const void* h, size_t bytes) {
        void* d = dev::alloc(bytes > 0 ? bytes : 8);
        allocs_.push_back(d);
        if (bytes) dev::h2d(d, h, bytes, ctx_.stream);
        return d;
    };
    EngineDev& E = E_;
    E.S = S;
    E.ni = 0;
    E.nj = 0;
    E.sub_base = 0;
    E.npts = npts_;
    E.cfl = cfg_.cfl;
    E.T = cfg_.T;
    for (int k = 0; k < 4; ++k) E.visc_c[k] = cfg_.visc_c[k];
    E.abs_floor = cfg_.abs_floor;
    E.smear_radius = cfg_.smear_radius;
    E.reference_order = cfg_.reference_order ? 1 : 0;
    E.cartesian = 0;

    // per-slot tables in storage order; BC tables per line (rows then columns
    // of each slot)
    std::vector<double> h1(S), h2(S);
    std::vector<int> ci(S), cj(S);
    std::vector<BcDev> rlo, rhi, clo, chi;
    std::vector<long> row_off(S), col_off(S);
    std::vector<uint8_t> mask(npts_);
    std::vector<double> geo[7];
    for (int k = 0; k < 7; ++k) geo[k].resize(npts_);
    for (int slot = 0; slot < S; ++slot) {
        const auto& sp = subs_[id_of_slot_[slot]];
        h1[slot] = sp.h1;
        h2[slot] = sp.h2;
        ci[slot] = sp.cut_i;
        cj[slot] = sp.cut_j;
        auto pad = [](const std::vector<BcDev>& v, size_t n) {
            std::vector<BcDev> o = v;
            BcDev none{};
            none.kind = -1;
            o.resize(n, none);
            return o;
        };
        row_off[slot] = static_cast<long>(rlo.size());
        col_off[slot] = static_cast<long>(clo.size());
        auto ra = pad(sp.row_lo, sp.nj), rb = pad(sp.row_hi, sp.nj), ca = pad(sp.col_lo, sp.ni), cb = pad(sp.col_hi, sp.ni);
        rlo.insert(rlo.end(), ra.begin(), ra.end());
        rhi.insert(rhi.end(), rb.begin(), rb.end());
        clo.insert(clo.end(), ca.begin(), ca.end());
        chi.insert(chi.end(), cb.begin(), cb.end());
        const long off = off_of_slot_[slot];
        std::copy(sp.mask.begin(), sp.mask.end(), mask.begin() + off);
        const std::vector<double>* src[7] = {&sp.iq1x, &sp.iq2x, &sp.iq1y, &sp.iq2y, &sp.h_min, &sp.h_max, &sp.w_norm};
        for (int k = 0; k < 7; ++k) std::copy(src[k]->begin(), src[k]->end(), geo[k].begin() + off);
    }
    // per-slot uniform metric (affine axis-aligned subpatches: iq1x and iq2y
    // are one value over the whole point set): the Cartesian passes then read
    // it per subpatch instead of staging it per point
    std::vector<double> q1c(S, 0.0), q2c(S, 0.0);
    std::vector<char> quni(S, 0);
    for (int slot = 0; slot < S; ++slot) {
        const auto& sp = subs_[id_of_slot_[slot]];
        if (sp.cut_i > 0 || sp.iq1x.empty()) continue;
        const double a = sp.iq1x[0], b = sp.iq2y[0];
        bool u = true;
        for (size_t q = 0; q < sp.iq1x.size() && u; ++q) u = sp.iq1x[q] == a && sp.iq2y[q] == b;
        quni[slot] = u;
        q1c[slot] = a;
        q2c[slot] = b;
    }
    E.iq1x_c = static_cast<const double*>(up(q1c.data(), S * sizeof(double)));
    E.iq2y_c = static_cast<const double*>(up(q2c.data(), S * sizeof(double)));
    E.h1 = static_cast<const double*>(up(h1.data(), S * sizeof(double)));
    E.h2 = static_cast<const double*>(up(h2.data(), S * sizeof(double)));
    E.cut_i = static_cast<const int*>(up(ci.data(), S * sizeof(int)));
    E.cut_j = static_cast<const int*>(up(cj.data(), S * sizeof(int)));
    E.bc_row_lo = static_cast<const BcDev*>(up(rlo.data(), rlo.size() * sizeof(BcDev)));
    E.bc_row_hi = static_cast<const BcDev*>(up(rhi.data(), rhi.size() * sizeof(BcDev)));
    E.bc_col_lo = static_cast<const BcDev*>(up(clo.data(), clo.size() * sizeof(BcDev)));
    E.bc_col_hi = static_cast<const BcDev*>(up(chi.data(), chi.size() * sizeof(BcDev)));
    E.mask = static_cast<const uint8_t*>(up(mask.data(), mask.size()));
    check_donor_purity(mask);
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
    // the FP32-screened classifier's fixup lists (one counter per shape group)
    E.cls_fix_list = dev::alloc_n<int>(static_cast<size_t>(std::max(npts_, 1L)));
    E.cls_fix_count = dev::alloc_n<unsigned>(std::max<size_t>(groups_.size(), 1));
    allocs_.push_back(E.cls_fix_list);
    allocs_.push_back(E.cls_fix_count);
    // tau is 0 until the first phase 0 (a zero-filled Field, as in the
    // reference; Classifier::classify then writes every point)
    {
        std::vector<double> one(npts_, 1.0);
        dev::memset0(E.tau, npts_ * sizeof(double), ctx_.stream);
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
        if (!xi_dst_.empty()) {
            E.xi_dst = static_cast<const long*>(up(xi_dst_.data(), xi_dst_.size() * sizeof(long)));
            E.xi_src = static_cast<const long*>(up(xi_src_.data(), xi_src_.size() * sizeof(long)));
            E.xi_pitch = static_cast<const int*>(up(xi_pitch_.data(), xi_pitch_.size() * sizeof(int)));
            E.xi_w = static_cast<const double*>(up(xi_w_.data(), xi_w_.size() * sizeof(double)));
        }
        E.n_xi = static_cast<long>(xi_dst_.size());
        if (!vi_src_.empty()) {
            E.vi_off = static_cast<const int*>(up(vi_off_.data(), vi_off_.size() * sizeof(int)));
            E.vi_src = static_cast<const long*>(up(vi_src_.data(), vi_src_.size() * sizeof(long)));
            E.vi_pitch = static_cast<const int*>(up(vi_pitch_.data(), vi_pitch_.size() * sizeof(int)));
            E.vi_w = static_cast<const double*>(up(vi_w_.data(), vi_w_.size() * sizeof(double)));
        }
    }
    if (static_cast<int>(mlp_.size()) != kMlpWeights) mlp_.assign(kMlpWeights, 0.0);  // fallback: unused
    E.mlp = static_cast<const double*>(up(mlp_.data(), mlp_.size() * sizeof(double)));
    {
        const std::vector<double> fr = mlp_mma_fragments(mlp_);
        E.mlp_frag = static_cast<const double*>(up(fr.data(), fr.size() * sizeof(double)));
        E.cls_fast_margin = mlp_fast_margin(mlp_);
        E.cls_margin32 = mlp_f32_margin(mlp_);
        mlp32_ = std::make_unique<MlpF32>(mlp_f32_weights(mlp_));
    }
    {
        std::vector<double> tt(kTanhTable);
        for (int k = 0; k < kTanhTable; ++k) tt[k] = static_cast<double>(tanhl(static_cast<long double>(k) / 64.0L));
        E.tanh_tab = static_cast<const double*>(up(tt.data(), tt.size() * sizeof(double)));
    }
    if (cfg_.classifier != 0 && cfg_.classifier != 1) throw Error(kConfig, "unknown classifier variant");
    if (cfg_.classifier == 1 && cfg_.classifier_window > kFbMaxWindow)
        throw Error(kConfig, "fallback classifier window > 64 is not supported");
    E.cls_variant = cfg_.classifier;
    E.fb_window = cfg_.classifier_window;
    E.fb_ncont = 25;  // OperatorCache::get(w) (src/fc_core.cpp:404-406)
    if (cfg_.classifier == 1) {
        // one table per window length the lines can produce: w = min(window, n), n >= 12
        std::vector<int> off(kFbMaxWindow + 1, -1);
        std::vector<double> tab;
        for (int w = kFbMinWindow; w <= cfg_.classifier_window; ++w) {
            const SpectrumTail t = build_spectrum_tail(w, E.fb_ncont);
            off[w] = static_cast<int>(tab.size());
            tab.insert(tab.end(), t.table.begin(), t.table.end());
        }
        E.fb_off = static_cast<const int*>(up(off.data(), off.size() * sizeof(int)));
        E.fb_tab = static_cast<const double*>(up(tab.data(), tab.size() * sizeof(double)));
    }
    halo_e_.clear();
    halo_mu_.clear();
    // send lists: points, or (loc = -1 - m) interpolation m of hi_[which]
    for (int which = 0; which < 2; ++which) {
        const HaloInterps& h = hi_[which];
        std::vector<long> src(h.sub.size());
        std::vector<int> pitch(h.sub.size());
        for (size_t m = 0; m < h.sub.size(); ++m) {
            const int ss = h.sub[m];
            if (ss < 0 || ss >= S) throw Error(kUsage, "halo interpolation donor out of range");
            const auto& sp = subs_[ss];
            if (h.si0[m] < 0 || h.sj0[m] < 0 || h.si0[m] + 6 > sp.ni || h.sj0[m] + 6 > sp.nj)
                throw Error(kUsage, "interpolation stencil outside the donor subpatch");
            src[m] = gidx(ss, h.sj0[m] * sp.ni + h.si0[m]);
            pitch[m] = sp.ni;
        }
        if (!src.empty()) {
            hp_[which].src = static_cast<const long*>(up(src.data(), src.size() * sizeof(long)));
            hp_[which].pitch = static_cast<const int*>(up(pitch.data(), pitch.size() * sizeof(int)));
            hp_[which].w = static_cast<const double*>(up(h.w.data(), h.w.size() * sizeof(double)));
        }
        auto& lst = which == 0 ? halo_e_src_ : halo_mu_src_;
        auto& out = which == 0 ? halo_e_ : halo_mu_;
        for (auto [sb, lc] : lst) {
            if (lc < 0) {
                if (-1 - lc >= static_cast<int>(h.sub.size())) throw Error(kUsage, "halo interpolation index out of range");
                out.push_back(lc);
            } else {
                out.push_back(gidx(sb, lc));
            }
        }
    }
    if (!halo_e_.empty()) d_halo_e_ = static_cast<long*>(up(halo_e_.data(), halo_e_.size() * sizeof(long)));
    if (!halo_mu_.empty()) d_halo_mu_ = static_cast<long*>(up(halo_mu_.data(), halo_mu_.size() * sizeof(long)));
    StepScalars sc{};
    double inf = kInf;
    std::memcpy(&sc.dtmin_bits, &inf, 8);
    E.sc = static_cast<StepScalars*>(up(&sc, sizeof(sc)));

    // group views: every pointer offset to the group's first point / slot /
    // line; line sets per orientation and length
    G_.clear();
    chunks_.clear();
    chunk_edge_.clear();
    bool all_cart = true;
    // view of slots [g.slot0 + k0, g.slot0 + k0 + n) of group g
    auto make_view = [&](const Group& g, int k0, int n) {
        EngineDev V = E;
        const int slot0 = g.slot0 + k0;
        V.S = n;
        V.ni = g.ni;
        V.nj = g.nj;
        V.sub_base = slot0;
        V.npts = static_cast<long>(n) * g.ni * g.nj;
        V.div_ni = make_fastdiv(static_cast<unsigned>(g.ni));
        V.div_sz = make_fastdiv(static_cast<unsigned>(g.ni * g.nj));
        const long p0 = g.p0 + static_cast<long>(k0) * g.ni * g.nj;
        auto offp = [p0](auto* ptr) { return ptr ? ptr + p0 : ptr; };
        V.mask = offp(E.mask);
        V.iq1x = offp(E.iq1x);
        V.iq2x = offp(E.iq2x);
        V.iq1y = offp(E.iq1y);
        V.iq2y = offp(E.iq2y);
        V.h_min = offp(E.h_min);
        V.h_max = offp(E.h_max);
        V.w_norm = offp(E.w_norm);
        for (int c = 0; c < 4; ++c) {
            V.e[c] = offp(E.e[c]);
            V.e0[c] = offp(E.e0[c]);
            V.e2[c] = offp(E.e2[c]);
            V.e3[c] = offp(E.e3[c]);
            V.rhs3[c] = offp(E.rhs3[c]);
            V.rhs[c] = offp(E.rhs[c]);
            V.tA[c] = offp(E.tA[c]);
            V.tW[c] = offp(E.tW[c]);
            V.tS4[c] = offp(E.tS4[c]);
            V.tS5[c] = offp(E.tS5[c]);
            V.tF[c] = offp(E.tF[c]);
        }
        V.mu_hat = offp(E.mu_hat);
        V.mu = offp(E.mu);
        V.tau = offp(E.tau);
        V.speed = offp(E.speed);
        V.proxy = offp(E.proxy);
        V.seed = offp(E.seed);
        V.m01 = offp(E.m01);
        V.h1 = E.h1 + slot0;
        V.iq1x_c = E.iq1x_c + slot0;
        V.iq2y_c = E.iq2y_c + slot0;
        V.uniform_q = 1;
        for (int k = 0; k < n; ++k) V.uniform_q = V.uniform_q && quni[slot0 + k];
        V.h2 = E.h2 + slot0;
        V.cut_i = E.cut_i + slot0;
        V.cut_j = E.cut_j + slot0;
        V.bc_row_lo = E.bc_row_lo + row_off[slot0];
        V.bc_row_hi = E.bc_row_hi + row_off[slot0];
        V.bc_col_lo = E.bc_col_lo + col_off[slot0];
        V.bc_col_hi = E.bc_col_hi + col_off[slot0];
        // the global-view plan structures are not used through a group view
        V.visc_off = nullptr;
        V.vi_off = nullptr;
        V.n_x = 0;
        V.n_xi = 0;
        return V;
    };
    for (const Group& g : groups_) {
        GroupLaunch gl;
        EngineDev V = make_view(g, 0, g.n);
        // Cartesian group: iq2x == iq1y == 0 at every point
        V.cartesian = cfg_.allow_cartesian ? 1 : 0;
        for (int k = 0; k < g.n && V.cartesian; ++k) {
            const auto& sp = subs_[id_of_slot_[g.slot0 + k]];
            for (size_t q = 0; q < sp.iq2x.size(); ++q)
                if (sp.iq2x[q] != 0.0 || sp.iq1y[q] != 0.0) {
                    V.cartesian = 0;
                    break;
                }
        }
        all_cart = all_cart && V.cartesian;
        // line sets: lengths n of the group's rows / columns; descriptor runs
        // only when a subpatch of the group is L-shaped
        bool any_l = false;
        for (int k = 0; k < g.n; ++k) any_l = any_l || subs_[id_of_slot_[g.slot0 + k]].cut_i > 0;
        for (int orient = 0; orient < 2; ++orient) {
            const int nlines = orient == 0 ? g.nj : g.ni, nfull = orient == 0 ? g.ni : g.nj;
            std::vector<LineSet>& sets = orient == 0 ? gl.rows : gl.cols;
            auto make_set = [&](int n) {
                LineSet L{};
                const int op = ctx_.get_op(n, cfg_.n_cont, 2, cfg_.filter);
                L.pl = ctx_.op(op).plan;
                L.scr = step_scr_cap(L.pl);
                if (!line_pass_smem_fits(L.pl, L.scr))
                    throw Error(kConfig, "subpatch lines of " + std::to_string(n) +
                                             " points exceed the line passes' shared memory (227 KB per CTA)");
                return L;
            };
            if (!any_l) {
                sets.push_back(make_set(nfull));
                continue;
            }
            // runs of consecutive lines of one slot with one begin, per length
            std::vector<std::pair<int, std::vector<std::array<int, 3>>>> runs;  // n -> (sub, line, begin)
            for (int k = 0; k < g.n; ++k) {
                const auto& sp = subs_[id_of_slot_[g.slot0 + k]];
                for (int line = 0; line < nlines; ++line) {
                    const int begin = orient == 0 ? (line < sp.cut_j ? sp.cut_i : 0) : (line < sp.cut_i ? sp.cut_j : 0);
                    const int n = nfull - begin;
                    size_t r = 0;
                    while (r < runs.size() && runs[r].first != n) ++r;
                    if (r == runs.size()) runs.push_back({n, {}});
                    runs[r].second.push_back({k, line, begin});
                }
            }
            for (auto& [n, lines] : runs) {
                LineSet L = make_set(n);
                for (int li = 0; li < 3; ++li) {
                    const int lb = kDescLB[li];
                    std::vector<LineDesc> desc;
                    for (size_t q = 0; q < lines.size();) {
                        LineDesc d{lines[q][0], lines[q][1], 1, lines[q][2]};
                        size_t r = q + 1;
                        while (r < lines.size() && d.nl < lb && lines[r][0] == d.sub && lines[r][1] == d.line0 + d.nl &&
                               lines[r][2] == d.begin) {
                            ++d.nl;
                            ++r;
                        }
                        desc.push_back(d);
                        q = r;
                    }
                    L.desc[li] = static_cast<const LineDesc*>(up(desc.data(), desc.size() * sizeof(LineDesc)));
                    L.n[li] = static_cast<int>(desc.size());
                }
                sets.push_back(L);
            }
        }
        gl.E = V;
        gl.E.cls_fix_list = E.cls_fix_list + g.p0;
        gl.E.cls_fix_count = E.cls_fix_count + (&g - groups_.data());
        if (cfg_.classifier == 0) gl.w32 = mlp32_.get();
        // stage chunks: the group's slots in up to stage_chunks contiguous
        // runs (groups with explicit line runs stay whole)
        // (a chunk keeps >= kChunkPoints points: smaller kernels lose more to
        // launch gaps than they gain from the overlap)
        const long by_size = static_cast<long>(g.n) * g.ni * g.nj / kChunkPoints;
        std::vector<int> cuts;  // chunk boundaries in the group's slots
        if (!halo_e_src_.empty()) {
            // multi-rank: the edge run, then the interior run (L-shaped
            // groups, whose line runs are not split, stay whole)
            cuts = {0};
            if (!any_l && g.n_edge > 0 && g.n_edge < g.n) cuts.push_back(g.n_edge);
            cuts.push_back(g.n);
        } else {
            const int nch = any_l ? 1 : static_cast<int>(std::max(1L, std::min<long>({by_size, cfg_.stage_chunks, g.n})));
            for (int c = 0; c <= nch; ++c) cuts.push_back(static_cast<int>(static_cast<long>(g.n) * c / nch));
        }
        const int nch = static_cast<int>(cuts.size()) - 1;
        for (int c = 0; c < nch; ++c) {
            const int k0 = cuts[c], k1 = cuts[c + 1];
            GroupLaunch cl = gl;
            if (nch > 1) {
                cl.E = make_view(g, k0, k1 - k0);
                cl.E.cartesian = V.cartesian;
            }
            chunks_.push_back({cl});
            chunk_edge_.push_back(k0 < g.n_edge ? 1 : 0);
        }
        G_.push_back(std::move(gl));
    }
    E.cartesian = all_cart ? 1 : 0;
    // several shape groups run their stage passes side by side on the stream
    // pool: a persistent warp-pass grid that fills every SM would hold the
    // other groups' CTAs back until it ends (config 4: 4.47 -> 3.99 ms per
    // superstep with 3 of 4 CTAs per SM; config 3 unchanged; 2 costs config 3 7%)
    static const int cap_env = [] {  // A/B runs: FCSG_WPASS_CAP = CTAs per SM (0 = no cap)
        const char* v = std::getenv("FCSG_WPASS_CAP");
        return v ? std::atoi(v) : -1;
    }();
    const int cap = groups_.size() > 1 ? (cap_env >= 0 ? cap_env : kMultiGroupWpassCap) : 0;
    for (GroupLaunch& g : G_) g.E.wpass_cap = cap;
    for (auto& c : chunks_)
        for (GroupLaunch& g : c) g.E.wpass_cap = cap;
    finalized_ = true;
}

int Engine::launches_per_step() const {
    int n = fcsg::launches_per_step(G_);
    if (dev::is_cuda() && chunks_.size() > 1) {  // enqueue_step's chunked stages
        n -= 5 * (stage_launches(G_) + static_cast<int>(G_.size()));
        for (const auto& c : chunks_) n += 5 * (stage_launches(c) + 1);
    }
    if (comm_) {  // pack / unpack kernels of the halos (NCCL's own kernels not counted)
        n += (halo_mu_.empty() ? 0 : 1) + (n_recv_mu_ ? 1 : 0);
        n += 5 * ((halo_e_.empty() ? 0 : 1) + (n_recv_e_ ? 1 : 0));
    }
    return n;
}

bool Engine::cartesian() const {
    for (const GroupLaunch& g : G_)
        if (!g.E.cartesian) return false;
    return !G_.empty();
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
    if (w == "grad") {
        if (!E.diag) throw Error(kUsage, "grad: call fcsg_engine_gradient first");
        return E.diag;
    }
    throw Error(kUsage, "unknown field " + w);
}

void Engine::set_state(int sub, const double* e4) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (sub < 0 || sub >= static_cast<int>(subs_.size())) throw Error(kUsage, "bad subpatch id");
    const long sz = sub_points(sub), off = off_of_slot_[slot_of_[sub]];
    for (int c = 0; c < 4; ++c) dev::h2d(E_.e[c] + off, e4 + c * sz, sz * sizeof(double), ctx_.stream);
}

// host layout [4][sum of points]: per component the subpatches in id order,
// each [nj][ni]; one copy per component when the storage order is the id order
void Engine::set_state_bulk(const double* e) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    bool identity = true;
    for (size_t k = 0; k < slot_of_.size(); ++k) identity = identity && slot_of_[k] == static_cast<int>(k);
    for (int c = 0; c < 4; ++c) {
        if (identity) {
            dev::h2d_async(E_.e[c], e + c * npts_, npts_ * sizeof(double), ctx_.stream);
        } else {
            long src = 0;
            for (int id = 0; id < static_cast<int>(subs_.size()); ++id) {
                const long sz = sub_points(id);
                dev::h2d_async(E_.e[c] + off_of_slot_[slot_of_[id]], e + c * npts_ + src, sz * sizeof(double),
                               ctx_.stream);
                src += sz;
            }
        }
    }
    dev::sync(ctx_.stream);
}

void Engine::get_state_bulk(double* e) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    bool identity = true;
    for (size_t k = 0; k < slot_of_.size(); ++k) identity = identity && slot_of_[k] == static_cast<int>(k);
    for (int c = 0; c < 4; ++c) {
        if (identity) {
            dev::d2h_async(e + c * npts_, E_.e[c], npts_ * sizeof(double), ctx_.stream);
        } else {
            long dst = 0;
            for (int id = 0; id < static_cast<int>(subs_.size()); ++id) {
                const long sz = sub_points(id);
                dev::d2h_async(e + c * npts_ + dst, E_.e[c] + off_of_slot_[slot_of_[id]], sz * sizeof(double),
                               ctx_.stream);
                dst += sz;
            }
        }
    }
    dev::sync(ctx_.stream);
}

void Engine::get_field(int sub, const std::string& name, int comp, double* out) {
    if (sub < 0 || sub >= static_cast<int>(subs_.size())) throw Error(kUsage, "bad subpatch id");
    double* f = field_ptr(name, comp);
    dev::d2h(out, f + off_of_slot_[slot_of_[sub]], sub_points(sub) * sizeof(double), ctx_.stream);
}

void Engine::set_field(int sub, const std::string& name, int comp, const double* in) {
    if (sub < 0 || sub >= static_cast<int>(subs_.size())) throw Error(kUsage, "bad subpatch id");
    double* f = field_ptr(name, comp);
    dev::h2d(f + off_of_slot_[slot_of_[sub]], in, sub_points(sub) * sizeof(double), ctx_.stream);
}

void Engine::gradient(int comp) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (comp < 0 || comp > 3) throw Error(kUsage, "bad component");
    if (!E_.diag) {
        E_.diag = static_cast<double*>(dev::alloc(npts_ * sizeof(double)));
        allocs_.push_back(E_.diag);
        dev::memset0(E_.diag, npts_ * sizeof(double), ctx_.stream);
        // views: the same offset as their state pointers
        auto fix = [&](GroupLaunch& g) { g.E.diag = E_.diag + (g.E.e[0] - E_.e[0]); };
        for (auto& g : G_) fix(g);
        for (auto& c : chunks_)
            for (auto& g : c) fix(g);
    }
    launch_gradient(G_, comp, ctx_.stream);
    dev::check("gradient");
}

void Engine::set_quadrature(int sub, const double* wq) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (sub < 0 || sub >= static_cast<int>(subs_.size())) throw Error(kUsage, "bad subpatch id");
    if (!E_.wq) {
        double* w = static_cast<double*>(dev::alloc(npts_ * sizeof(double)));
        allocs_.push_back(w);
        dev::memset0(w, npts_ * sizeof(double), ctx_.stream);
        E_.wq = w;
        wq_set_.assign(subs_.size(), 0);
    }
    dev::h2d(const_cast<double*>(E_.wq) + off_of_slot_[slot_of_[sub]], wq, sub_points(sub) * sizeof(double),
             ctx_.stream);
    wq_set_[sub] = 1;
}

void Engine::integrals(int comp, double* per_sub) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (comp < -1 || comp > 3) throw Error(kUsage, "bad component");
    const int S = static_cast<int>(subs_.size());
    for (int k = 0; k < S; ++k)
        if (!E_.wq || !wq_set_[k]) throw Error(kUsage, "quadrature weights not set for every subpatch");
    if (!d_slot_off_) {
        std::vector<long> off(S + 1);
        for (int s = 0; s < S; ++s) off[s] = off_of_slot_[s];
        off[S] = npts_;
        d_slot_off_ = static_cast<long*>(dev::alloc(off.size() * sizeof(long)));
        allocs_.push_back(d_slot_off_);
        dev::h2d(d_slot_off_, off.data(), off.size() * sizeof(long), ctx_.stream);
        d_quad_out_ = static_cast<double*>(dev::alloc(S * sizeof(double)));
        allocs_.push_back(d_quad_out_);
    }
    launch_integrals(E_, comp, d_slot_off_, S, d_quad_out_, ctx_.stream);
    std::vector<double> by_slot(S);
    dev::d2h(by_slot.data(), d_quad_out_, S * sizeof(double), ctx_.stream);
    // total += acc * p.h1 * p.h2 per subpatch (src/workbench.cpp:207)
    for (int id = 0; id < S; ++id) per_sub[id] = by_slot[slot_of_[id]] * subs_[id].h1 * subs_[id].h2;
}

void Engine::sample(long n, const int* sub, const int* il, const int* jl, const double* fu, const double* fv,
                    double* out) {
    if (!E_.diag) throw Error(kUsage, "sample: call fcsg_engine_gradient first");
    std::vector<long> base(n);
    std::vector<int> pitch(n);
    for (long k = 0; k < n; ++k) {
        const int s = sub[k];
        if (s < 0) {
            base[k] = -1;
            pitch[k] = 0;
            continue;
        }
        if (s >= static_cast<int>(subs_.size())) throw Error(kUsage, "bad subpatch id");
        const SubSpec& d = subs_[s];
        if (il[k] < 0 || jl[k] < 0 || il[k] > d.ni - 2 || jl[k] > d.nj - 2) throw Error(kUsage, "sample outside subpatch");
        base[k] = off_of_slot_[slot_of_[s]] + static_cast<long>(jl[k]) * d.ni + il[k];
        pitch[k] = d.ni;
    }
    const size_t nb = static_cast<size_t>(n);
    long* db = static_cast<long*>(dev::alloc(nb * sizeof(long)));
    int* dp = static_cast<int*>(dev::alloc(nb * sizeof(int)));
    double* du = static_cast<double*>(dev::alloc(nb * sizeof(double)));
    double* dv = static_cast<double*>(dev::alloc(nb * sizeof(double)));
    double* dout = static_cast<double*>(dev::alloc(nb * sizeof(double)));
    dev::h2d(db, base.data(), nb * sizeof(long), ctx_.stream);
    dev::h2d(dp, pitch.data(), nb * sizeof(int), ctx_.stream);
    dev::h2d(du, fu, nb * sizeof(double), ctx_.stream);
    dev::h2d(dv, fv, nb * sizeof(double), ctx_.stream);
    launch_sample(E_.diag, n, db, dp, du, dv, dout, ctx_.stream);
    dev::d2h(out, dout, nb * sizeof(double), ctx_.stream);
    for (void* p : {static_cast<void*>(db), static_cast<void*>(dp), static_cast<void*>(du), static_cast<void*>(dv),
                    static_cast<void*>(dout)})
        dev::free(p);
}

void Engine::check_error() {
    StepScalars sc;
    dev::d2h(&sc, E_.sc, sizeof(sc), ctx_.stream);
    if (sc.err.code == 0) return;
    // clear so the engine can report the next failure
    StepScalars clr = sc;
    clr.err = DevError{0, 0, 0, 0, -1};
    dev::h2d(E_.sc, &clr, sizeof(clr), ctx_.stream);
    int slot = sc.err.sub, i = sc.err.i, j = sc.err.j;
    if (sc.err.gp >= 0) {  // global point index -> (slot, i, j)
        slot = static_cast<int>(std::upper_bound(off_of_slot_.begin(), off_of_slot_.end(), sc.err.gp) -
                                off_of_slot_.begin()) - 1;
        const long loc = sc.err.gp - off_of_slot_[slot];
        const int ni = subs_[id_of_slot_[slot]].ni;
        i = static_cast<int>(loc % ni);
        j = static_cast<int>(loc / ni);
    }
    const int id = id_of_slot_.at(slot);
    const auto& sp = subs_.at(id);
    const char* msg = sc.err.code == 1   ? "nonpositive density or pressure"
                      : sc.err.code == 2 ? "nonpositive density or pressure (viscosity proxy)"
                                         : "nonfinite wave speed";
    throw StateError(msg, sp.patch, id, sp.i0 + i, sp.j0 + j, sc.t);
}

void Engine::finish_ic() {
    launch_bc(G_, ctx_.stream);
    halo(0, ctx_.stream);
    launch_exchange(E_, ctx_.stream);
    dev::check("finish_ic");
    dev::sync(ctx_.stream);
}

void Engine::phase(int ph, int stage) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    static const char* kPhaseRange[7] = {"fcsg phase 0", "fcsg phase 1", "fcsg phase 2", "fcsg phase 3", "", "",
                                         "fcsg phase 6"};
    const Range range(ph >= 0 && ph < 7 && kPhaseRange[ph][0] ? kPhaseRange[ph] : "fcsg phase");
    switch (ph) {
        case 0: launch_phase0(E_, G_, host_step_ == 0, ctx_.stream); break;
        case 1:
            halo(1, ctx_.stream);
            launch_phase1(E_, ctx_.stream);
            break;
        case 2:
            launch_phase2(G_, host_step_ == 0, ctx_.stream);
            launch_bc(G_, ctx_.stream);
            break;
        case 3:
            if (stage < 0 || stage > 4) throw Error(kUsage, "bad stage");
            launch_stage(G_, stage, ctx_.stream);
            launch_bc(G_, ctx_.stream);
            break;
        case 6:
            halo(0, ctx_.stream);
            launch_exchange(E_, ctx_.stream);
            break;
        default: throw Error(kUsage, "bad phase");
    }
    dev::check("phase");
    dev::sync(ctx_.stream);
    check_error();
}

double Engine::reduce_dt() {
    reduce_dtmin(ctx_.stream);
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

void Engine::ensure_streams() {
    if (!cstreams_.empty()) return;
    int ns = kStageStreams;
    if (const char* v = std::getenv("FCSG_STAGE_STREAMS")) ns = std::atoi(v);
    ns = std::max(2, ns);
    for (int k = 0; k < ns; ++k) {
        cstreams_.push_back(dev::create_stream());
        cevents_.push_back(dev::create_event());
    }
    ev_stage_ = dev::create_event();
}

void Engine::enqueue_step(bool step0) {
    const Range step_range(step0 ? "fcsg superstep (t=0)" : "fcsg superstep");
    range_push("fcsg phases 0-2 (classifier, blend, filter, BC, dt)");
    void* s = ctx_.stream;
    // phase 0 reads e only in the proxy (and, at t = 0, in the classifier's
    // density windows); the phase-2 filter writes e and touches nothing
    // phases 0-1 read or write, so in steady steps it runs on a side stream
    // next to the classifier and the blend
    const bool fork = !step0 && dev::is_cuda();
    if (fork && G_.size() > 1) {
        // several shape groups: each group's classifier and filter on its own
        // stream (classifiers on the first half of the pool, filters on the
        // second); the blend joins the classifiers, the BCs the filters
        ensure_streams();
        const int ns = static_cast<int>(cstreams_.size()), half = ns / 2;
        launch_proxy(E_, s);
        dev::record(ev_stage_, s);
        for (int k = 0; k < ns; ++k) dev::wait(cstreams_[k], ev_stage_);
        for (size_t g = 0; g < G_.size(); ++g) {
            const std::vector<GroupLaunch> one{G_[g]};
            launch_classify(E_, one, false, cstreams_[g % half]);
            launch_phase2(one, false, cstreams_[half + g % (ns - half)]);
        }
        for (int k = 0; k < ns; ++k) dev::record(cevents_[k], cstreams_[k]);
        for (int k = 0; k < half; ++k) dev::wait(s, cevents_[k]);
        halo(1, s);
        launch_phase1(E_, s);
        reduce_dtmin(s);
        for (int k = half; k < ns; ++k) dev::wait(s, cevents_[k]);
    } else {
        if (fork && !side_) {
            side_ = dev::create_stream();
            ev_fork_ = dev::create_event();
            ev_join_ = dev::create_event();
        }
        launch_proxy(E_, s);
        if (fork) {
            dev::record(ev_fork_, s);
            dev::wait(side_, ev_fork_);
            launch_phase2(G_, false, side_);
            dev::record(ev_join_, side_);
        }
        launch_classify(E_, G_, step0, s);
        halo(1, s);
        launch_phase1(E_, s);
        reduce_dtmin(s);
        if (fork) dev::wait(s, ev_join_);
        else launch_phase2(G_, step0, s);
    }
    launch_bc(G_, s);
    launch_finalize_dt(E_, s);
    range_pop();
    // RK stages: the chunks' line passes and BCs on side streams (a chunk's
    // passes and BCs touch only its own subpatches), joined before the
    // exchange. The GPU then runs one chunk's pass Y next to another's pass X
    // and fills each kernel's last wave with the next kernel's blocks.
    const bool chunked = dev::is_cuda() && chunks_.size() > 1;
    if (chunked) ensure_streams();
    bool edge_first = false;  // multi-rank with an edge / interior split
    for (size_t c = 0; c < chunk_edge_.size(); ++c) edge_first = edge_first || (comm_ && !chunk_edge_[c]);
    edge_first = edge_first && chunked;
    for (int st = 0; st < 5; ++st) {
        const Range stage_range(kStageRange[st]);
        if (edge_first) {
            // the edge runs' passes and BCs, then their halo (pack, grouped
            // ncclSend/Recv, unpack) on stream 0; the interior runs' passes on
            // the other streams meanwhile; the exchange after both
            const int ns = static_cast<int>(cstreams_.size());
            dev::record(ev_stage_, s);
            for (int k = 0; k < ns; ++k) dev::wait(cstreams_[k], ev_stage_);
            int next = 1;
            for (size_t c = 0; c < chunks_.size(); ++c) {
                void* cs = chunk_edge_[c] ? cstreams_[0] : cstreams_[1 + (next++ - 1) % (ns - 1)];
                launch_stage(chunks_[c], st, cs);
                launch_bc(chunks_[c], cs);
            }
            halo(0, cstreams_[0]);
            for (int k = 0; k < ns; ++k) {
                dev::record(cevents_[k], cstreams_[k]);
                dev::wait(s, cevents_[k]);
            }
            launch_exchange(E_, s);
            continue;
        }
        if (chunked) {
            const int ns = std::min(static_cast<int>(cstreams_.size()), static_cast<int>(chunks_.size()));
            dev::record(ev_stage_, s);
            for (int k = 0; k < ns; ++k) dev::wait(cstreams_[k], ev_stage_);
            for (size_t c = 0; c < chunks_.size(); ++c) {
                void* cs = cstreams_[c % ns];
                launch_stage(chunks_[c], st, cs);
                launch_bc(chunks_[c], cs);
            }
            for (int k = 0; k < ns; ++k) {
                dev::record(cevents_[k], cstreams_[k]);
                dev::wait(s, cevents_[k]);
            }
        } else {
            launch_stage(G_, st, s);
            launch_bc(G_, s);
        }
        halo(0, s);
        launch_exchange(E_, s);
    }
    launch_advance(E_, s);
}

void Engine::launch_group(int which) {
    void* s = ctx_.stream;
    switch (which) {
        case 0: launch_phase0(E_, G_, false, s); break;
        case 1: launch_phase1(E_, s); break;
        case 2: launch_phase2(G_, false, s); break;
        case 3: launch_pass_a(G_, s); break;
        case 4: launch_pass_b(G_, 1, s); break;
        case 5: launch_pass_c(G_, 1, s); break;
        case 6: launch_bc(G_, s); break;
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

// state <-> a bulk buffer ([4][sum of points], subpatches in id order) on the device
void Engine::bulk_d2d(double* bulk, const double* src, bool to_state, void* stream) {
    bool identity = true;
    for (size_t k = 0; k < slot_of_.size(); ++k) identity = identity && slot_of_[k] == static_cast<int>(k);
    for (int c = 0; c < 4; ++c) {
        if (identity) {
            if (to_state) dev::d2d(E_.e[c], src + c * npts_, npts_ * sizeof(double), stream);
            else dev::d2d(bulk + c * npts_, E_.e[c], npts_ * sizeof(double), stream);
            continue;
        }
        long pos = 0;
        for (int id = 0; id < static_cast<int>(subs_.size()); ++id) {
            const long sz = sub_points(id), off = off_of_slot_[slot_of_[id]];
            if (to_state) dev::d2d(E_.e[c] + off, src + c * npts_ + pos, sz * sizeof(double), stream);
            else dev::d2d(bulk + c * npts_ + pos, E_.e[c] + off, sz * sizeof(double), stream);
            pos += sz;
        }
    }
}

long Engine::run_host(long n, const double* in, long in_stride, double* out, long out_stride) {
    if (!finalized_) throw Error(kUsage, "engine not finalized");
    if (n <= 0) return 0;
    const bool finite_T = std::isfinite(cfg_.T);
    if (!dev::is_cuda() || finite_T) {  // one step at a time (and the T check)
        long done = 0;
        for (; done < n; ++done) {
            if (finite_T && time() >= cfg_.T - 1e-15) break;
            set_state_bulk(in + done * in_stride);
            run_steps(1, true);
            get_state_bulk(out + done * out_stride);
        }
        return done;
    }
    const size_t bytes = 4 * static_cast<size_t>(npts_) * sizeof(double);
    if (!cp_in_) {
        for (int b = 0; b < 2; ++b) {
            stage_in_[b] = static_cast<double*>(dev::alloc(bytes));
            stage_out_[b] = static_cast<double*>(dev::alloc(bytes));
            allocs_.push_back(stage_in_[b]);
            allocs_.push_back(stage_out_[b]);
            ev_in_ready_[b] = dev::create_event();
            ev_in_used_[b] = dev::create_event();
            ev_out_ready_[b] = dev::create_event();
            ev_out_done_[b] = dev::create_event();
        }
        cp_in_ = dev::create_stream();
        cp_out_ = dev::create_stream();
    }
    void* s = ctx_.stream;
    // nothing queued on s may still use the staging buffers
    dev::sync(s);
    for (int b = 0; b < 2; ++b) {
        dev::record(ev_in_used_[b], s);
        dev::record(ev_out_done_[b], s);
    }
    for (long k = 0; k < n; ++k) {
        const int b = static_cast<int>(k & 1);
        // upload: into the staging buffer step k-2 has finished reading
        dev::wait(cp_in_, ev_in_used_[b]);
        dev::h2d_async(stage_in_[b], in + k * in_stride, bytes, cp_in_);
        dev::record(ev_in_ready_[b], cp_in_);
        // the step: state <- staging, superstep, staging <- state
        dev::wait(s, ev_in_ready_[b]);
        bulk_d2d(nullptr, stage_in_[b], true, s);
        dev::record(ev_in_used_[b], s);
        enqueue_steps(1);
        dev::wait(s, ev_out_done_[b]);
        bulk_d2d(stage_out_[b], nullptr, false, s);
        dev::record(ev_out_ready_[b], s);
        // download on the other copy engine
        dev::wait(cp_out_, ev_out_ready_[b]);
        dev::d2h_async(out + k * out_stride, stage_out_[b], bytes, cp_out_);
        dev::record(ev_out_done_[b], cp_out_);
    }
    dev::sync(cp_in_);
    dev::sync(s);
    dev::sync(cp_out_);
    check_error();
    return n;
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
