// Host Engine: the drop-in for fcs::run::Engine's step loop
// (include/fcs/runtime.hpp:79-127, src/runtime.cpp:316-530) over device-
// resident subpatch data. Geometry, masks, metrics, windows and the exchange
// plan are built at init time by the caller (the reference's
// init_subpatch_data / build_plan equivalents) and uploaded once.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "comm.h"
#include "context.h"
#include "fc_tables.h"
#include "step_kernels.h"

namespace fcsg {

// InvalidStateError{patch, subpatch, i, j, t} (include/fcs/errors.hpp:32-39)
struct StateError : Error {
    int patch, sub, i, j;
    double t;
    StateError(const std::string& m, int patch_, int sub_, int i_, int j_, double t_)
        : Error(kInvalidState, m), patch(patch_), sub(sub_), i(i_), j(j_), t(t_) {}
};

// EngineConfig (include/fcs/runtime.hpp:59-73), the fields the step uses
struct EngineConfig {
    double cfl = 0.5;
    double T = 1.0;
    int n_cont = 25;
    FilterSpec filter;
    double visc_c[4] = {1.5, 1.0, 0.25, 0.0};  // ViscosityWeights (include/fcs/viscosity.hpp:72-74)
    double abs_floor = 1e-4;                   // ClassifierConfig::abs_floor
    int smear_radius = 10;
    bool debug_rhs = false;                    // keep the last stage's rhs for parity hooks
    bool allow_cartesian = true;               // use the zero-metric-term passes when they apply
    bool reference_order = false;              // euler_rhs's accumulation order instead of the flux form
    int classifier = 0;                        // ClassifierConfig::Variant: 0 ann (MLP), 1 fallback (FC spectrum)
    int classifier_window = 32;                // ClassifierConfig::window (fallback), 12..64
    int stage_chunks = 2;                      // RK-stage line passes of a large shape group in up to this many slot runs
};

struct SubSpec {
    int patch = 0, i0 = 0, j0 = 0;
    int ni = 0, nj = 0;
    int cut_i = 0, cut_j = 0;  // L-shaped: local points (i < cut_i && j < cut_j) are not in the set
    double h1 = 0, h2 = 0;
    std::vector<uint8_t> mask;
    std::vector<double> iq1x, iq2x, iq1y, iq2y, h_min, h_max, w_norm;
    std::vector<BcDev> row_lo, row_hi, col_lo, col_hi;
};

class Engine {
  public:
    Engine(Ctx& ctx, const EngineConfig& cfg);
    ~Engine();

    int add_subpatch(SubSpec s);
    // CommPlan (include/fcs/runtime.hpp:16-49) copies: solution copies
    // (dst_sub, dst, src_sub, src) and viscosity copies with weights.
    void set_plan(std::vector<int> sol_dst_sub, std::vector<int> sol_dst, std::vector<int> sol_src_sub,
                  std::vector<int> sol_src, std::vector<int> v_dst_sub, std::vector<int> v_dst,
                  std::vector<int> v_src_sub, std::vector<int> v_src, std::vector<double> v_w);
    // CommPlan interpolations (InterpEntry, include/fcs/runtime.hpp:25-31):
    // which 0 = solution, 1 = viscosity blend; donor stencil origin (si0, sj0)
    // in the donor subpatch, weights wx[6], wy[6] per entry (and w for the blend)
    void set_plan_interps(int which, std::vector<int> dst_sub, std::vector<int> dst, std::vector<int> src_sub,
                          std::vector<int> si0, std::vector<int> sj0, std::vector<double> wx, std::vector<double> wy,
                          std::vector<double> w);
    // Cross-rank halo (multi-GPU): donor points this rank packs for other
    // ranks (solution state and mu_hat), and how many values it receives.
    // Received values land in extra slots after the local points; plan
    // entries address them with src_sub = -1, src = slot. Call before
    // set_plan.
    void set_halo(std::vector<int> e_sub, std::vector<int> e_loc, long n_recv_e, std::vector<int> mu_sub,
                  std::vector<int> mu_loc, long n_recv_mu);
    // interpolated send entries: an entry of set_halo's lists with loc = -1 - m
    // sends the 6x6 Lagrange interpolation m of this list (donor sub, stencil
    // origin si0 / sj0, wx[6], wy[6]) instead of a point value; call after
    // set_halo (which 0 = state, 1 = mu_hat)
    void set_halo_interps(int which, std::vector<int> sub, std::vector<int> si0, std::vector<int> sj0,
                          std::vector<double> wx, std::vector<double> wy);
    void pack_e(double* d_buf);          // [k][4]
    void unpack_e(const double* d_buf);  // [k][4] -> extra slots
    void pack_mu(double* d_buf);
    void unpack_mu(const double* d_buf);
    long halo_size(int which) const;     // 0 send e, 1 recv e, 2 send mu, 3 recv mu
    // Device-ordered multi-rank transport (after finalize): the halos and the
    // dt minimum are then part of every superstep the engine enqueues
    // (finish_ic, phase / reduce_dt, enqueue_step, hence the CUDA graph).
    // peers in wire order (ascending rank) with the per-peer value counts of
    // the packed send / receive buffers (sums = the set_halo sizes).
    void attach_comm(std::unique_ptr<Comm> comm, std::vector<int> peers, std::vector<long> e_send,
                     std::vector<long> e_recv, std::vector<long> mu_send, std::vector<long> mu_recv);
    bool has_comm() const { return comm_ != nullptr; }
    // one part of a superstep (multi-rank driver): 0 viscosity, 1 blend + dt
    // minimum, 2 filter/smear + BC + dt, 3 stage `stage` (passes + BC),
    // 4 exchange copies, 5 advance
    void enqueue_part(int part, int stage);
    unsigned long long* dtmin_device_ptr() const { return &E_.sc->dtmin_bits; }
    void set_mlp_packed(const std::vector<double>& w);  // kMlpWeights, per layer W then b
    void load_mlp_file(const std::string& path);        // FCNN v1 (src/viscosity.cpp:63-89)
    void finalize();

    void set_state(int sub, const double* e4);
    // all subpatches at once, component-major host layout [4][S][nj][ni]
    void set_state_bulk(const double* e);
    void get_state_bulk(double* e);
    void get_field(int sub, const std::string& name, int comp, double* out);
    void set_field(int sub, const std::string& name, int comp, const double* in);

    void finish_ic();                  // enforce_bc + exchange (src/runtime.cpp:284-286)
    void phase(int ph, int stage);     // Engine::step_phase bodies 0,1,2,3,6
    double reduce_dt();                // worker-0 dt block (src/runtime.cpp:492-497)
    void advance();                    // t += dt, step++ (src/runtime.cpp:505-507)
    // n full supersteps; the steady-state step is replayed from a CUDA graph.
    // Stops early when t >= T - 1e-15 (checked every step only if T is finite).
    long run_steps(long n, bool use_graph);
    void enqueue_step(bool step0);
    // n supersteps enqueued without host synchronisation (graph replay after step 0)
    void enqueue_steps(long n);
    // n supersteps with host I/O per step: state <- in + k in_stride, one
    // superstep, out + k out_stride <- state (layouts as set/get_state_bulk).
    // Copies go through device staging buffers on two copy streams, so the
    // upload of step k+1's input and the download of step k-1's result
    // overlap step k's kernels; returns the steps done.
    long run_host(long n, const double* in, long in_stride, double* out, long out_stride);
    double time();
    long steps() const { return host_step_; }
    long total_points() const { return npts_; }
    // every shape group on the Cartesian (zero metric term) passes
    bool cartesian() const;
    int n_groups() const { return static_cast<int>(G_.size()); }
    void check_error();

    // diagnostics (src/workbench.cpp:187-239): |grad e_comp| into the "grad"
    // field; per-subpatch window quadrature h1 h2 sum wq value (value = 1 for
    // comp < 0, else e_comp) once every subpatch's weights are set; bilinear
    // samples of "grad" at raster pixels (sub < 0: outside -> 0)
    void gradient(int comp);
    void set_quadrature(int sub, const double* wq);
    void integrals(int comp, double* per_sub);
    void sample(long n, const int* sub, const int* il, const int* jl, const double* fu, const double* fv,
                double* out);
    // average device milliseconds of one launch group (profiling hook):
    // 0 phase 0 (proxy + classifier), 1 phase 1 (blend + dt), 2 phase 2
    // (filter rows + cols), 3 pass A, 4 pass B, 5 pass C (stage 1), 6 BC,
    // 7 exchange
    double time_pass(int which, int reps);
    int launches_per_step() const;
    void launch_group(int which);
    void* stream() const { return ctx_.stream; }

  private:
    double* field_ptr(const std::string& name, int comp);
    void layout();                          // storage order by shape group (after the last add_subpatch)
    long gidx(int sub, int loc) const;      // global point index of (subpatch id, local index)
    void check_donor_purity(const std::vector<uint8_t>& mask) const;
    long sub_points(int sub) const { return static_cast<long>(subs_.at(sub).ni) * subs_.at(sub).nj; }
    Ctx& ctx_;
    EngineConfig cfg_;
    std::vector<SubSpec> subs_;             // by subpatch id
    bool finalized_ = false, laid_out_ = false;
    long npts_ = 0;
    // storage: subpatches grouped by (ni, nj), ids in order within a group
    struct Group {
        int ni, nj, slot0, n;
        long p0;
        int n_edge;  // multi-rank: the first n_edge slots own donors other ranks read (edge-first order)
    };
    std::vector<Group> groups_;
    std::vector<int> slot_of_, id_of_slot_;
    std::vector<long> off_of_slot_;         // first point of each storage slot
    EngineDev E_{};                         // global view
    std::vector<GroupLaunch> G_;            // group views + line sets
    std::vector<std::vector<GroupLaunch>> chunks_;  // stage chunks (one view each)
    std::vector<char> chunk_edge_;                  // multi-rank: the chunk holds donors of the state halo
    std::vector<void*> allocs_;
    double* pool_ = nullptr;
    std::vector<double> mlp_;
    std::unique_ptr<MlpF32> mlp32_;         // FP32 copy for the classifier's screening pass (stable address)
    // plan (host staging until finalize)
    std::vector<long> x_dst_, x_src_;
    std::vector<int> visc_off_;
    std::vector<long> visc_src_;
    std::vector<double> visc_w_;
    std::vector<long> xi_dst_, xi_src_;
    std::vector<int> xi_pitch_;
    std::vector<double> xi_w_;
    std::vector<int> vi_off_;
    std::vector<long> vi_src_;
    std::vector<int> vi_pitch_;
    std::vector<double> vi_w_;
    bool have_plan_ = false;
    std::vector<long> halo_e_, halo_mu_;  // packed donor points (global local-engine indices)
    long n_recv_e_ = 0, n_recv_mu_ = 0;
    std::vector<std::pair<int, int>> halo_e_src_, halo_mu_src_;
    long* d_halo_e_ = nullptr;
    long* d_halo_mu_ = nullptr;
    // interpolated send entries per list: (sub, si0, sj0) and 12 weights
    struct HaloInterps {
        std::vector<int> sub, si0, sj0;
        std::vector<double> w;
    } hi_[2];
    HaloPackDev hp_[2]{};
    // attached transport: peers, per-peer counts (0 e send, 1 e recv, 2 mu
    // send, 3 mu recv) and the device wire buffers
    std::unique_ptr<Comm> comm_;
    std::vector<int> peers_;
    std::vector<long> wire_cnt_[4];
    double* d_wire_[4] = {nullptr, nullptr, nullptr, nullptr};
    void halo(int which, void* stream);  // pack -> grouped send / recv -> unpack (which 0 = e, 1 = mu_hat)
    void reduce_dtmin(void* stream);     // all-reduce(MIN) of the dt minimum's bits
    long host_step_ = 0;
    void* graph_exec_ = nullptr;
    void* graph_ = nullptr;
    // side stream of the steady step: the filter (phase 2 line passes) runs
    // next to the classifier and blend (phases 0-1), which neither read nor
    // write what it touches
    void* side_ = nullptr;
    void* ev_fork_ = nullptr;
    void* ev_join_ = nullptr;
    // streams of the RK-stage chunks (enqueue_step)
    static constexpr int kStageStreams = 8;
    static constexpr long kChunkPoints = 1L << 21;
    static constexpr int kMultiGroupWpassCap = 3;  // CTAs per SM of the persistent warp passes when several shape groups run side by side
    std::vector<void*> cstreams_, cevents_;
    void ensure_streams();
    std::vector<char> wq_set_;
    // run_host staging: two input and two output state buffers, copy streams
    double* stage_in_[2] = {nullptr, nullptr};
    double* stage_out_[2] = {nullptr, nullptr};
    void* cp_in_ = nullptr;
    void* cp_out_ = nullptr;
    void* ev_in_ready_[2] = {nullptr, nullptr};
    void* ev_in_used_[2] = {nullptr, nullptr};
    void* ev_out_ready_[2] = {nullptr, nullptr};
    void* ev_out_done_[2] = {nullptr, nullptr};
    void bulk_d2d(double* dst_state, const double* src_bulk, bool to_state, void* stream);
    long* d_slot_off_ = nullptr;
    double* d_quad_out_ = nullptr;
    void* ev_stage_ = nullptr;
};

}  // namespace fcsg
