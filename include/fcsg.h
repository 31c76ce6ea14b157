/*
 * fcsg -- B200-native FC-SDNN time step, C ABI.
 *
 * Plain C: pointers, sizes and int status codes; no exception crosses this
 * boundary and no torch or CUDA type appears in a signature (streams are
 * passed as void*). A context is bound to one CUDA device and is used from
 * one host thread. Every call returns FCSG_OK or one of the error kinds
 * below; fcsg_last_error() describes the last failure of that context. The
 * kinds map one-to-one onto the reference's exception types
 * (include/fcs/errors.hpp:10-43) so a C++ or Python wrapper can rethrow
 * ConfigError / UsageError / DecompositionError / InvalidStateError.
 *
 * Each entry point names the reference interface it replaces (paths relative
 * to the reference's proj/ directory).
 */
#ifndef FCSG_H
#define FCSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    FCSG_OK = 0,
    FCSG_CONFIG = 1,          /* fcs::ConfigError        */
    FCSG_USAGE = 2,           /* fcs::UsageError         */
    FCSG_GEOMETRY = 3,        /* fcs::GeometryError      */
    FCSG_DECOMPOSITION = 4,   /* fcs::DecompositionError */
    FCSG_INVALID_STATE = 5,   /* fcs::InvalidStateError  */
    FCSG_CUDA_ERROR = 8,
    FCSG_OTHER = 9
};

/* line-operator modes: FcOperator::derivative(order 1|2), filter, strong_filter */
enum { FCSG_D1 = 1, FCSG_D2 = 2, FCSG_FILTER = 3, FCSG_SMEAR = 4 };

typedef struct fcsg_ctx fcsg_ctx;

/* ---- context ----------------------------------------------------------- */
int fcsg_create(int device, fcsg_ctx** out);
int fcsg_destroy(fcsg_ctx* ctx);
/* Last error of this context. i/j are global lattice indices, as
 * InvalidStateError{patch, subpatch, i, j, t} (include/fcs/errors.hpp:32-39). */
int fcsg_last_error(fcsg_ctx* ctx, char* msg, int msg_len, int* kind, int* patch, int* subpatch,
                    int* i, int* j, double* t);
/* 1 if this build runs on a CUDA device, 0 for the CPU emulation harness. */
int fcsg_is_cuda_build(void);
int fcsg_synchronize(fcsg_ctx* ctx);

/* device memory helpers for callers that do not own an allocator */
int fcsg_device_alloc(fcsg_ctx* ctx, size_t bytes, void** ptr);
int fcsg_device_free(fcsg_ctx* ctx, void* ptr);
int fcsg_memcpy_h2d(fcsg_ctx* ctx, void* dst, const void* src, size_t bytes);
int fcsg_memcpy_d2h(fcsg_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ---- FC operator --------------------------------------------------------
 * Replaces fcs::fc::OperatorCache::get(n_points, n_cont, FilterSpec)
 * (include/fcs/fc_core.hpp:96-105, src/fc_core.cpp:391-402) and the
 * FcOperator constructor (src/fc_core.cpp:190-217). degree = 2 is the
 * reference operator (FcOperator::degree, include/fcs/fc_core.hpp:35); other
 * degrees are the generalised Gram basis. Same key -> same op_id.
 * Errors: FCSG_CONFIG for n_points < 10, n_cont < 4, a failed blend fit. */
int fcsg_operator(fcsg_ctx* ctx, int n_points, int n_cont, int degree, double alpha, int p,
                  int p_smear, int* op_id);
/* Sizes and tables of an operator: FcOperator::n_ext/n_modes/period/
 * filter_profile/smear_profile/blend_matrix (include/fcs/fc_core.hpp:42-74).
 * Output arrays may be NULL; blend is (n_cont-1) x (degree+1) row-major,
 * profiles have n_modes entries. */
int fcsg_operator_info(fcsg_ctx* ctx, int op_id, int* n_ext, int* n_modes, double* period,
                       double* blend, double* filter_profile, double* smear_profile);

/* Batched line operator on DEVICE buffers. Line l, element i is read at
 * in[l*in_line_stride + i*in_stride] and written, times `scale`, at
 * out[l*out_line_stride + i*out_stride]; in == out is allowed when the two
 * layouts coincide. Replaces a loop of FcOperator::derivative(in, in_stride,
 * out, out_stride, order) / filter / strong_filter (src/fc_core.cpp:257-306)
 * and, with scale = inv_len, SubpatchData::deriv_q1/deriv_q2
 * (src/subpatch_data.cpp:9-28). Errors: FCSG_USAGE for a bad mode (the
 * reference's "order must be 1 or 2"). `stream` is a cudaStream_t; NULL is the
 * default (legacy) stream, so torch's default stream orders correctly. */
int fcsg_fc_lines(fcsg_ctx* ctx, int op_id, int mode, const double* d_in, long in_line_stride,
                  long in_stride, double* d_out, long out_line_stride, long out_stride, long n_lines,
                  double scale, void* stream);
/* Same on HOST buffers (copies in and out, synchronous). */
int fcsg_fc_lines_host(fcsg_ctx* ctx, int op_id, int mode, const double* h_in, long in_line_stride,
                       long in_stride, double* h_out, long out_line_stride, long out_stride,
                       long n_lines, double scale);

/* ---- Engine (the FC-SDNN superstep) ---------------------------------------
 * Replaces fcs::run::Engine's step loop (include/fcs/runtime.hpp:79-127,
 * src/runtime.cpp:316-530) for subpatches whose init-time data
 * (SubpatchData geometry/masks/metrics/line BCs, init_subpatch_data,
 * src/subpatch_data.cpp:69-154; CommPlan, build_plan, src/runtime.cpp:89-274)
 * is built by the caller and uploaded once. Subpatches may have different
 * shapes (ni x nj, with an L-cut for corner patches); the engine stores them
 * grouped by shape and runs each group's line passes on its own plans. */
typedef struct fcsg_engine fcsg_engine;

/* EngineConfig (include/fcs/runtime.hpp:59-73) fields used by the step */
typedef struct {
    double cfl;
    double T;
    int n_cont;              /* 25 */
    double filter_alpha;     /* FilterSpec (include/fcs/fc_core.hpp:11-15) */
    int filter_p;
    int filter_p_smear;
    double visc_c[4];        /* ViscosityWeights {1.5, 1, 0.25, 0} */
    double abs_floor;        /* ClassifierConfig::abs_floor, 1e-4 */
    int smear_radius;        /* 10 */
    int debug_rhs;           /* keep the last stage's rhs readable (parity hooks) */
    int force_general;       /* 1: never use the Cartesian (zero metric term) passes */
    int reference_order;     /* 1: accumulate the rhs in euler_rhs's order (40 line derivatives);
                                0: flux form div(mu grad w - f), 24 */
    int classifier;          /* ClassifierConfig::variant (include/fcs/viscosity.hpp:45-52):
                                0 ann (the MLP; fcsg_engine_load_mlp before finalize),
                                1 fallback (FC-spectrum decay, src/viscosity.cpp:161-208) */
    int classifier_window;   /* ClassifierConfig::window of the fallback variant, 32 (<= 64) */
} fcsg_engine_config;

/* BcKind codes (include/fcs/bc.hpp:10-17); -1 = no boundary condition */
enum {
    FCSG_BC_NONE = -1,
    FCSG_BC_INFLOW = 0,
    FCSG_BC_OUTFLOW_PRESSURE = 1,
    FCSG_BC_SLIP_WALL = 2,
    FCSG_BC_NOSLIP_ADIABATIC = 3,
    FCSG_BC_SUPERSONIC_OUTFLOW = 4,
    FCSG_BC_ZERO_NORMAL_ALL = 5
};

int fcsg_engine_create(fcsg_ctx* ctx, const fcsg_engine_config* cfg, fcsg_engine** out);
int fcsg_engine_destroy(fcsg_engine* eng);

/* One SubpatchData (include/fcs/subpatch_data.hpp:15-63, built by
 * init_subpatch_data, src/subpatch_data.cpp:69-153): lattice origin (i0, j0)
 * of patch `patch` (for error reports), shape ni x nj (subpatches of any
 * shapes may be mixed), L-cut (geom::Subpatch::i_cut/j_cut - i0/j0: local
 * points with i < cut_i && j < cut_j are not in the set; 0, 0 = rectangle;
 * rows j < cut_j then begin at cut_i, columns i < cut_i at cut_j), parameter
 * spacings h1/h2 (LineInfo::inv_len = 1/((n-1) h)), per-point mask (0 outside
 * the set, 1 interior, 2 fringe), metrics iq1x, iq2x,
 * iq1y, iq2y, h_min, h_max, w_norm ([nj][ni] row-major), and the resolved
 * line-end BCs: bc_kind / bc_state[4] / bc_pressure for rows' low ends (nj),
 * rows' high ends (nj), columns' low ends (ni), columns' high ends (ni), in
 * that order. */
int fcsg_engine_add_subpatch(fcsg_engine* eng, int patch, int i0, int j0, int ni, int nj, int cut_i, int cut_j,
                             double h1, double h2, const uint8_t* mask, const double* iq1x, const double* iq2x, const double* iq1y,
                             const double* iq2y, const double* h_min, const double* h_max, const double* w_norm,
                             const int* bc_kind, const double* bc_state, const double* bc_pressure, int* sub_id);
/* CommPlan copies (include/fcs/runtime.hpp:17-22): solution copies
 * (recipient subpatch, local index) <- (donor subpatch, local index), and
 * viscosity-blend copies with weights, applied per recipient in the given
 * order. */
int fcsg_engine_set_plan(fcsg_engine* eng, long n_sol, const int* sol_dst_sub, const int* sol_dst,
                         const int* sol_src_sub, const int* sol_src, long n_visc, const int* v_dst_sub,
                         const int* v_dst, const int* v_src_sub, const int* v_src, const double* v_w);
/* CommPlan interpolations (InterpEntry, include/fcs/runtime.hpp:25-31): which
 * 0 = solution exchange (phase 6, src/runtime.cpp:440-452), 1 = viscosity
 * blend (phase 1, src/runtime.cpp:359-368, weights w). Entry k: recipient
 * (dst_sub[k], dst[k]) <- sum_b wy[6k+b] sum_a wx[6k+a] f(donor src_sub[k] at
 * (si0[k]+a, sj0[k]+b)); donors must be local subpatches, except that a
 * viscosity entry (which 1) with src_sub = -1 reads the value another rank
 * evaluated into halo slot si0[k] (fcsg_engine_set_halo_interps). Call after
 * the copies (fcsg_engine_set_plan). */
int fcsg_engine_set_plan_interps(fcsg_engine* eng, int which, long n, const int* dst_sub, const int* dst,
                                 const int* src_sub, const int* si0, const int* sj0, const double* wx, const double* wy,
                                 const double* w);
/* MlpClassifier::load (src/viscosity.cpp:63-89): FCNN v1 file, 7-16-16-16-16-4 tanh */
int fcsg_engine_load_mlp(fcsg_engine* eng, const char* path);
int fcsg_engine_finalize(fcsg_engine* eng);

/* state e = (rho, rho u, rho v, E), [4][nj][ni] (State, include/fcs/subpatch_data.hpp:15) */
int fcsg_engine_set_state(fcsg_engine* eng, int sub, const double* e4);
/* fields: "e","e0","e2","e3","rhs3","rhs" (comp 0..3), "mu_hat","mu","tau",
 * "speed","proxy","m01","iq1x","iq2x","iq1y","iq2y","h_min","h_max","w_norm",
 * "grad" (after fcsg_engine_gradient) */
int fcsg_engine_get_field(fcsg_engine* eng, int sub, const char* name, int comp, double* out);

/* Measurements on the device (src/workbench.cpp:187-294, replacing the
 * per-subpatch CPU loops of energy_integral / area_integral /
 * density_gradient_raster; the writers and the raster's point location stay
 * with the caller).
 * fcsg_engine_gradient: |grad e_comp| = hypot(iq1x d1 + iq2x d2, iq1y d1 + iq2y d2)
 *   with d1, d2 the FC derivatives along rows / columns (deriv_q1/q2), into
 *   the "grad" field.
 * fcsg_engine_set_quadrature: per-point weights of window_quadrature for one
 *   subpatch, [nj][ni]: w_norm |det J|, halved on the first/last point of
 *   each row segment and of each column segment, 0 outside the set.
 * fcsg_engine_integrals: per subpatch (id order) h1 h2 sum wq v, v = 1
 *   (comp = -1, area_integral) or e_comp (comp = 3: energy_integral); the
 *   caller adds them in id order.
 * fcsg_engine_sample: bilinear samples of "grad" at n points given as
 *   (subpatch id, local cell origin il, jl, fractions fu, fv) -- the raster
 *   pixel's containing subpatch as density_gradient_raster picks it; sub < 0
 *   gives 0. */
int fcsg_engine_gradient(fcsg_engine* eng, int comp);
int fcsg_engine_set_quadrature(fcsg_engine* eng, int sub, const double* wq);
int fcsg_engine_integrals(fcsg_engine* eng, int comp, double* per_sub);
int fcsg_engine_sample(fcsg_engine* eng, long n, const int* sub, const int* il, const int* jl, const double* fu,
                       const double* fv, double* out);
/* whole state of every subpatch in one call, component-major host layout
 * [4][S][nj][ni] (pinned host memory gives full PCIe/C2C bandwidth) */
int fcsg_engine_set_state_bulk(fcsg_engine* eng, const double* e);
int fcsg_engine_get_state_bulk(fcsg_engine* eng, double* e);
int fcsg_engine_set_field(fcsg_engine* eng, int sub, const char* name, int comp, const double* in);
/* apply_ic tail: enforce_bc on every subpatch, then one fringe exchange (src/runtime.cpp:284-286) */
int fcsg_engine_finish_ic(fcsg_engine* eng);
/* Engine::step_phase(phase, stage) for phase 0 (viscosity), 1 (blend),
 * 2 (filter/smear + E + BC), 3 (RHS + SSPRK stage + BC), 6 (exchange) */
int fcsg_engine_phase(fcsg_engine* eng, int phase, int stage);
/* dt = cfl min dt_local, clipped at T (src/runtime.cpp:492-497) */
int fcsg_engine_reduce_dt(fcsg_engine* eng, double* dt);
/* t += dt, step += 1 (src/runtime.cpp:505-507) */
int fcsg_engine_advance(fcsg_engine* eng);
/* n complete supersteps (Engine::run body, src/runtime.cpp:482-511); steady
 * steps replay one CUDA graph. Stops when t >= T - 1e-15. *done = steps run.
 * Errors: FCSG_INVALID_STATE with fcsg_last_error's patch/subpatch/i/j/t. */
int fcsg_engine_run(fcsg_engine* eng, long n, int use_graph, long* done);
/* n supersteps with host I/O every step (Engine::run plus the host-side state
 * exchange a driver does around it): step k reads its state from
 * in + k * in_stride and leaves its result in out + k * out_stride (doubles;
 * layout of fcsg_engine_set_state_bulk / get_state_bulk; stride 0 = the same
 * buffer every step). The copies run on two copy streams through device
 * staging buffers, so step k+1's upload and step k-1's download overlap step
 * k's kernels; use pinned host memory for that overlap. Returns when every
 * result is in host memory (errors as fcsg_engine_run). */
int fcsg_engine_run_host(fcsg_engine* eng, long n, const double* in, long in_stride, double* out, long out_stride,
                         long* done);
/* enqueue n supersteps on `stream`-ordered engine work without any host
 * synchronisation (benchmark path; errors surface at the next sync). */
int fcsg_engine_enqueue(fcsg_engine* eng, long n);
int fcsg_engine_time(fcsg_engine* eng, double* t, long* steps);
int fcsg_engine_total_points(fcsg_engine* eng, long* n);
/* 1 when every subpatch has iq2x == iq1y == 0 and the engine runs the
 * 12-transform Cartesian stage passes, 0 for the general 20-transform passes */
int fcsg_engine_is_cartesian(fcsg_engine* eng, int* yes);
/* the engine's CUDA stream (cudaStream_t), for event timing by the caller */
int fcsg_engine_stream(fcsg_engine* eng, void** stream);
/* ---- multi-rank (one process per GPU) -------------------------------------
 * The reference's workers read donor subpatches directly after a barrier
 * (src/runtime.cpp:436-452, 357-368). Across GPUs, each rank owns a block of
 * subpatches; donors on other ranks are packed into a contiguous device
 * buffer on the donor rank, moved by the caller's transport (NCCL send/recv
 * over NVLink, gloo in the CPU tests), and unpacked into halo slots on the
 * recipient, which its plan entries address with src_sub = -1. */
/* donor points this rank packs (state: [k][4], mu_hat: [k]) and the number
 * of values it receives; call before fcsg_engine_set_plan */
int fcsg_engine_set_halo(fcsg_engine* eng, long n_send_e, const int* e_sub, const int* e_loc, long n_recv_e,
                         long n_send_mu, const int* mu_sub, const int* mu_loc, long n_recv_mu);
/* Interpolated send entries (which 0 = state e, 1 = mu_hat): a send-list
 * entry with e_loc / mu_loc = -1 - m sends the 6x6 Lagrange interpolation m
 * of this list (donor subpatch, stencil origin si0 / sj0, wx[6 m..],
 * wy[6 m..]) evaluated on this rank (InterpEntry, include/fcs/runtime.hpp:
 * 25-31, whose donor lives here and whose recipient does not). Call after
 * fcsg_engine_set_halo. On the recipient the value lands in a halo slot: a
 * solution copy from that slot, or a viscosity interpolation entry with
 * src_sub = -1 and si0 = the slot (fcsg_engine_set_plan_interps, which 1). */
int fcsg_engine_set_halo_interps(fcsg_engine* eng, int which, long n, const int* sub, const int* si0, const int* sj0,
                                 const double* wx, const double* wy);
/* which: 0 = send e, 1 = recv e, 2 = send mu, 3 = recv mu */
int fcsg_engine_halo_size(fcsg_engine* eng, int which, long* n);
/* which: 0 = state e, 1 = mu_hat; d_buf is device memory on the engine's device */
int fcsg_engine_pack(fcsg_engine* eng, int which, void* d_buf);
int fcsg_engine_unpack(fcsg_engine* eng, int which, const void* d_buf);
/* one part of a superstep, enqueued on the engine stream: 0 viscosity
 * (phase 0), 1 blend + dt_local minimum (phase 1), 2 filter/smear + BC + dt
 * (phase 2 + dt), 3 stage `stage` (RHS + SSPRK + BC), 4 exchange copies
 * (phase 6), 5 advance. A multi-rank step: 0, mu halo, 1, all-reduce(min) of
 * the dt minimum, 2, then 5 x (3, state halo, 4), then 5. */
int fcsg_engine_enqueue_part(fcsg_engine* eng, int part, int stage);
/* device address of the dt minimum (a positive double stored as its
 * uint64 bit pattern, so an int64 MIN all-reduce is exact) */
int fcsg_engine_dtmin_ptr(fcsg_engine* eng, void** dptr);
/* 8-byte device copy of that minimum to (to_engine = 0) or from (1) a
 * caller buffer, ordered on the engine stream */
int fcsg_engine_copy_dtmin(fcsg_engine* eng, void* d_buf, int to_engine);
/* ---- device-ordered multi-rank transport ----------------------------------
 * Replaces the caller-driven parts above with the engine's own transport:
 * after fcsg_engine_attach_comm every superstep the engine enqueues
 * (fcsg_engine_finish_ic, _phase / _reduce_dt, _run, _enqueue, _run_host)
 * packs its halos, exchanges them with the neighbour ranks only (grouped
 * ncclSend / ncclRecv over NVLink) and all-reduces the dt minimum
 * (ncclAllReduce MIN on its bits) on the engine stream, with no host
 * synchronisation, so a steady multi-rank superstep is one CUDA graph.
 * Stands for the reference's barriers and cross-worker reads
 * (src/runtime.cpp:352-371, 433-454, 482-512).
 * fcsg_comm_unique_id: a rendezvous id (ncclUniqueId, 128 bytes) made on rank
 * 0 and broadcast by the caller. fcsg_engine_attach_comm (collective, after
 * finalize and the halo lists): peers = the ranks this one exchanges with,
 * ascending (itself allowed: a send to self); per peer the number of values (points) in the packed send
 * and receive buffers of the state and mu_hat halos, in that peer order (the
 * sums equal fcsg_engine_halo_size 0..3). */
int fcsg_comm_unique_id(char* id);
int fcsg_engine_attach_comm(fcsg_engine* eng, int nranks, int rank, const char* id, int n_peers, const int* peers,
                            const long* e_send, const long* e_recv, const long* mu_send, const long* mu_recv);
/* synchronise the engine stream and raise a pending device-side error */
int fcsg_engine_check_error(fcsg_engine* eng);

/* profiling hooks: average device ms of one launch group over `reps`
 * back-to-back launches (0 viscosity/classifier, 1 blend+dt, 2 filter,
 * 3 pass A, 4 pass B, 5 pass C, 6 BC, 7 exchange), and the number of kernel
 * launches one superstep issues */
int fcsg_engine_time_group(fcsg_engine* eng, int which, int reps, double* ms);
int fcsg_engine_launches_per_step(fcsg_engine* eng, int* n);

#ifdef __cplusplus
}
#endif

#endif
