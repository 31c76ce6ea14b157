// Device-side state of one engine and the kernel launchers of the FC-SDNN
// superstep (see step_kernels.cu for what each kernel restates).
#pragma once

#include <cstdint>
#include <vector>

#include "fcsg_common.h"

namespace fcsg {

constexpr int kMlpIn = 7;
constexpr int kMlpHidden = 16;
constexpr int kMlpOut = 4;
constexpr int kMlpLayers = 5;  // 7-16-16-16-16-4 (src/viscosity.cpp:366)
// packed: per layer W (rows x cols, row-major) then b (rows)
constexpr int kMlpWeights = (16 * 7 + 16) + 3 * (16 * 16 + 16) + (4 * 16 + 4);

// device scalars of the running step (one per engine)
struct StepScalars {
    unsigned long long dtmin_bits;  // min over interior points of 1/(S/h + mu/h^2), as ordered bits
    double dt;
    double t;
    long long step;
    DevError err;
};

// n / d for 0 <= n < 2^31 by one multiply and shift: m = ceil(2^(31+l) / d),
// l = ceil(log2 d), so n m / 2^(31+l) exceeds n / d by less than 1/d and the
// floor is exact (n m < 2^63)
struct FastDiv {
    unsigned d;
    int s;
    unsigned long long m;
};
inline FastDiv make_fastdiv(unsigned d) {
    int l = 0;
    while ((1ull << l) < d) ++l;
    FastDiv f;
    f.d = d;
    f.s = 31 + l;
    f.m = ((1ull << f.s) + d - 1) / d;
    return f;
}
FCSG_HD unsigned fdiv(const FastDiv& f, unsigned n) {
    return static_cast<unsigned>((static_cast<unsigned long long>(n) * f.m) >> f.s);
}

// BC table entry for one line end (BcSpec, include/fcs/bc.hpp:19-23)
struct BcDev {
    int kind;  // -1 none, else BcKind order: 0 inflow .. 5 zero_normal_all
    int pad;
    double state[4];
    double pressure;
};

// Device view of the engine's data. The engine stores subpatches grouped by
// shape (every field one array over all points, [slot][j][i] per subpatch);
// a *group view* covers the subpatches of one shape (S, ni, nj set, every
// pointer offset to the group's first point / subpatch / line), the *global
// view* covers all points (S = all subpatches, ni = nj = 0) and is used by the
// kernels that never need a point's (i, j): blend, exchange, dt, advance,
// halo pack/unpack and the proxy.
struct EngineDev {
    int S, ni, nj;
    int sub_base;   // storage slot of the view's first subpatch (error reports)
    int cartesian;  // 1: iq2x == iq1y == 0 at every point of the view
    int wpass_cap;  // persistent warp passes: CTAs per SM at most (0 = all that fit); engines with several
                    // shape groups leave room for the other groups' CTAs, which a full persistent grid starves
    int reference_order;  // 1: euler_rhs's own accumulation order (3 passes); 0: flux form
    long npts;      // points of the view (< 2^31)
    FastDiv div_ni, div_sz;  // by ni and by ni * nj (group views)
    double cfl, T;
    double visc_c[4];
    double abs_floor;
    int smear_radius;
    // per subpatch
    const double* h1;        // S: lattice spacing along q1 (LineInfo::inv_len = 1/((n-1) h1))
    const double* iq1x_c;    // S: iq1x / iq2y of subpatches where each is one value (uniform_q)
    const double* iq2y_c;
    int uniform_q;           // every subpatch of this view has uniform iq1x and iq2y
    const double* h2;
    const int* cut_i;        // S: L-shaped subpatch: points (i < cut_i && j < cut_j) are not
    const int* cut_j;        //    in the set (local, 0 = rectangular; geom::Subpatch::valid)
    const BcDev* bc_row_lo;  // S * nj (group view)
    const BcDev* bc_row_hi;
    const BcDev* bc_col_lo;  // S * ni
    const BcDev* bc_col_hi;
    // per-point geometry
    const uint8_t* mask;
    const double *iq1x, *iq2x, *iq1y, *iq2y, *h_min, *h_max, *w_norm;
    // state
    double* e[4];
    double* e0[4];
    double* e2[4];
    double* e3[4];
    double* rhs3[4];
    double* rhs[4];  // optional (nullptr unless debug_rhs): rhs of the last stage
    double *mu_hat, *mu, *tau, *speed, *proxy, *seed, *m01;
    // pass temporaries
    double* tA[4];   // inviscid partials, then the partial rhs
    double* tW[4];   // d/dq1 of w
    double* tS4[4];  // mu * grad_x w
    double* tS5[4];  // mu * grad_y w
    double* tF[4];   // filter/smear row results
    // diagnostics (workbench.cpp measurements): |grad e_c| per point
    // (allocated on first use) and the quadrature weights w_norm |det J|
    // x trapezoid factors (set by the caller)
    double* diag;
    const double* wq;
    // viscosity blend plan, CSR by recipient point (global view): copies,
    // then 6x6 tensor Lagrange interpolations (w, wx[6], wy[6] per entry)
    const int* visc_off;     // npts + 1
    const long* visc_src;    // global point index of donor
    const double* visc_w;
    const int* vi_off;       // npts + 1
    const long* vi_src;      // global index of the donor stencil origin (si0, sj0)
    const int* vi_pitch;     // donor ni
    const double* vi_w;      // 13 per entry: wx[6], wy[6], w
    // fringe exchange (global view): copies dst <- src, then interpolations
    const long* x_dst;
    const long* x_src;
    long n_x;
    const long* xi_dst;
    const long* xi_src;      // donor stencil origin
    const int* xi_pitch;
    const double* xi_w;      // 12 per entry: wx[6], wy[6]
    long n_xi;
    // classifier weights
    const double* mlp;       // kMlpWeights, FCNN order (per layer W row-major, then b)
    const double* mlp_frag;  // kMlpFrags x 32: per-lane DMMA operand fragments (mlp_mma_fragments)
    const double* tanh_tab;  // tanh(k/64), k = 0..1280 (classifier tanh table)
    double cls_fast_margin;  // logit margin above which the fast-tanh class is exact (mlp_fast_margin)
    double cls_margin32;     // logit margin above which the FP32 screen's class is exact (mlp_f32_margin)
    int* cls_fix_list;       // points the FP32 screen left to the exact classifier (capacity npts)
    unsigned* cls_fix_count; // (one counter per shape group view)
    // classifier variant (ClassifierConfig::Variant, include/fcs/viscosity.hpp:45-52):
    // 0 = ann (the MLP), 1 = fallback (FC spectrum decay, window fb_window)
    int cls_variant;
    int fb_window;
    int fb_ncont;
    const int* fb_off;     // fb_tab offset of window length w's table (build_spectrum_tail), w <= 64
    const double* fb_tab;
    StepScalars* sc;
};

// A run of consecutive lines of one subpatch that starts at `begin` along the
// line (L-shaped subpatches: rows j < cut_j begin at cut_i): one CTA's lines
// when a line set is given by descriptors.
struct LineDesc {
    int sub, line0, nl, begin;
};

// One launch's set of lines of one length n and orientation: FC plan and,
// for groups with L-shaped subpatches, descriptor lists for every CTA line
// count a pass uses (desc[k], n[k]: runs of at most kDescLB[k] lines; null:
// every line of every subpatch of the view, begin 0). A pass launched with LB
// lines per CTA takes exactly the LB list (desc_index), so no run is longer
// than its CTA.
constexpr int kDescLB[3] = {2, 4, 8};
inline int desc_index(int lb) { return lb == 2 ? 0 : (lb == 4 ? 1 : 2); }
struct LineSet {
    FcPlanDev pl;
    int scr;
    const LineDesc* desc[3];
    int n[3];
};

// everything the launchers need for one shape group
struct MlpF32;
struct GroupLaunch {
    EngineDev E;
    std::vector<LineSet> rows, cols;
    const MlpF32* w32 = nullptr;  // FP32 classifier weights (steady steps, ann variant), host copy
};

// The classifier on the FP64 tensor cores (mma.m8n8k4.f64): per warp, 8
// stencils x 8 neurons per MMA tile. Fragments: 0-3 layer-1 B (W1^T), 4-27
// hidden-layer B, 28-31 output-layer B, 32-47 hidden biases (C), 48-49 output
// bias; see classify_mma in step_kernels.cu for the lane layout.
constexpr int kMlpFrags = 50;
constexpr int kTanhTable = 1281;  // tanh(k/64), k = 0..1280
std::vector<double> mlp_mma_fragments(const std::vector<double>& packed);
double mlp_fast_margin(const std::vector<double>& packed);

int step_scr_cap(const FcPlanDev& pl);
// warp-per-line Cartesian flux passes on the n_ext = 280 prime-factor
// transform (wpass.cu): rows = pass X, else pass Y (stage = RK stage)
bool wpass_applies(const EngineDev& E, const FcPlanDev& pl, bool rows);
void launch_wpass(const EngineDev& E, const FcPlanDev& pl, bool rows, int stage, void* stream);
// the same passes on the register-resident 8 x 35 transform (wctpass.cu;
// FCSG_WPASS_CT=1 -- an A/B variant, measured slower than the prime-factor
// kernels of wpass.cu, which stay the default)
void launch_wctpass(const EngineDev& E, const FcPlanDev& pl, bool rows, int stage, void* stream);
// the phase-2 per-step filter (steady steps) on the same transform: rows
// (e -> tF) or columns (tF -> e)
void launch_wfilter(const EngineDev& E, const FcPlanDev& pl, bool rows, void* stream);
// dynamic shared memory of a line-pass CTA (lb lines, `slots` staging doubles
// per point) and the per-CTA opt-in limit of sm_100a (227 KB)
constexpr size_t kMaxLinePassSmem = 227 * 1024;
size_t line_pass_smem(const FcPlanDev& pl, int scr_cap, int slots, int lb);
// false when a line set's lines are too long for any pass's CTA shape
bool line_pass_smem_fits(const FcPlanDev& pl, int scr_cap);
// phase 0: proxy over all points (global view), classifier per group
void launch_phase0(const EngineDev& Eall, const std::vector<GroupLaunch>& G, bool step0, void* stream);
void launch_proxy(const EngineDev& Eall, void* stream);
void launch_classify(const EngineDev& Eall, const std::vector<GroupLaunch>& G, bool step0, void* stream);
void launch_phase1(const EngineDev& Eall, void* stream);
void launch_phase2(const std::vector<GroupLaunch>& G, bool step0, void* stream);
void launch_stage(const std::vector<GroupLaunch>& G, int stage, void* stream);
// the line passes of a stage, separately (profiling hooks)
void launch_pass_a(const std::vector<GroupLaunch>& G, void* stream);
void launch_pass_b(const std::vector<GroupLaunch>& G, int stage, void* stream);
void launch_pass_c(const std::vector<GroupLaunch>& G, int stage, void* stream);
// line-pass launches per stage (2 per line set for the Cartesian flux form, else 3)
int stage_launches(const std::vector<GroupLaunch>& G);
// diagnostics: |grad e_comp| into E.diag (two line passes per group);
// per-slot window quadrature sums of wq * (comp < 0 ? 1 : e_comp) into
// out[slot] (device, S doubles; slot_off = S + 1 point offsets); bilinear
// samples of E.diag at n raster pixels (corner point index, row pitch,
// fractions; base < 0 = outside the domain -> 0) into out (device)
void launch_gradient(const std::vector<GroupLaunch>& G, int comp, void* stream);
void launch_integrals(const EngineDev& Eall, int comp, const long* slot_off, int S, double* out, void* stream);
void launch_sample(const double* f, long n, const long* base, const int* pitch, const double* fu, const double* fv,
                   double* out, void* stream);
// kernel launches per superstep (excluding the t=0 dilation)
int launches_per_step(const std::vector<GroupLaunch>& G);
void launch_bc(const std::vector<GroupLaunch>& G, void* stream);
void launch_exchange(const EngineDev& Eall, void* stream);
void launch_finalize_dt(const EngineDev& Eall, void* stream);
void launch_advance(const EngineDev& Eall, void* stream);
// halo send list: idx[k] >= 0 is a point (global index); idx[k] = -1 - m
// sends the 6x6 interpolation m (stencil origin src[m], donor row pitch[m],
// weights w[12 m..]: wx[6], wy[6])
struct HaloPackDev {
    const long* src;
    const int* pitch;
    const double* w;
};
// halo pack/unpack (which: 0 state e as [k][4], 1 mu_hat as [k])
void launch_pack(const EngineDev& Eall, int which, const long* idx, long n, const HaloPackDev& hp, double* buf,
                 void* stream);
void launch_unpack(const EngineDev& Eall, int which, long n, const double* buf, void* stream);

}  // namespace fcsg
