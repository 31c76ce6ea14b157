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

struct EngineDev {
    int S, ni, nj;  // subpatches of one uniform rectangular shape
    int cartesian;  // 1: iq2x == iq1y == 0 at every point (axis-aligned maps)
    int reference_order;  // 1: euler_rhs's own accumulation order (3 passes); 0: flux form
    long npts;      // S * ni * nj (< 2^31)
    FastDiv div_ni, div_sz;  // by ni and by ni * nj (point index -> subpatch, row)
    double cfl, T;
    double visc_c[4];
    double abs_floor;
    int smear_radius;
    // per-subpatch
    const double* inv_len1;  // S
    const double* inv_len2;  // S
    const int* sub_i0;       // S: global lattice origin (error reports)
    const int* sub_j0;
    const int* sub_patch;
    const BcDev* bc_row_lo;  // S * nj
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
    // viscosity blend plan, CSR by recipient point
    const int* visc_off;     // npts + 1
    const long* visc_src;    // global point index of donor
    const double* visc_w;
    // fringe exchange (copies): dst/src global point indices
    const long* x_dst;
    const long* x_src;
    long n_x;
    // classifier weights
    const double* mlp;       // kMlpWeights, FCNN order (per layer W row-major, then b)
    const double* mlp_frag;  // kMlpFrags x 32: per-lane DMMA operand fragments (mlp_mma_fragments)
    const double* tanh_tab;  // tanh(k/64), k = 0..1280 (classifier tanh table)
    StepScalars* sc;
};

// The classifier on the FP64 tensor cores (mma.m8n8k4.f64): per warp, 8
// stencils x 8 neurons per MMA tile. Fragments: 0-3 layer-1 B (W1^T), 4-27
// hidden-layer B, 28-31 output-layer B, 32-47 hidden biases (C), 48-49 output
// bias; see classify_mma in step_kernels.cu for the lane layout.
constexpr int kMlpFrags = 50;
constexpr int kTanhTable = 1281;  // tanh(k/64), k = 0..1280
std::vector<double> mlp_mma_fragments(const std::vector<double>& packed);

// FC plans for the two line orientations (rows: n = ni, cols: n = nj)
struct LinePlans {
    FcPlanDev row, col;
    int scr_row, scr_col;
};

int step_scr_cap(const FcPlanDev& pl);
void launch_phase0(const EngineDev& E, bool step0, void* stream);
void launch_phase1(const EngineDev& E, void* stream);
void launch_phase2(const EngineDev& E, const LinePlans& P, bool step0, void* stream);
void launch_stage(const EngineDev& E, const LinePlans& P, int stage, void* stream);
// the three line passes of a stage, separately (profiling hooks)
void launch_pass_a(const EngineDev& E, const LinePlans& P, void* stream);
void launch_pass_b(const EngineDev& E, const LinePlans& P, int stage, void* stream);
void launch_pass_c(const EngineDev& E, const LinePlans& P, int stage, void* stream);
// line-pass launches per stage (2 for the Cartesian flux form, else 3)
int stage_launches(const EngineDev& E);
// kernel launches per superstep (excluding the t=0 dilation)
inline int launches_per_step(const EngineDev& E) { return 18 + 5 * stage_launches(E); }
void launch_bc(const EngineDev& E, void* stream);
void launch_exchange(const EngineDev& E, void* stream);
void launch_finalize_dt(const EngineDev& E, void* stream);
void launch_advance(const EngineDev& E, void* stream);
// halo pack/unpack (which: 0 state e as [k][4], 1 mu_hat as [k])
void launch_pack(const EngineDev& E, int which, const long* idx, long n, double* buf, void* stream);
void launch_unpack(const EngineDev& E, int which, long n, const double* buf, void* stream);

}  // namespace fcsg
