// Kernels of one FC-SDNN superstep (Engine::run body, src/runtime.cpp:482-511).
//
//  phase 0  proxy_kernel         proxy_value / mwsb_value per point (src/viscosity.cpp:13-29,
//                                runtime.cpp:327-346)
//           classify_mma_kernel  row + column 7-point stencils -> MLP on the FP64 tensor
//                                cores -> min -> mu_hat (src/viscosity.cpp:48-59,108-160,211-251)
//  phase 1  blend_kernel         mu = max(w_norm mu_hat + copies + 6x6 interpolations, 0) and
//                                the dt_bound_local min (src/runtime.cpp:352-371, euler.cpp:223-236)
//  phase 2  filter rows/cols + E rebuild (or the t=0 smear) (src/runtime.cpp:373-424,
//                                subpatch_data.cpp:30-67), dilation at t=0
//  stage    line passes          euler_rhs (src/euler.cpp:25-101) in the flux form
//                                div(mu grad w - f) and ssprk_stage_update (:182-221):
//                                Cartesian X (rows) + Y (cols), general GA + GB + C;
//                                reference accumulation order: A' B' C' / A B C
//           bc_kernel            enforce_bc, row ends then column ends (src/euler.cpp:105-180)
//           exchange_kernel      phase 6 copies and interpolations (src/runtime.cpp:433-454)
//
// Each line pass keeps two real quantities per complex FFT line (fft_line.h)
// and runs on one shape group of subpatches (step_kernels.h, EngineDev).
#include "dev.h"
#include "fft_line.h"
#include "pass_common.h"
#include "step_kernels.h"
#include "classify_f32.h"
#include "mlp_common.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

namespace fcsg {

// ---------------------------------------------------------------------------
// generic line pass

struct LineCtx {
    int sub;
    int line0;
    int nl_valid;
    int begin;  // first point along the line (L-shaped subpatches)
    long base;
    int ni;
    bool rows;
    double qy;  // the subpatch's uniform iq2y (EngineDev::uniform_q)
};

FCSG_HD long pidx(const LineCtx& c, int l, int i) {
    return c.rows ? c.base + static_cast<long>(c.line0 + l) * c.ni + c.begin + i
                  : c.base + static_cast<long>(c.begin + i) * c.ni + c.line0 + l;
}

// asynchronous 8-byte global -> shared copies (cp.async), used to prefetch the
// epilogue inputs of a round while its FFT runs
FCSG_HD void stage_copy(double* dst, const double* src) {
#if FCSG_CUDA
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
#else
    *dst = *src;
#endif
}
FCSG_HD void stage_commit() {
#if FCSG_CUDA
    asm volatile("cp.async.commit_group;\n" ::: "memory");
#endif
}
FCSG_HD void stage_wait() {
#if FCSG_CUDA
    asm volatile("cp.async.wait_all;\n" ::: "memory");
#endif
}

// Pass::kFetchAtEnd: the pass also prefetches (fetch) for the epilogue of
// its last round, which runs after the last transform with no load
template <class P, class = void>
struct FetchAtEnd {
    static constexpr bool v = false;
};
template <class P>
struct FetchAtEnd<P, std::void_t<decltype(P::kFetchAtEnd)>> {
    static constexpr bool v = P::kFetchAtEnd;
};

// One CTA owns LB lines of one subpatch (rows: stride-1 lines of length ni;
// columns: stride-ni lines of length nj). For every round r of the pass it
// loads two real quantities per point as one complex line, runs the FC
// transform in shared memory and hands the scaled result to the pass's
// epilogue. NE > 0 selects the compile-time plan for n_ext = NE (then
// N = NE - 24); NE = 0 is the runtime-generic plan. NTHR is the CTA size
// (1 in the CPU emulation harness).
//
// The epilogue of round r-1 and the load of round r share one loop (each
// shared-memory slot is read and rewritten by the same thread, so no barrier
// sits between them). The epilogue's global inputs (read-modify-write
// partials, metrics, mu, RK registers) are prefetched into shared memory with
// cp.async right before the round's FFT and waited for after it, so their
// latency hides behind the transform. Each thread stages and consumes only its
// own slots (stage[k * total + w]): kStage cp.async slots (a null source
// leaves a slot as the previous round staged it), then kStash slots the pass
// itself writes in load/store to keep per-point values across rounds. The
// double2 store(r - 1) returns is handed to load(r) at the same point (a round
// whose input is computed from the previous round's result).
template <int LB, class Pass, int NE, int NTHR>
FCSG_HD void line_pass(Thr t, int block, double2* smem, const Pass& P, const EngineDev& E, const FcPlanDev& pl,
                       int scr_cap, const LineDesc* desc) {
    constexpr bool rows = Pass::kRows;
    constexpr int pitch = LB;  // line index fastest, no padding: see fft_line.h
    constexpr int KS = Pass::kStage;
    const int ni = E.ni, nj = E.nj;
    const int N = NE > 0 ? NE - 24 : pl.n;  // the line length of this launch
    LineCtx c;
    if (desc) {  // explicit line runs (groups with L-shaped subpatches)
        const LineDesc d = desc[block];
        c.sub = d.sub;
        c.line0 = d.line0;
        c.nl_valid = d.nl < LB ? d.nl : LB;  // runs are built per LB (LineSet::desc); never longer
        c.begin = d.begin;
    } else {     // every line of every subpatch of the view
        const int nlines = rows ? nj : ni;
        const int bps = (nlines + LB - 1) / LB;
        c.sub = block / bps;
        c.line0 = (block - c.sub * bps) * LB;
        c.nl_valid = (nlines - c.line0 < LB) ? nlines - c.line0 : LB;
        c.begin = 0;
    }
    c.base = static_cast<long>(c.sub) * ni * nj;
    c.ni = ni;
    c.rows = rows;
    c.qy = E.uniform_q ? E.iq2y_c[c.sub] : 0.0;
    double2* buf = smem;
    double2* scr = smem + (NE > 0 ? NE : pl.n_ext) * pitch;
    double2* tabs = scr + scr_cap;
    double* stg = reinterpret_cast<double*>(tabs + table_slots(pl));
    const FcPlanDev spl = stage_tables(Thr{t.tid, NTHR}, pl, P.mode(0), tabs);  // one mode per pass
    // LineInfo::inv_len = 1 / ((n - 1) h) (src/subpatch_data.cpp:134,147)
    const double inv_len = P.kScaled ? 1.0 / ((N - 1) * (rows ? E.h1[c.sub] : E.h2[c.sub])) : 1.0;
    const int total = N * LB;
    const int tid = t.tid;
    for (int r = 0; r <= Pass::kRounds; ++r) {
        // the points of this thread, in chunks of KC: first every global read
        // the loads of the chunk need (registers), then the epilogue of round
        // r-1 and the load of round r per point. Issuing the reads first lets
        // them overlap each other and the epilogue stores, which the compiler
        // may not move them across (it cannot rule out aliasing).
        constexpr int PPT = NE > 0 ? ((NE - 24) * LB + NTHR - 1) / NTHR : 1;
        constexpr int KC = (NE > 0 && PPT >= 2) ? 2 : 1;
        constexpr bool kExact = NE > 0 && ((NE - 24) * LB) % (NTHR * KC) == 0;
        const int nch = NE > 0 ? (PPT + KC - 1) / KC : (total - tid + NTHR - 1) / NTHR;
        for (int ch = 0; ch < nch; ++ch) {
            double fv[KC][Pass::kFetch];
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int w = tid + (ch * KC + k) * NTHR;
                if (!kExact && w >= total) continue;
                // rows: consecutive lanes on consecutive points of one line
                // (coalesced global access); columns: across lines
                const int l = rows ? w / N : w % LB, i = rows ? w % N : w / LB;
                if ((r < Pass::kRounds || FetchAtEnd<Pass>::v) && l < c.nl_valid) P.fetch(r, pidx(c, l, i), fv[k]);
            }
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int w = tid + (ch * KC + k) * NTHR;
                if (!kExact && w >= total) continue;
                // rows: consecutive lanes on consecutive points of one line
                // (coalesced global access); columns: across lines
                const int l = rows ? w / N : w % LB, i = rows ? w % N : w / LB;
                if (l < c.nl_valid) {
                    const long p = pidx(c, l, i);
                    double2 carry = mk2(0.0, 0.0);
                    if (r > 0) {
                        const double2 v = buf[i * pitch + l];
                        carry = P.store(r - 1, p, mk2(v.x * inv_len, v.y * inv_len), stg + w, total, c, fv[k]);
                    }
                    if (r < Pass::kRounds) buf[i * pitch + l] = P.load(r, p, c, carry, fv[k], stg + w, total);
                } else if (r < Pass::kRounds) {
                    buf[i * pitch + l] = mk2(0.0, 0.0);
                }
            }
        }
        if (r == Pass::kRounds) break;
        if constexpr (KS > 0) {
            for (int w = tid; w < total; w += NTHR) {
                // rows: consecutive lanes on consecutive points of one line
                // (coalesced global access); columns: across lines
                const int l = rows ? w / N : w % LB, i = rows ? w % N : w / LB;
                if (l >= c.nl_valid) continue;
                const double* src[KS > 0 ? KS : 1];
                const int n = P.stage_srcs(r, pidx(c, l, i), src);
                for (int k = 0; k < n; ++k)
                    if (src[k]) stage_copy(stg + k * total + w, src[k]);
            }
            stage_commit();
        }
        FCSG_SYNC();
        if constexpr (NE > 0) {
            fc_transform_ct<NE, LB, NTHR>(tid, buf, spl, P.mode(r), scr, scr_cap);
        } else {
            fc_transform(Thr{tid, NTHR}, buf, pitch, LB, spl, P.mode(r), scr, scr_cap);
        }
        if constexpr (KS > 0) stage_wait();
    }
    FCSG_SYNC();
    P.finish(Thr{tid, NTHR}, c, N);
}

// interior positivity diagnostic of euler_rhs (src/euler.cpp:37-39)
FCSG_HD void check_positive(const EngineDev& E, const Prim& q, long p, const LineCtx& c) {
    const double pr = q.theta * ((q.rho != 0.0) ? q.rho : 1e-300);
    // the mask (interior points only) is read only for a failing point
    if ((!(q.rho > 0.0) || !(pr > 0.0) || !finite_d(pr)) && E.mask[p] == 1) {
        const long loc = p - c.base;
        raise_error(E.sc, 1, E.sub_base + c.sub, static_cast<int>(loc % c.ni), static_cast<int>(loc / c.ni));
    }
}

// Pass A (rows): D1 of F_c, G_c (rounds 0..3) and of w = (rho, rho u, rho v, theta) (4, 5)
// staged per store(r < 4): iq1x, iq1y
struct PassA {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 6;
    static constexpr int kStage = 2;
    static constexpr int kStash = 0;
    static constexpr int kLB = 8;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassA(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int, long p, double* v) const { fetch_e(E, p, v); }
    FCSG_HD double2 load(int r, long p, const LineCtx& c, double2, const double* fv, double*, int) const {
        const Prim q = prim_of(fv);
        if (r == 0) check_positive(E, q, p, c);
        if (r < 4) return flux_pair(q, r);
        if (r == 4) return mk2(q.rho, q.mx);
        return mk2(q.my, q.theta);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        if (r >= 4) return 0;
        s[0] = E.iq1x + p;
        s[1] = E.iq1y + p;
        return 2;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        if (r < 4) {
            E.tA[r][p] = st[0] * v.x + st[ss] * v.y;
        } else {
            const int c0 = 2 * (r - 4);
            E.tW[c0][p] = v.x;
            E.tW[c0 + 1][p] = v.y;
        }
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// Pass B (cols): D2 of F, G, w; inviscid rhs and mu grad w; then D2 of mu grad w.
// load(r >= 6) reads tS4/tS5[r-6], written by store(4 or 5) in an earlier round.
struct PassB {
    static constexpr bool kRows = false;
    static constexpr int kRounds = 10;
    static constexpr int kStage = 7;
    static constexpr int kStash = 0;
    static constexpr int kLB = 4;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassB(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int r, long p, double* v) const {
        if (r >= 6) {  // written by this thread in round 4 or 5
            v[0] = E.tS4[r - 6][p];
            v[1] = E.tS5[r - 6][p];
        } else {
            fetch_e(E, p, v);
        }
    }
    FCSG_HD double2 load(int r, long, const LineCtx&, double2, const double* fv, double*, int) const {
        if (r >= 6) return mk2(fv[0], fv[1]);
        const Prim q = prim_of(fv);
        if (r < 4) return flux_pair(q, r);
        if (r == 4) return mk2(q.rho, q.mx);
        return mk2(q.my, q.theta);
    }
    // r<4: tA[r], iq2x, iq2y; r=4,5: iq2x, iq2y, iq1x, iq1y, mu, tW x2; r>=6: tA[r-6], iq2x, iq2y
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        s[0] = E.iq2x + p;
        s[1] = E.iq2y + p;
        if (r < 4) {
            s[2] = E.tA[r] + p;
            return 3;
        }
        if (r < 6) {
            const int c0 = 2 * (r - 4);
            s[2] = E.iq1x + p;
            s[3] = E.iq1y + p;
            s[4] = E.mu + p;
            s[5] = E.tW[c0] + p;
            s[6] = E.tW[c0 + 1] + p;
            return 7;
        }
        s[2] = E.tA[r - 6] + p;
        return 3;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        const double b = st[0], d = st[ss];
        if (r < 4) {
            E.tA[r][p] = -(st[2 * ss] + (b * v.x + d * v.y));
        } else if (r < 6) {
            const int c0 = 2 * (r - 4);
            const double a = st[2 * ss], cc = st[3 * ss], mu = st[4 * ss];
            const double d1[2] = {st[5 * ss], st[6 * ss]};
            const double d2[2] = {v.x, v.y};
            for (int k = 0; k < 2; ++k) {
                const double gx = a * d1[k] + b * d2[k];
                const double gy = cc * d1[k] + d * d2[k];
                E.tS4[c0 + k][p] = mu * gx;
                E.tS5[c0 + k][p] = mu * gy;
            }
        } else {
            E.tA[r - 6][p] = st[2 * ss] + (b * v.x + d * v.y);
        }
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// Pass C (rows): D1 of mu grad w, rhs, SSPRK(5,4) stage update
// staged per store(c): tA[c], iq1x, iq1y, e[c]
struct PassC {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 4;
    static constexpr int kStage = 4;
    static constexpr int kStash = 0;
    static constexpr int kLB = 4;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    int stage;
    double dt;  // the step size (finalize_dt_kernel), read once per block
    FCSG_HD PassC(const EngineDev& e, int s) : E(e), stage(s), dt(e.sc->dt) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 2;
    FCSG_HD void fetch(int r, long p, double* v) const {
        v[0] = ldg1(E.tS4[r] + p);
        v[1] = ldg1(E.tS5[r] + p);
    }
    FCSG_HD double2 load(int, long, const LineCtx&, double2, const double* fv, double*, int) const {
        return mk2(fv[0], fv[1]);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        s[0] = E.tA[r] + p;
        s[1] = E.iq1x + p;
        s[2] = E.iq1y + p;
        s[3] = E.e[r] + p;
        return 4;
    }
    FCSG_HD double2 store(int c, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        ssprk_update(E, stage, c, p, st[3 * ss], st[0] + (st[ss] * v.x + st[2 * ss] * v.y), dt);
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// ---- diagnostics: |grad e_c| (density_gradient_raster, src/workbench.cpp:222-239)
// rows: d/dq1 of e_c into tA[0] (SubpatchData::deriv_q1); columns: d/dq2,
// then gx = iq1x d1 + iq2x d2, gy = iq1y d1 + iq2y d2, |grad| = hypot(gx, gy)
// at the points of the set, 0 elsewhere
struct PassDiagR {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 1;
    static constexpr int kStage = 0;
    static constexpr int kStash = 0;
    static constexpr int kLB = 8;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    int comp;
    FCSG_HD PassDiagR(const EngineDev& e, int c) : E(e), comp(c) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 1;
    FCSG_HD void fetch(int, long p, double* v) const { v[0] = ldg1(E.e[comp] + p); }
    FCSG_HD double2 load(int, long, const LineCtx&, double2, const double* fv, double*, int) const {
        return mk2(fv[0], 0.0);
    }
    FCSG_HD int stage_srcs(int, long, const double**) const { return 0; }
    FCSG_HD double2 store(int, long p, double2 v, const double*, int, const LineCtx&, const double*) const {
        E.tA[0][p] = v.x;
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};
struct PassDiagC {
    static constexpr bool kRows = false;
    static constexpr int kRounds = 1;
    static constexpr int kStage = 0;
    static constexpr int kStash = 0;
    static constexpr int kLB = 4;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    int comp;
    FCSG_HD PassDiagC(const EngineDev& e, int c) : E(e), comp(c) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 1;
    FCSG_HD void fetch(int, long p, double* v) const { v[0] = ldg1(E.e[comp] + p); }
    FCSG_HD double2 load(int, long, const LineCtx&, double2, const double* fv, double*, int) const {
        return mk2(fv[0], 0.0);
    }
    FCSG_HD int stage_srcs(int, long, const double**) const { return 0; }
    FCSG_HD double2 store(int, long p, double2 v, const double*, int, const LineCtx&, const double*) const {
        const double d1 = E.tA[0][p], d2 = v.x;
        const double gx = E.iq1x[p] * d1 + E.iq2x[p] * d2;
        const double gy = E.iq1y[p] * d1 + E.iq2y[p] * d2;
        E.diag[p] = hypot(gx, gy);
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// ---- Cartesian subpatches --------------------------------------------------
// When iq2x and iq1y vanish identically (axis-aligned affine maps, every
// subpatch of BASELINE configs 2 and 5), the reference still computes
// D2 F_c, D1 G_c, D2 (mu grad_x w) and D1 (mu grad_y w) but multiplies them by
// those exact zeros (src/euler.cpp:16-21,109,126,137-138,144,147). Dropping
// the zero products changes nothing but FMA-contraction rounding choices
// (m*x + 0*y == m*x exactly). These passes drop them: 12 instead of 20
// complex line transforms per stage. Engines with any curvilinear subpatch
// use the general passes above.

// A': D1 of F_c (rounds 0, 1) and of w (2, 3); staged per store(r < 2): iq1x
struct PassAc {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 4;
    static constexpr int kStage = 1;
    static constexpr int kStash = 0;
    static constexpr int kLB = 8;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassAc(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int, long p, double* v) const { fetch_e(E, p, v); }
    FCSG_HD double2 load(int r, long p, const LineCtx& c, double2, const double* fv, double*, int) const {
        const Prim q = prim_of(fv);
        if (r == 0) check_positive(E, q, p, c);
        if (r < 2) {
            const double2 f0 = flux_pair(q, 2 * r), f1 = flux_pair(q, 2 * r + 1);
            return mk2(f0.x, f1.x);
        }
        if (r == 2) return mk2(q.rho, q.mx);
        return mk2(q.my, q.theta);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        if (r >= 2) return 0;
        s[0] = E.iq1x + p;
        return 1;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int, const LineCtx&, const double*) const {
        if (r < 2) {
            const double a = st[0];
            E.tA[2 * r][p] = a * v.x;
            E.tA[2 * r + 1][p] = a * v.y;
        } else {
            const int c0 = 2 * (r - 2);
            E.tW[c0][p] = v.x;
            E.tW[c0 + 1][p] = v.y;
        }
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// B': D2 of G_c (0, 1) and of w (2, 3) -> inviscid rhs, mu grad w; D2 of mu grad_y w (4, 5)
// staged: iq2y and r<2: tA pair; r=2,3: iq1x, mu, tW pair; r=4,5: tA pair
struct PassBc {
    static constexpr bool kRows = false;
    static constexpr int kRounds = 6;
    static constexpr int kStage = 5;
    static constexpr int kStash = 0;
    static constexpr int kLB = 4;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassBc(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int r, long p, double* v) const {
        if (r >= 4) {  // written by this thread in round 2 or 3
            v[0] = E.tS5[2 * (r - 4)][p];
            v[1] = E.tS5[2 * (r - 4) + 1][p];
        } else {
            fetch_e(E, p, v);
        }
    }
    FCSG_HD double2 load(int r, long, const LineCtx&, double2, const double* fv, double*, int) const {
        if (r >= 4) return mk2(fv[0], fv[1]);
        const Prim q = prim_of(fv);
        if (r < 2) {
            const double2 f0 = flux_pair(q, 2 * r), f1 = flux_pair(q, 2 * r + 1);
            return mk2(f0.y, f1.y);
        }
        if (r == 2) return mk2(q.rho, q.mx);
        return mk2(q.my, q.theta);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        s[0] = E.iq2y + p;
        if (r < 2) {
            s[1] = E.tA[2 * r] + p;
            s[2] = E.tA[2 * r + 1] + p;
            return 3;
        }
        if (r < 4) {
            const int c0 = 2 * (r - 2);
            s[1] = E.tW[c0] + p;
            s[2] = E.tW[c0 + 1] + p;
            s[3] = E.iq1x + p;
            s[4] = E.mu + p;
            return 5;
        }
        s[1] = E.tA[2 * (r - 4)] + p;
        s[2] = E.tA[2 * (r - 4) + 1] + p;
        return 3;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        const double d = st[0], t0 = st[ss], t1 = st[2 * ss];
        if (r < 2) {
            E.tA[2 * r][p] = -(t0 + d * v.x);
            E.tA[2 * r + 1][p] = -(t1 + d * v.y);
        } else if (r < 4) {
            const int c0 = 2 * (r - 2);
            const double a = st[3 * ss], mu = st[4 * ss];
            E.tS4[c0][p] = mu * (a * t0);
            E.tS4[c0 + 1][p] = mu * (a * t1);
            E.tS5[c0][p] = mu * (d * v.x);
            E.tS5[c0 + 1][p] = mu * (d * v.y);
        } else {
            const int c0 = 2 * (r - 4);
            E.tA[c0][p] = t0 + d * v.x;
            E.tA[c0 + 1][p] = t1 + d * v.y;
        }
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// C': D1 of mu grad_x w -> rhs -> SSPRK stage update; staged: tA pair, iq1x, e pair
struct PassCc {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 2;
    static constexpr int kStage = 5;
    static constexpr int kStash = 0;
    static constexpr int kLB = 4;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    int stage;
    double dt;  // the step size (finalize_dt_kernel), read once per block
    FCSG_HD PassCc(const EngineDev& e, int s) : E(e), stage(s), dt(e.sc->dt) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 2;
    FCSG_HD void fetch(int r, long p, double* v) const {
        v[0] = ldg1(E.tS4[2 * r] + p);
        v[1] = ldg1(E.tS4[2 * r + 1] + p);
    }
    FCSG_HD double2 load(int, long, const LineCtx&, double2, const double* fv, double*, int) const {
        return mk2(fv[0], fv[1]);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        s[0] = E.tA[2 * r] + p;
        s[1] = E.tA[2 * r + 1] + p;
        s[2] = E.iq1x + p;
        s[3] = E.e[2 * r] + p;
        s[4] = E.e[2 * r + 1] + p;
        return 5;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        const double a = st[2 * ss];
        ssprk_update(E, stage, 2 * r, p, st[3 * ss], st[0] + a * v.x, dt);
        ssprk_update(E, stage, 2 * r + 1, p, st[4 * ss], st[ss] + a * v.y, dt);
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// ---- flux form (default) ---------------------------------------------------
// euler_rhs accumulates, per component c (src/euler.cpp:43-100),
//   -(iq1x D1F + iq2x D2F) - (iq1y D1G + iq2y D2G) + (iq1x D1s4 + iq2x D2s4) + (iq1y D1s5 + iq2y D2s5)
// with s4 = mu grad_x w and s5 = mu grad_y w. The FC derivative is linear and
// the same metric factor multiplies D_k F and D_k s4 (resp. D_k G and D_k s5),
// so the rhs equals
//   iq1x D1(s4 - F) + iq2x D2(s4 - F) + iq1y D1(s5 - G) + iq2y D2(s5 - G),
// i.e. div(mu grad w - f): the same operator, differing only by round-off
// reassociation, with 24 line derivatives per stage instead of 40 (16 instead
// of 24 on Cartesian subpatches, where iq2x = iq1y = 0 as above).
// EngineConfig::reference_order keeps the reference's accumulation (passes
// A/B/C and A'/B'/C' above).

// Cartesian flux form, pass X (rows, 4 rounds): D1 of (rho, rho u) ->
// Phi_x = mu iq1x D1 w - F (handed to the next round) -> D1 Phi_x ->
// tA = iq1x D1 Phi_x; then the same for (rho v, theta).
// slots: 0 iq1x, 1 mu (staged in the rounds that differentiate w, kept after)
struct PassXc {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 4;
    static constexpr int kStage = 2;
    static constexpr int kStash = 2;
    static constexpr int kLB = 2;
    static constexpr int kNT = 128;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassXc(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    // the w rounds read e and stash the pair of x-fluxes the next round needs
    // (slots 2, 3); the Phi rounds read nothing from global memory
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int r, long p, double* v) const {
        if (!(r & 1)) fetch_e(E, p, v);
    }
    FCSG_HD double2 load(int r, long p, const LineCtx& c, double2 carry, const double* fv, double* st, int ss) const {
        if (r & 1) return mk2(carry.x - st[2 * ss], carry.y - st[3 * ss]);
        const Prim q = prim_of(fv);
        const double2 f0 = flux_pair(q, r), f1 = flux_pair(q, r + 1);
        st[2 * ss] = f0.x;
        st[3 * ss] = f1.x;
        if (r == 0) {
            check_positive(E, q, p, c);
            return mk2(q.rho, q.mx);
        }
        return mk2(q.my, q.theta);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        // iq1x and mu once, in round 0: the slots keep them for every later round
        if (r != 0) return 0;
        s[0] = E.iq1x + p;  // (staged even when uniform: measured faster than a per-subpatch value here)
        s[1] = E.mu + p;
        return 2;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        const double a = st[0];
        if (!(r & 1)) {
            const double m = st[ss];
            return mk2(m * (a * v.x), m * (a * v.y));  // s4 = mu (iq1x D1 w + 0 D2 w)
        }
        const int c0 = r - 1;
        E.tA[c0][p] = a * v.x;
        E.tA[c0 + 1][p] = a * v.y;
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// Cartesian flux form, pass Y (cols, 4 rounds): D2 of (rho v, theta) ->
// Phi_y = mu iq2y D2 w - G -> D2 Phi_y -> rhs = tA + iq2y D2 Phi_y -> SSPRK
// update of components 2, 3; then the same for (rho, rho u). Components 2, 3
// are updated first: G_0 = rho v and G_1 = rho u v need the old rho v, kept in
// stash slot 3 by the first load (rho and rho u are still unmodified then).
// The updates' current values u come from the stash too: slots 3, 4 hold
// (rho v, E) from the first load for the first update, then (rho, rho u)
// from the last load for the second.
// slots: 0 iq2y, 1 mu | 1, 2 tA pair (update rounds), 3-4 stash
#ifndef FCSG_YC_LB
#define FCSG_YC_LB 4  // lines per CTA of the block-transform pass Y (A/B knob; 2 runs 128-thread CTAs: measured slower)
#endif
struct PassYc {
    static constexpr bool kRows = false;
    static constexpr int kRounds = 4;
    static constexpr int kStage = 3;
    static constexpr int kStash = 2;
    static constexpr int kLB = FCSG_YC_LB;
    static constexpr int kNT = FCSG_YC_LB == 2 ? 128 : 256;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    int stage;
    double dt;  // the step size (finalize_dt_kernel), read once per block
    FCSG_HD PassYc(const EngineDev& e, int s) : E(e), stage(s), dt(e.sc->dt) {}
    FCSG_HD int mode(int) const { return 1; }
    // fetch: the load's values in v[0..3] (rounds 0, 1) or v[0..1] (rounds 2,
    // 3); in rounds 2 and 4 (after the last transform) also the register e0
    // of the components the preceding update writes, in v[2..3]
    static constexpr int kFetch = 4;
    static constexpr bool kFetchAtEnd = true;
    FCSG_HD void fetch(int r, long p, double* v) const {
        if (r == 0) {
            fetch_e(E, p, v);
            return;
        }
        if (r == 1) {  // rho v and E come from the round-0 stash (e is unmodified until round 2)
            v[0] = ldg1(E.e[0] + p);
            v[1] = ldg1(E.e[1] + p);
            return;
        }
        if (r < 4) {  // rho (and in round 2 rho u): updated only in the last round
            v[0] = ldg1(E.e[0] + p);
            if (r == 2) v[1] = ldg1(E.e[1] + p);  // round 3 takes rho u from the stash
        }
        if (!(r & 1) && stage >= 1 && stage <= 3) {
            const int c0 = r == 2 ? 2 : 0;
            v[2] = ldg1(E.e0[c0] + p);
            v[3] = ldg1(E.e0[c0 + 1] + p);
        }
    }
    FCSG_HD double2 load(int r, long, const LineCtx&, double2 carry, const double* fv, double* st, int ss) const {
        switch (r) {
            case 0: {
                const Prim q = prim_of(fv);
                st[3 * ss] = q.my;
                st[4 * ss] = q.E;
                return mk2(q.my, q.theta);
            }
            case 1: {
                const double f4[4] = {fv[0], fv[1], st[3 * ss], st[4 * ss]};
                const Prim q = prim_of(f4);
                return mk2(carry.x - flux_pair(q, 2).y, carry.y - flux_pair(q, 3).y);
            }
            case 2:
                st[4 * ss] = fv[1];  // rho u for round 3 (slot 4's E was last read by store(1))
                return mk2(fv[0], fv[1]);
            default: {
                const double rho = fv[0], mx = st[4 * ss], my = st[3 * ss];
                st[3 * ss] = rho;  // u of the last update
                st[4 * ss] = mx;
                const double v = my / rho;
                return mk2(carry.x - my, carry.y - mx * v);  // G_0, G_1 (src/euler.cpp:64-75)
            }
        }
    }
    // slots: 0 iq2y, 1 mu (even rounds) / tA pair in 1, 2 (odd rounds); with a
    // uniform iq2y (read per subpatch) the tA pair goes to 0, 2 instead, so mu
    // staged in round 0 stays in slot 1 for round 2
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        const bool u = E.uniform_q;
        if (!(r & 1)) {
            if (u && r == 2) return 0;
            s[0] = u ? nullptr : E.iq2y + p;
            s[1] = E.mu + p;
            return 2;
        }
        const int c0 = r == 1 ? 2 : 0;
        s[0] = u ? E.tA[c0] + p : nullptr;  // not uniform: keep iq2y
        s[1] = u ? nullptr : E.tA[c0] + p;  // uniform: keep mu
        s[2] = E.tA[c0 + 1] + p;
        return 3;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx& c,
                          const double* fv) const {
        const double d = E.uniform_q ? c.qy : st[0];
        if (!(r & 1)) {
            const double m = st[ss];
            return mk2(m * (d * v.x), m * (d * v.y));  // s5 = mu (0 D1 w + iq2y D2 w)
        }
        const int c0 = r == 1 ? 2 : 0;
        const double ta = E.uniform_q ? st[0] : st[ss];
        ssprk_update_e0(E, stage, c0, p, st[3 * ss], ta + d * v.x, fv[2], dt);
        ssprk_update_e0(E, stage, c0 + 1, p, st[4 * ss], st[2 * ss] + d * v.y, fv[3], dt);
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// General flux form, pass A (rows, 2 rounds): D1 w -> tW
struct PassGA {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 2;
    static constexpr int kStage = 0;
    static constexpr int kStash = 0;
    static constexpr int kLB = 8;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassGA(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int, long p, double* v) const { fetch_e(E, p, v); }
    FCSG_HD double2 load(int r, long p, const LineCtx& c, double2, const double* fv, double*, int) const {
        const Prim q = prim_of(fv);
        if (r == 0) {
            check_positive(E, q, p, c);
            return mk2(q.rho, q.mx);
        }
        return mk2(q.my, q.theta);
    }
    FCSG_HD int stage_srcs(int, long, const double**) const { return 0; }
    FCSG_HD double2 store(int r, long p, double2 v, const double*, int, const LineCtx&, const double*) const {
        E.tW[2 * r][p] = v.x;
        E.tW[2 * r + 1][p] = v.y;
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// General flux form, pass B (cols, 6 rounds per component pair):
// D2 w -> Phi_x = mu grad_x w - F (tS4), Phi_y = mu grad_y w - G (tS5, and
// the next round's input) -> D2 Phi_y -> tA = iq2y D2 Phi_y -> D2 Phi_x ->
// tA += iq2x D2 Phi_x. Pass C then adds iq1x D1 Phi_x + iq1y D1 Phi_y and
// updates (PassC reads tS4/tS5 = Phi_x/Phi_y).
// slots: 0 iq1x, 1 iq2x, 2 iq1y, 3 iq2y, 4 mu, 5-6 tW pair (staged in the w rounds)
struct PassGB {
    static constexpr bool kRows = false;
    static constexpr int kRounds = 6;
    static constexpr int kStage = 7;
    static constexpr int kStash = 0;
    static constexpr int kLB = 4;
    static constexpr bool kScaled = true;
    const EngineDev& E;
    FCSG_HD PassGB(const EngineDev& e, int) : E(e) {}
    FCSG_HD int mode(int) const { return 1; }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int r, long p, double* v) const {
        const int k = r % 3, c0 = 2 * (r / 3);
        if (k == 0) {
            fetch_e(E, p, v);
        } else if (k == 2) {  // written by this thread in round r - 2
            v[0] = E.tS4[c0][p];
            v[1] = E.tS4[c0 + 1][p];
        }
    }
    FCSG_HD double2 load(int r, long, const LineCtx&, double2 carry, const double* fv, double*, int) const {
        const int k = r % 3, c0 = 2 * (r / 3);
        if (k == 1) return carry;
        if (k == 2) return mk2(fv[0], fv[1]);
        const Prim q = prim_of(fv);
        return c0 == 0 ? mk2(q.rho, q.mx) : mk2(q.my, q.theta);
    }
    FCSG_HD int stage_srcs(int r, long p, const double** s) const {
        if (r % 3 != 0) return 0;  // metric slots kept from the w round
        const int c0 = 2 * (r / 3);
        s[0] = E.iq1x + p;
        s[1] = E.iq2x + p;
        s[2] = E.iq1y + p;
        s[3] = E.iq2y + p;
        s[4] = E.mu + p;
        s[5] = E.tW[c0] + p;
        s[6] = E.tW[c0 + 1] + p;
        return 7;
    }
    FCSG_HD double2 store(int r, long p, double2 v, const double* st, int ss, const LineCtx&, const double*) const {
        const int k = r % 3, c0 = 2 * (r / 3);
        if (k == 0) {
            const double a = st[0], b = st[ss], cc = st[2 * ss], d = st[3 * ss], mu = st[4 * ss];
            const double d1[2] = {st[5 * ss], st[6 * ss]};
            const double d2[2] = {v.x, v.y};
            const Prim q = prim_rhs(E, p);
            double phy[2];
            for (int j = 0; j < 2; ++j) {
                const double2 fg = flux_pair(q, c0 + j);
                const double gx = a * d1[j] + b * d2[j];
                const double gy = cc * d1[j] + d * d2[j];
                E.tS4[c0 + j][p] = mu * gx - fg.x;
                phy[j] = mu * gy - fg.y;
                E.tS5[c0 + j][p] = phy[j];
            }
            return mk2(phy[0], phy[1]);
        }
        if (k == 1) {
            const double d = st[3 * ss];
            E.tA[c0][p] = d * v.x;
            E.tA[c0 + 1][p] = d * v.y;
            return {};
        }
        const double b = st[ss];
        E.tA[c0][p] = E.tA[c0][p] + b * v.x;
        E.tA[c0 + 1][p] = E.tA[c0 + 1][p] + b * v.y;
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// lines per CTA of the phase-2 filter passes (A/B knob): 4 gives a single
// 512 x 512 subpatch 128 CTAs instead of 64 (config 2: filter 0.175 -> 0.088 ms,
// superstep 1.17 -> 1.08 ms; 2 lines per CTA the same; configs 3 and 4 unchanged)
#ifndef FCSG_FILTER_LB
#define FCSG_FILTER_LB 4
#endif

// Phase 2 rows: filter (or, at t=0, smear) rho, rho u, rho v, theta
// (src/runtime.cpp:375-411, subpatch_data.cpp:30-67). Writes tF only.
struct PassFR {
    static constexpr bool kRows = true;
    static constexpr int kRounds = 2;
    static constexpr int kStage = 0;
    static constexpr int kStash = 0;
    static constexpr int kLB = FCSG_FILTER_LB;
    static constexpr bool kScaled = false;
    const EngineDev& E;
    bool smear;
    FCSG_HD PassFR(const EngineDev& e, int sm) : E(e), smear(sm != 0) {}
    FCSG_HD int mode(int) const { return smear ? 4 : 3; }
    FCSG_HD static double2 orig(const EngineDev& E, int r, long p) {
        const double rho = ldg1(E.e[0] + p), mx = ldg1(E.e[1] + p);
        if (r == 0) return mk2(rho, mx);
        const double my = ldg1(E.e[2] + p), En = ldg1(E.e[3] + p);
        const double th = kGm1 * (En - 0.5 * (mx * mx + my * my) / rho) / rho;
        return mk2(my, th);
    }
    static constexpr int kFetch = 4;
    FCSG_HD void fetch(int r, long p, double* v) const {
        v[0] = ldg1(E.e[0] + p);
        v[1] = ldg1(E.e[1] + p);
        if (r == 1) {
            v[2] = ldg1(E.e[2] + p);
            v[3] = ldg1(E.e[3] + p);
        }
    }
    FCSG_HD double2 load(int r, long, const LineCtx&, double2, const double* fv, double*, int) const {
        if (r == 0) return mk2(fv[0], fv[1]);
        const double rho = fv[0], mx = fv[1], my = fv[2], En = fv[3];
        return mk2(my, kGm1 * (En - 0.5 * (mx * mx + my * my) / rho) / rho);
    }
    FCSG_HD int stage_srcs(int, long, const double**) const { return 0; }
    FCSG_HD double2 store(int r, long p, double2 v, const double*, int, const LineCtx&, const double*) const {
        if (smear) {
            const double m = E.m01[p];
            const double2 f = orig(E, r, p);
            v = mk2(m * v.x + (1.0 - m) * f.x, m * v.y + (1.0 - m) * f.y);
        }
        E.tF[2 * r][p] = v.x;
        E.tF[2 * r + 1][p] = v.y;
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// Phase 2 cols: filter/smear columns of the row results, then E rebuild
struct PassFC {
    static constexpr bool kRows = false;
    static constexpr int kRounds = 2;
    static constexpr int kStage = 0;
    static constexpr int kStash = 0;
    static constexpr int kLB = FCSG_FILTER_LB;
    static constexpr bool kScaled = false;
    const EngineDev& E;
    bool smear;
    FCSG_HD PassFC(const EngineDev& e, int sm) : E(e), smear(sm != 0) {}
    FCSG_HD int mode(int) const { return smear ? 4 : 3; }
    static constexpr int kFetch = 2;
    FCSG_HD void fetch(int r, long p, double* v) const {
        v[0] = E.tF[2 * r][p];
        v[1] = E.tF[2 * r + 1][p];
    }
    FCSG_HD double2 load(int, long, const LineCtx&, double2, const double* fv, double*, int) const {
        return mk2(fv[0], fv[1]);
    }
    FCSG_HD int stage_srcs(int, long, const double**) const { return 0; }
    FCSG_HD double2 store(int r, long p, double2 v, const double*, int, const LineCtx&, const double*) const {
        if (smear) {
            const double m = E.m01[p];
            const double fa = E.tF[2 * r][p], fb = E.tF[2 * r + 1][p];
            v = mk2(m * v.x + (1.0 - m) * fa, m * v.y + (1.0 - m) * fb);
        }
        if (r == 0) {
            E.e[0][p] = v.x;
            E.e[1][p] = v.y;
        } else {
            // E = rho theta/(gamma-1) + |m|^2 / (2 rho) (src/runtime.cpp:413-420);
            // rho, rho u were written at this point by this thread in round 0
            const double rho = E.e[0][p], mx = E.e[1][p], my = v.x;
            E.e[2][p] = my;
            E.e[3][p] = rho * v.y / kGm1 + 0.5 * (mx * mx + my * my) / rho;
        }
        return {};
    }
    FCSG_HD void finish(Thr, const LineCtx&, int) const {}
};

// ---------------------------------------------------------------------------
// pointwise kernels

// phase 0, part 1: Mach proxy and wave-speed bound (src/viscosity.cpp:13-29)
FCSG_HD void proxy_body(Thr t, int block, int nblocks, const EngineDev& E) {
    const long step = static_cast<long>(nblocks) * t.nthr;
    for (long p = static_cast<long>(block) * t.nthr + t.tid; p < E.npts; p += step) {
        if (!E.mask[p]) {
            E.proxy[p] = 0.0;
            E.speed[p] = 1.0;
            continue;
        }
        const double rho = E.e[0][p], ru = E.e[1][p], rv = E.e[2][p], En = E.e[3][p];
        const double u = ru / rho, v = rv / rho;
        const double ke = 0.5 * rho * (u * u + v * v);
        const double pr = kGm1 * (En - ke);
        if (!(rho > 0.0) || !(pr > 0.0)) {
            raise_error_gp(E.sc, 2, p);
            E.proxy[p] = 0.0;
            E.speed[p] = 1.0;
            continue;
        }
        const double um = sqrt(u * u + v * v);
        E.proxy[p] = um * sqrt(rho / (kG * pr));
        E.speed[p] = um + sqrt(kG * pr / rho);
    }
}

// classifier weights: in the CUDA build they live in the constant bank (every
// thread of a warp reads the same weight at the same time, so each DFMA takes
// its weight straight from c[][]); refreshed from E.mlp before each launch
#if FCSG_CUDA
__constant__ double c_mlp[kMlpWeights];
struct MlpW {
    FCSG_HD double operator()(int k) const { return c_mlp[k]; }
};
#else
struct MlpW {
    const double* p;
    double operator()(int k) const { return p[k]; }
};
#endif


#if FCSG_CUDA
// tanh on the FP32 pipe and the SFU (|error| <= 4e-7 absolute: ex2 and rcp
// approximations, two roundings to float), for the classifier's fast pass:
// the FP64 pipe stays with the DMMA layers. Only the argmax of the logits
// is used, and the fast pass's result is kept only where its logit margin
// exceeds EngineDev::cls_fast_margin, twice a rigorous bound of the logit
// error this tanh can cause (mlp_fast_margin); elsewhere the group is
// classified again with tanh_tab.
//
// The double <-> float conversions are done on the integer bits (ALU pipe)
// instead of F2F, which issues on the same XU pipe as the two MUFU ops and
// made it the classifier's limiter: |z| is truncated to float (relative error
// 2^-23, i.e. <= 6e-8 absolute on tanh; |z| < 2^-126 becomes 0, |z| > 2^128
// FLT_MAX), the result in [0, 1] is widened exactly.
__device__ __forceinline__ double tanh_fast(double z) {
    const unsigned hi = static_cast<unsigned>(__double2hiint(z)), lo = static_cast<unsigned>(__double2loint(z));
    int a = static_cast<int>(hi & 0x7fffffffu) - 0x38000000;  // exponent bias 1023 -> 127
    a = min(max(a, 0), 0x0fefffff);
    const float ax = __uint_as_float((static_cast<unsigned>(a) << 3) | (lo >> 29));
    float t, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(2.8853900817779268f * ax));  // e^(2|x|)
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t + 1.0f));
    const unsigned yb = __float_as_uint(fmaxf(fmaf(-2.0f, r, 1.0f), 0.0f));  // tanh |x| = 1 - 2 / (e^(2|x|) + 1)
    const unsigned dhi = yb == 0u ? 0u : (yb >> 3) + 0x38000000u;
    return __hiloint2double(static_cast<int>(dhi | (hi & 0x80000000u)), static_cast<int>(yb << 29));
}
#endif

// normalize_stencil (src/viscosity.cpp:48-59): false = class-4 guard
FCSG_HD bool normalize7(const double* s, double abs_floor, double* x) {
    double lo = s[0], hi = s[0];
#pragma unroll
    for (int k = 1; k < kMlpIn; ++k) {
        lo = s[k] < lo ? s[k] : lo;
        hi = s[k] > hi ? s[k] : hi;
    }
    const double span = hi - lo;
    double scale = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
    scale = scale > 1e-100 ? scale : 1e-100;
    if (span <= 1e-13 * scale || span <= abs_floor) return false;
#pragma unroll
    for (int k = 0; k < kMlpIn; ++k) x[k] = 2.0 * (s[k] - lo) / span - 1.0;
    return true;
}


// Classifier::classify (src/viscosity.cpp:211-238) for one point of a
// subpatch: min of the row-window and column-window classes. The row of the
// point is the segment [rb, ni), its column [cb, nj) (L-shaped subpatches:
// row_begin / col_begin); window start = clamp(pos - 3, 0, n - 7) within it.
template <class WA>
FCSG_HD int classify_point(const WA& W, const double* tab, const double* f, long base, int ni, int nj, int i, int j,
                           int rb, int cb, double abs_floor) {
    double s[kMlpIn];
    int cr = 4, cc = 4;
    if (ni - rb >= kMlpIn) {
        int st = i - rb - kMlpIn / 2;
        st = rb + (st < 0 ? 0 : (st > ni - rb - kMlpIn ? ni - rb - kMlpIn : st));
#pragma unroll
        for (int k = 0; k < kMlpIn; ++k) s[k] = f[base + static_cast<long>(j) * ni + st + k];
        cr = classify_stencil(W, tab, s, abs_floor);
    }
    if (nj - cb >= kMlpIn) {
        int st = j - cb - kMlpIn / 2;
        st = cb + (st < 0 ? 0 : (st > nj - cb - kMlpIn ? nj - cb - kMlpIn : st));
#pragma unroll
        for (int k = 0; k < kMlpIn; ++k) s[k] = f[base + static_cast<long>(st + k) * ni + i];
        cc = classify_stencil(W, tab, s, abs_floor);
    }
    return cr < cc ? cr : cc;
}

// phase 0, part 2: tau, mu_hat = c(tau) h_max S on interior points
// (src/viscosity.cpp:240-251); at t=0 also the density class for the smear seed
template <class WA>
FCSG_HD void classify_body(Thr t, int block, int nblocks, const WA& W, double* tab, const EngineDev& E, bool step0) {
    for (int k = t.tid; k < kTanhTable; k += t.nthr) tab[k] = E.tanh_tab[k];
    FCSG_SYNC();
    const long sz = static_cast<long>(E.ni) * E.nj;
    const long step = static_cast<long>(nblocks) * t.nthr;
    for (long p = static_cast<long>(block) * t.nthr + t.tid; p < E.npts; p += step) {
        const long base = (p / sz) * sz;
        const long loc = p - base;
        const int i = static_cast<int>(loc % E.ni), j = static_cast<int>(loc / E.ni);
        const int sub = static_cast<int>(p / sz), ci = E.cut_i[sub], cj = E.cut_j[sub];
        if (i < ci && j < cj) {  // not in the point set of an L-shaped subpatch
            E.tau[p] = 4.0;
            E.mu_hat[p] = 0.0;
            if (step0) E.seed[p] = 0.0;
            continue;
        }
        const int rb = j < cj ? ci : 0, cb = i < ci ? cj : 0;
        const int tau = classify_point(W, tab, E.proxy, base, E.ni, E.nj, i, j, rb, cb, E.abs_floor);
        E.tau[p] = tau;
        E.mu_hat[p] = (E.mask[p] == 1) ? E.visc_c[tau - 1] * E.h_max[p] * E.speed[p] : 0.0;
        if (step0) {
            const int tr = classify_point(W, tab, E.e[0], base, E.ni, E.nj, i, j, rb, cb, E.abs_floor);
            E.seed[p] = (E.mask[p] != 0 && (tau <= 2 || tr <= 2)) ? 1.0 : 0.0;
        }
    }
}

// ---- FC-spectrum ("fallback") classifier -----------------------------------
// Classifier::classify_line's default variant (src/viscosity.cpp:161-208):
// per point, the window of w = min(window, n) values starting at
// clamp(pos - w/2, 0, n - w) is normalised (normalize_stencil, class 4 under
// the guard), continued and transformed (FcOperator::spectrum), and the decay
// exponent s = -slope of the least-squares fit of log |c_k| / n_ext against
// log k over the top quarter of the modes picks the class (tail peak < 2e-4:
// 4; s < 1.6: 1; < 2.6: 2; < 3.6: 3; else 4). Continuation + DFT of the NK
// tail modes is one linear map (build_spectrum_tail): 2 NK multiply-adds per
// window value, no FFT. Window value k sits at f[p0 + k * stride].
template <int NK>
FCSG_HD int spectrum_class(const double* f, long p0, long stride, int w, int n_ext, const double* tab,
                           double abs_floor) {
    double lo = f[p0], hi = lo;
    for (int k = 1; k < w; ++k) {
        const double v = f[p0 + k * stride];
        lo = v < lo ? v : lo;  // std::min(lo, v)
        hi = hi < v ? v : hi;  // std::max(hi, v)
    }
    const double span = hi - lo;
    double scale = fabs(lo);
    scale = scale < fabs(hi) ? fabs(hi) : scale;
    scale = scale < 1e-100 ? 1e-100 : scale;
    if (span <= 1e-13 * scale || span <= abs_floor) return 4;
    double acc[2 * NK];
#pragma unroll
    for (int q = 0; q < 2 * NK; ++q) acc[q] = 0.0;
    for (int k = 0; k < w; ++k) {
        const double x = 2.0 * (f[p0 + k * stride] - lo) / span - 1.0;
        const double* T = tab + k * 2 * NK;
#pragma unroll
        for (int q = 0; q < 2 * NK; ++q) acc[q] = fma(ldg1(T + q), x, acc[q]);
    }
    const double* lx = tab + w * 2 * NK;
    const double sx = ldg1(lx + NK), sxx = ldg1(lx + NK + 1);
    double sy = 0.0, sxy = 0.0, tail_peak = 0.0;
#pragma unroll
    for (int q = 0; q < NK; ++q) {
        const double m = hypot(acc[2 * q], acc[2 * q + 1]) / n_ext;  // std::abs(c_k) / n_ext
        tail_peak = tail_peak < m ? m : tail_peak;
        const double ly = log(m > 1e-300 ? m : 1e-300);
        sy += ly;
        sxy += ldg1(lx + q) * ly;
    }
    const double slope = (NK * sxy - sx * sy) / (NK * sxx - sx * sx);
    const double sd = -slope;
    if (tail_peak < 2e-4) return 4;
    if (sd < 1.6) return 1;
    if (sd < 2.6) return 2;
    if (sd < 3.6) return 3;
    return 4;
}

// one window of a line of n points (n >= kFbMinWindow) around position pos
FCSG_HD int spectrum_line_class(const EngineDev& E, const double* f, long line0, long stride, int n, int pos) {
    const int w = n < E.fb_window ? n : E.fb_window;
    int st = pos - w / 2;
    st = st < 0 ? 0 : (st > n - w ? n - w : st);
    const double* tab = E.fb_tab + E.fb_off[w];
    const int n_ext = w + E.fb_ncont - 1;
    const int nb = n_ext / 2 + 1;
    const long p0 = line0 + st * stride;
    switch (nb - (3 * (nb - 1)) / 4) {
        case 6: return spectrum_class<6>(f, p0, stride, w, n_ext, tab, E.abs_floor);
        case 7: return spectrum_class<7>(f, p0, stride, w, n_ext, tab, E.abs_floor);
        case 8: return spectrum_class<8>(f, p0, stride, w, n_ext, tab, E.abs_floor);
        case 9: return spectrum_class<9>(f, p0, stride, w, n_ext, tab, E.abs_floor);
        case 10: return spectrum_class<10>(f, p0, stride, w, n_ext, tab, E.abs_floor);
        case 11: return spectrum_class<11>(f, p0, stride, w, n_ext, tab, E.abs_floor);
        default: return spectrum_class<12>(f, p0, stride, w, n_ext, tab, E.abs_floor);
    }
}

// Classifier::classify (src/viscosity.cpp:211-238) with the spectrum variant:
// rows (segment [rb, ni)), then columns ([cb, nj)) by min; lines shorter than
// 12 points are class 4
FCSG_HD int spectrum_point(const EngineDev& E, const double* f, long base, int i, int j, int rb, int cb) {
    int cr = 4, cc = 4;
    if (E.fb_window < kFbMinWindow) return 4;  // w = min(window, n) < 12 on every line
    if (E.ni - rb >= kFbMinWindow) cr = spectrum_line_class(E, f, base + static_cast<long>(j) * E.ni + rb, 1, E.ni - rb, i - rb);
    if (E.nj - cb >= kFbMinWindow)
        cc = spectrum_line_class(E, f, base + static_cast<long>(cb) * E.ni + i, E.ni, E.nj - cb, j - cb);
    return cr < cc ? cr : cc;
}

FCSG_HD void classify_spectrum_body(Thr t, int block, int nblocks, const EngineDev& E, bool step0) {
    const long sz = static_cast<long>(E.ni) * E.nj;
    const long step = static_cast<long>(nblocks) * t.nthr;
    for (long p = static_cast<long>(block) * t.nthr + t.tid; p < E.npts; p += step) {
        const long base = (p / sz) * sz;
        const long loc = p - base;
        const int i = static_cast<int>(loc % E.ni), j = static_cast<int>(loc / E.ni);
        const int sub = static_cast<int>(p / sz), ci = E.cut_i[sub], cj = E.cut_j[sub];
        if (i < ci && j < cj) {  // not in the point set of an L-shaped subpatch
            E.tau[p] = 4.0;
            E.mu_hat[p] = 0.0;
            if (step0) E.seed[p] = 0.0;
            continue;
        }
        const int rb = j < cj ? ci : 0, cb = i < ci ? cj : 0;
        const int tau = spectrum_point(E, E.proxy, base, i, j, rb, cb);
        E.tau[p] = tau;
        E.mu_hat[p] = (E.mask[p] == 1) ? E.visc_c[tau - 1] * E.h_max[p] * E.speed[p] : 0.0;
        if (step0) {
            const int tr = spectrum_point(E, E.e[0], base, i, j, rb, cb);
            E.seed[p] = (E.mask[p] != 0 && (tau <= 2 || tr <= 2)) ? 1.0 : 0.0;
        }
    }
}

// ---- classifier on the FP64 tensor cores ----------------------------------
// MlpClassifier::forward (src/viscosity.cpp:108-133) as mma.m8n8k4.f64 tiles:
// a warp classifies 8 stencils at a time -- the row and column windows of 4
// points -- with stencils as the M rows, neurons as N and layer inputs as K.
// Lane (g, t) = (lane / 4, lane % 4) holds A[g][t] (input t of the k-step, of
// stencil g), B[t][g] (weight of neuron g of the n-tile for input t) and
// D[g][2t], D[g][2t+1]. A layer's D fragments are the next layer's A fragments
// when the next layer's inputs are taken in the order
// P(ks, t) = 8 (ks / 2) + 2t + ks % 2 (the neuron this lane holds in its
// register ks), so activations never leave the registers: the permutation is
// folded into the B fragments here. Fragment f of lane l is fr[f * 32 + l].
// Twice a rigorous bound of how far the fast pass's logits can be from
// the exact pass's (tanh_fast within kEps of tanh_tab's values, tanh
// 1-Lipschitz, identical inputs and layer arithmetic otherwise): the error
// of layer l's activations is at most |W_l| (error of layer l-1) + kEps, the
// logits' at most |W_out| times the last one. A fast margin above twice that
// fixes the exact argmax. FCSG_EXACT_TANH=1 disables the fast pass.
double mlp_fast_margin(const std::vector<double>& w) {
    if (std::getenv("FCSG_EXACT_TANH")) return INFINITY;
    constexpr double kEps = 1e-6;  // 2.5x the measured worst case of tanh_fast
    const int rows[kMlpLayers] = {16, 16, 16, 16, 4}, cols[kMlpLayers] = {7, 16, 16, 16, 16};
    std::vector<double> err(16, kEps), nxt;
    int off = rows[0] * cols[0] + rows[0];
    double bound = 0.0;
    for (int l = 1; l < kMlpLayers; ++l) {
        nxt.assign(rows[l], 0.0);
        for (int n = 0; n < rows[l]; ++n) {
            double a = 0.0;
            for (int k = 0; k < cols[l]; ++k) a += std::fabs(w[off + n * cols[l] + k]) * err[k];
            nxt[n] = a * (1.0 + 1e-12) + (l + 1 < kMlpLayers ? kEps : 0.0);
            if (l + 1 == kMlpLayers) bound = std::max(bound, nxt[n]);
        }
        err = nxt;
        off += rows[l] * cols[l] + rows[l];
    }
    if (!std::isfinite(bound)) return INFINITY;
    return 2.0 * bound + 1e-9;
}

std::vector<double> mlp_mma_fragments(const std::vector<double>& w) {
    const int rows[kMlpLayers] = {16, 16, 16, 16, 4}, cols[kMlpLayers] = {7, 16, 16, 16, 16};
    int wo[kMlpLayers], bo[kMlpLayers];
    int off = 0;
    for (int l = 0; l < kMlpLayers; ++l) {
        wo[l] = off;
        off += rows[l] * cols[l];
        bo[l] = off;
        off += rows[l];
    }
    auto W = [&](int l, int n, int k) { return w[wo[l] + n * cols[l] + k]; };
    auto P = [](int ks, int t) { return 8 * (ks >> 1) + 2 * t + (ks & 1); };
    std::vector<double> fr(static_cast<size_t>(kMlpFrags) * 32, 0.0);
    for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        double* f = fr.data() + lane;
        for (int nt = 0; nt < 2; ++nt)
            for (int ks = 0; ks < 2; ++ks) {
                const int k = 4 * ks + t;
                f[(nt * 2 + ks) * 32] = k < kMlpIn ? W(0, 8 * nt + g, k) : 0.0;
            }
        for (int l = 0; l < 3; ++l)
            for (int nt = 0; nt < 2; ++nt)
                for (int ks = 0; ks < 4; ++ks) f[(4 + l * 8 + nt * 4 + ks) * 32] = W(l + 1, 8 * nt + g, P(ks, t));
        for (int ks = 0; ks < 4; ++ks) f[(28 + ks) * 32] = g < kMlpOut ? W(4, g, P(ks, t)) : 0.0;
        for (int L = 0; L < 4; ++L)
            for (int nt = 0; nt < 2; ++nt)
                for (int i = 0; i < 2; ++i) f[(32 + L * 4 + nt * 2 + i) * 32] = w[bo[L] + 8 * nt + 2 * t + i];
        for (int i = 0; i < 2; ++i) f[(48 + i) * 32] = (2 * t + i < kMlpOut) ? w[bo[4] + 2 * t + i] : 0.0;
    }
    return fr;
}

#if FCSG_CUDA
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// Classes 1..4 of NG independent stencil sets (each: the stencil held by this
// lane's quad), returned on all four lanes of the quad; every lane of the warp
// calls. s_a, s_b are window values t and 4 + t (s_b unused for t = 3);
// inactive quads get 4. normalize_stencil's min, max, guard and
// 2 (s - lo) / span - 1 are computed exactly as the reference's
// (src/viscosity.cpp:48-59). The NG sets are interleaved so every thread has
// 4 NG independent tanh chains per layer.
template <int NG, bool FAST>
__device__ void classify_mma(const double* fr, const double* tab, const double* s_a, const double* s_b,
                             const bool* active, double abs_floor, int lane, int* cls, bool* low = nullptr,
                             double fast_margin = 0.0) {
    auto act = [&](double z) {
        if constexpr (FAST) return tanh_fast(z);
        else return tanh_tab(z, tab);
    };
    constexpr unsigned kAll = 0xffffffffu;
    const int t = lane & 3;
    const bool has_b = t < 3;
    double a0[NG], a1[NG];
    bool guard[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        double lo = s_a[g], hi = s_a[g];
        if (has_b) {
            lo = s_b[g] < lo ? s_b[g] : lo;
            hi = s_b[g] > hi ? s_b[g] : hi;
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            const double l2 = __shfl_xor_sync(kAll, lo, o), h2 = __shfl_xor_sync(kAll, hi, o);
            lo = l2 < lo ? l2 : lo;
            hi = h2 > hi ? h2 : hi;
        }
        const double span = hi - lo;
        double scale = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
        scale = scale > 1e-100 ? scale : 1e-100;
        guard[g] = !active[g] || span <= 1e-13 * scale || span <= abs_floor;
        const double sp = guard[g] ? 1.0 : span;
        a0[g] = guard[g] ? 0.0 : 2.0 * (s_a[g] - lo) / sp - 1.0;
        a1[g] = (guard[g] || !has_b) ? 0.0 : 2.0 * (s_b[g] - lo) / sp - 1.0;
    }
    const double* F = fr + lane;
    double h[NG][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        const double b0 = F[(32 + nt * 2) * 32], b1 = F[(33 + nt * 2) * 32];
        const double w0 = F[(nt * 2) * 32], w1 = F[(nt * 2 + 1) * 32];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            double d0 = b0, d1 = b1;
            dmma(d0, d1, a0[g], w0);
            dmma(d0, d1, a1[g], w1);
            h[g][nt * 2] = d0;
            h[g][nt * 2 + 1] = d1;
        }
    }
#pragma unroll
    for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int k = 0; k < 4; ++k) h[g][k] = act(h[g][k]);
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        double z[NG][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const double b0 = F[(36 + l * 4 + nt * 2) * 32], b1 = F[(37 + l * 4 + nt * 2) * 32];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                z[g][nt * 2] = b0;
                z[g][nt * 2 + 1] = b1;
            }
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const double w = F[(4 + l * 8 + nt * 4 + ks) * 32];
#pragma unroll
                for (int g = 0; g < NG; ++g) dmma(z[g][nt * 2], z[g][nt * 2 + 1], h[g][ks], w);
            }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k) h[g][k] = act(z[g][k]);
    }
    double d0[NG], d1[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        d0[g] = F[48 * 32];
        d1[g] = F[49 * 32];
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const double w = F[(28 + ks) * 32];
#pragma unroll
        for (int g = 0; g < NG; ++g) dmma(d0[g], d1[g], h[g][ks], w);
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        // lane t = 0 holds logits 0, 1 and lane t = 1 logits 2, 3
        const double l2 = __shfl_xor_sync(kAll, d0[g], 1), l3 = __shfl_xor_sync(kAll, d1[g], 1);
        int best = 0;  // lowest-index argmax (strict >), without a dynamically indexed array
        double bv = d0[g];
        if (d1[g] > bv) {
            best = 1;
            bv = d1[g];
        }
        if (l2 > bv) {
            best = 2;
            bv = l2;
        }
        if (l3 > bv) best = 3;
        const int c = guard[g] ? 4 : best + 1;
        cls[g] = __shfl_sync(kAll, c, lane & ~3);
        if constexpr (FAST) {
            // margin top1 - top2 of the fast logits (lane t = 0 holds all four)
            const double m1 = fmax(d0[g], d1[g]), n1 = fmin(d0[g], d1[g]);
            const double m2 = fmax(l2, l3), n2 = fmin(l2, l3);
            const double top = fmax(m1, m2), second = fmax(fmin(m1, m2), fmax(n1, n2));
            const bool lw = !guard[g] && !(top - second > fast_margin);
            low[g] = __shfl_sync(kAll, lw, lane & ~3);
        }
    }
}

// classify_mma with the fast tanh, then exactly (tanh_tab) for the whole
// warp when any of its stencils lands within the fast pass's error margin
template <int NG>
__device__ void classify_mma_checked(const double* fr, const double* tab, const double* s_a, const double* s_b,
                                     const bool* active, double abs_floor, int lane, int* cls, double fast_margin) {
    bool low[NG];
    classify_mma<NG, true>(fr, tab, s_a, s_b, active, abs_floor, lane, cls, low, fast_margin);
    bool any = false;
#pragma unroll
    for (int g = 0; g < NG; ++g) any = any || low[g];
    if (__any_sync(0xffffffffu, any)) classify_mma<NG, false>(fr, tab, s_a, s_b, active, abs_floor, lane, cls);
}

// window value k of this lane's stencil (row or column window of point (i, j))
__device__ __forceinline__ double window_at(const double* f, long base, int ni, bool col, int st, int i, int j, int k) {
    return col ? f[base + static_cast<long>(st + k) * ni + i] : f[base + static_cast<long>(j) * ni + st + k];
}

// phase 0, part 2 on the tensor cores: one warp per group of 4 points;
// quads 0-3 hold the row windows, quads 4-7 the column windows
// (Classifier::classify, src/viscosity.cpp:211-251)
constexpr int kMmaThreads = 256;
__global__ void __launch_bounds__(kMmaThreads) classify_mma_kernel(const __grid_constant__ EngineDev E, bool step0) {
    __shared__ double tab[kTanhTable];
    __shared__ double fr[kMlpFrags * 32];
    for (int k = threadIdx.x; k < kTanhTable; k += blockDim.x) tab[k] = E.tanh_tab[k];
    for (int k = threadIdx.x; k < kMlpFrags * 32; k += blockDim.x) fr[k] = E.mlp_frag[k];
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int q = g & 3;
    const bool col = g >= 4;
    const long sz = static_cast<long>(E.ni) * E.nj;
    const long ngroups = (E.npts + 3) / 4;
    const long wstep = static_cast<long>(gridDim.x) * (kMmaThreads / 32);
    // window of this lane's stencil in group grp: point p, validity, start
    struct Win {
        long p, base;
        int i, j, st;
        bool valid, active, inset;
    };
    auto window = [&](long grp) {
        Win w;
        w.p = 4 * grp + q;
        w.valid = w.p < E.npts;
        const unsigned pp = w.valid ? static_cast<unsigned>(w.p) : 0u;
        const unsigned sub = fdiv(E.div_sz, pp);
        const unsigned loc = pp - sub * E.div_sz.d;
        w.j = static_cast<int>(fdiv(E.div_ni, loc));
        w.i = static_cast<int>(loc) - w.j * E.ni;
        w.base = static_cast<long>(sub) * sz;
        const int ci = E.cut_i[sub], cj = E.cut_j[sub];
        w.inset = !(w.i < ci && w.j < cj);  // L-shaped subpatches: row/column segments
        const int beg = col ? (w.i < ci ? cj : 0) : (w.j < cj ? ci : 0);
        const int n = (col ? E.nj : E.ni) - beg;
        w.active = w.valid && w.inset && n >= kMlpIn;
        const int st = (col ? w.j : w.i) - beg - kMlpIn / 2;
        w.st = beg + (st < 0 ? 0 : (st > n - kMlpIn ? n - kMlpIn : st));
        return w;
    };
    auto write = [&](const Win& w, int tau, int tr) {
        if (w.valid && !col && t == 0) {
            const long p = w.p;
            E.tau[p] = tau;
            E.mu_hat[p] = (E.mask[p] == 1) ? E.visc_c[tau - 1] * E.h_max[p] * E.speed[p] : 0.0;
            if (step0) E.seed[p] = (w.inset && E.mask[p] != 0 && (tau <= 2 || tr <= 2)) ? 1.0 : 0.0;
        }
    };
    auto minq = [](int c) {  // min of the row window (quad g) and column window (quad g + 4)
        const int o = __shfl_xor_sync(0xffffffffu, c, 16);
        return c < o ? c : o;
    };
    const long w0 = static_cast<long>(blockIdx.x) * (kMmaThreads / 32) + (threadIdx.x >> 5);
    if (step0) {
        // t = 0: the proxy windows and the density windows of one group together
        for (long grp = w0; grp < ngroups; grp += wstep) {
            const Win w = window(grp);
            double sa[2] = {0.0, 0.0}, sb[2] = {0.0, 0.0};
            const bool act[2] = {w.active, w.active};
            if (w.active) {
                sa[0] = window_at(E.proxy, w.base, E.ni, col, w.st, w.i, w.j, t);
                sa[1] = window_at(E.e[0], w.base, E.ni, col, w.st, w.i, w.j, t);
                if (t < 3) {
                    sb[0] = window_at(E.proxy, w.base, E.ni, col, w.st, w.i, w.j, 4 + t);
                    sb[1] = window_at(E.e[0], w.base, E.ni, col, w.st, w.i, w.j, 4 + t);
                }
            }
            int c[2];
            classify_mma_checked<2>(fr, tab, sa, sb, act, E.abs_floor, lane, c, E.cls_fast_margin);
            write(w, minq(c[0]), minq(c[1]));
        }
        return;
    }
    // steady steps: two groups per iteration
    const long npair = (ngroups + 1) / 2;
    for (long pr = w0; pr < npair; pr += wstep) {
        const Win wa = window(2 * pr), wb = window(2 * pr + 1);
        double sa[2] = {0.0, 0.0}, sb[2] = {0.0, 0.0};
        const bool act[2] = {wa.active, wb.active};
        if (wa.active) {
            sa[0] = window_at(E.proxy, wa.base, E.ni, col, wa.st, wa.i, wa.j, t);
            if (t < 3) sb[0] = window_at(E.proxy, wa.base, E.ni, col, wa.st, wa.i, wa.j, 4 + t);
        }
        if (wb.active) {
            sa[1] = window_at(E.proxy, wb.base, E.ni, col, wb.st, wb.i, wb.j, t);
            if (t < 3) sb[1] = window_at(E.proxy, wb.base, E.ni, col, wb.st, wb.i, wb.j, 4 + t);
        }
        int c[2];
        classify_mma_checked<2>(fr, tab, sa, sb, act, E.abs_floor, lane, c, E.cls_fast_margin);
        write(wa, minq(c[0]), 4);
        write(wb, minq(c[1]), 4);
    }
}
#endif

// t=0 smear mask: box dilation of radius smear_radius (src/runtime.cpp:393-402)
FCSG_HD void dilate_body(Thr t, int block, int nblocks, const EngineDev& E) {
    const long sz = static_cast<long>(E.ni) * E.nj;
    const long step = static_cast<long>(nblocks) * t.nthr;
    const int rad = E.smear_radius;
    for (long p = static_cast<long>(block) * t.nthr + t.tid; p < E.npts; p += step) {
        const long base = (p / sz) * sz;
        const long loc = p - base;
        const int i = static_cast<int>(loc % E.ni), j = static_cast<int>(loc / E.ni);
        double m = 0.0;
        for (int b = (j - rad < 0 ? 0 : j - rad); b <= (j + rad > E.nj - 1 ? E.nj - 1 : j + rad) && m == 0.0; ++b)
            for (int a = (i - rad < 0 ? 0 : i - rad); a <= (i + rad > E.ni - 1 ? E.ni - 1 : i + rad); ++a)
                if (E.seed[base + static_cast<long>(b) * E.ni + a] != 0.0) {
                    m = 1.0;
                    break;
                }
        E.m01[p] = m;
    }
}

// phase 1: viscosity blend + clamp, and the dt_bound_local minimum
FCSG_HD void blend_body(Thr t, int block, int nblocks, const EngineDev& E) {
    const long step = static_cast<long>(nblocks) * t.nthr;
    double best = INFINITY;
    for (long p = static_cast<long>(block) * t.nthr + t.tid; p < E.npts; p += step) {
        double m = E.w_norm[p] * E.mu_hat[p];
        if (E.visc_off) {
            const int e0 = E.visc_off[p], e1 = E.visc_off[p + 1];
            for (int k = e0; k < e1; ++k) m += E.visc_w[k] * E.mu_hat[E.visc_src[k]];
        }
        if (E.vi_off) {  // 6x6 Lagrange of the donor's mu_hat (src/runtime.cpp:359-368)
            const int e0 = E.vi_off[p], e1 = E.vi_off[p + 1];
            for (int k = e0; k < e1; ++k) {
                const double* w = E.vi_w + 13 * static_cast<long>(k);
                const int pitch = E.vi_pitch[k];
                // pitch 0: a donor on another rank evaluated the interpolation
                // into a halo slot
                const double val = pitch ? interp66(E.mu_hat, E.vi_src[k], pitch, w) : E.mu_hat[E.vi_src[k]];
                m += w[12] * val;
            }
        }
        m = m > 0.0 ? m : 0.0;
        E.mu[p] = m;
        if (E.mask[p] == 1) {
            const double h = E.h_min[p];
            const double rate = E.speed[p] / h + m / (h * h);
            if (!(rate > 0.0) || !finite_d(rate)) {
                raise_error_gp(E.sc, 3, p);
            } else {
                const double v = 1.0 / rate;
                best = v < best ? v : best;
            }
        }
    }
#if FCSG_CUDA
    unsigned long long b = dbits(best);
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, b, off);
        b = o < b ? o : b;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(&E.sc->dtmin_bits, b);
#else
    const unsigned long long b = dbits(best);
    if (b < E.sc->dtmin_bits) E.sc->dtmin_bits = b;
#endif
}

// dt = cfl * min dt_local, clipped at T (src/runtime.cpp:492-497)
FCSG_HD void finalize_dt_body(const EngineDev& E) {
    double m;
#if FCSG_CUDA
    m = __longlong_as_double(static_cast<long long>(E.sc->dtmin_bits));
#else
    std::memcpy(&m, &E.sc->dtmin_bits, 8);
#endif
    double dt = E.cfl * m;
    if (E.sc->t + dt > E.T) dt = E.T - E.sc->t;
    E.sc->dt = dt;
}

// t += dt; step += 1 (src/runtime.cpp:505-507); reset the dt minimum
FCSG_HD void advance_body(const EngineDev& E) {
    E.sc->t += E.sc->dt;
    E.sc->step += 1;
    E.sc->dtmin_bits = dbits(INFINITY);
}

// apply_bc_at (src/euler.cpp:105-165); p1/p2 are the first/second neighbours inward
FCSG_HD void apply_bc_at(const EngineDev& E, const BcDev& bc, long p, long p1, long p2, int axis) {
    double* const* e = E.e;
    switch (bc.kind) {
        case 0:
            for (int c = 0; c < 4; ++c) e[c][p] = bc.state[c];
            break;
        case 1: {
            const double rho = e[0][p], mx = e[1][p], my = e[2][p];
            e[3][p] = bc.pressure / kGm1 + 0.5 * (mx * mx + my * my) / rho;
            break;
        }
        case 2: {
            double nx = axis == 0 ? ldg1(E.iq1x + p) : ldg1(E.iq2x + p);
            double ny = axis == 0 ? ldg1(E.iq1y + p) : ldg1(E.iq2y + p);
            const double nn = hypot(nx, ny);
            nx /= nn;
            ny /= nn;
            const double rho = e[0][p], mx = e[1][p], my = e[2][p], En = e[3][p];
            const double pr = kGm1 * (En - 0.5 * (mx * mx + my * my) / rho);
            const double mn = mx * nx + my * ny;
            const double tmx = mx - mn * nx, tmy = my - mn * ny;
            e[1][p] = tmx;
            e[2][p] = tmy;
            e[3][p] = pr / kGm1 + 0.5 * (tmx * tmx + tmy * tmy) / rho;
            break;
        }
        case 3: {
            auto th = [&](long q) {
                const double rho = e[0][q], mx = e[1][q], my = e[2][q], En = e[3][q];
                return kGm1 * (En - 0.5 * (mx * mx + my * my) / rho) / rho;
            };
            const double tt = (4.0 * th(p1) - th(p2)) / 3.0;
            const double rho = e[0][p];
            e[1][p] = 0.0;
            e[2][p] = 0.0;
            e[3][p] = rho * tt / kGm1;
            break;
        }
        case 5:
            for (int c = 0; c < 4; ++c) e[c][p] = (4.0 * e[c][p1] - e[c][p2]) / 3.0;
            break;
        default:
            break;
    }
}

// enforce_bc (src/euler.cpp:167-180): one CTA per subpatch, all row ends, then
// all column ends; a line of an L-shaped subpatch starts at its row/column
// begin (LineInfo::begin)
FCSG_HD void bc_body(Thr t, int sub, const EngineDev& E) {
    const int ni = E.ni, nj = E.nj;
    const int ci = E.cut_i[sub], cj = E.cut_j[sub];
    const long base = static_cast<long>(sub) * ni * nj;
    for (int j = t.tid; j < nj; j += t.nthr) {
        const long r = base + static_cast<long>(j) * ni + (j < cj ? ci : 0);
        const long re = base + static_cast<long>(j) * ni + ni - 1;
        const BcDev& lo = E.bc_row_lo[static_cast<long>(sub) * nj + j];
        const BcDev& hi = E.bc_row_hi[static_cast<long>(sub) * nj + j];
        if (lo.kind >= 0) apply_bc_at(E, lo, r, r + 1, r + 2, 0);
        if (hi.kind >= 0) apply_bc_at(E, hi, re, re - 1, re - 2, 0);
    }
    FCSG_SYNC();
    for (int i = t.tid; i < ni; i += t.nthr) {
        const long c0 = base + static_cast<long>(i < ci ? cj : 0) * ni + i, c1 = base + static_cast<long>(nj - 1) * ni + i;
        const BcDev& lo = E.bc_col_lo[static_cast<long>(sub) * ni + i];
        const BcDev& hi = E.bc_col_hi[static_cast<long>(sub) * ni + i];
        if (lo.kind >= 0) apply_bc_at(E, lo, c0, c0 + ni, c0 + 2 * ni, 1);
        if (hi.kind >= 0) apply_bc_at(E, hi, c1, c1 - ni, c1 - 2 * ni, 1);
    }
}

// phase 6: fringe copies, then 6x6 tensor Lagrange interpolations from
// donor stencils (src/runtime.cpp:433-454). Donors are interior points, never
// written here, so copies and interpolations are independent.
FCSG_HD void exchange_body(Thr t, int block, int nblocks, const EngineDev& E) {
    const long step = static_cast<long>(nblocks) * t.nthr;
    const long n = E.n_x + E.n_xi;
    for (long k = static_cast<long>(block) * t.nthr + t.tid; k < n; k += step) {
        if (k < E.n_x) {
            const long d = E.x_dst[k], s = E.x_src[k];
            for (int c = 0; c < 4; ++c) E.e[c][d] = E.e[c][s];
        } else {
            const long q = k - E.n_x;
            const double* w = E.xi_w + 12 * q;
            const long s0 = E.xi_src[q], d = E.xi_dst[q];
            const int pitch = E.xi_pitch[q];
            for (int c = 0; c < 4; ++c) {
                double val = 0.0;
                for (int b = 0; b < 6; ++b) {
                    const double* row = E.e[c] + s0 + static_cast<long>(b) * pitch;
                    double sa = 0.0;
                    for (int a = 0; a < 6; ++a) sa += w[a] * row[a];
                    val += w[6 + b] * sa;
                }
                E.e[c][d] = val;
            }
        }
    }
}

// halo pack (donor side) / unpack (recipient side) for the multi-rank
// exchange; interpolated entries are evaluated on the donor
FCSG_HD void pack_body(Thr t, int block, int nblocks, const EngineDev& E, int which, const long* idx, long n,
                       HaloPackDev hp, double* buf) {
    const long step = static_cast<long>(nblocks) * t.nthr;
    for (long k = static_cast<long>(block) * t.nthr + t.tid; k < n; k += step) {
        const long p = idx[k];
        if (p >= 0) {
            if (which == 0)
                for (int c = 0; c < 4; ++c) buf[4 * k + c] = E.e[c][p];
            else
                buf[k] = E.mu_hat[p];
        } else {
            const long m = -1 - p;
            const double* w = hp.w + 12 * m;
            if (which == 0)
                for (int c = 0; c < 4; ++c) buf[4 * k + c] = interp66(E.e[c], hp.src[m], hp.pitch[m], w);
            else
                buf[k] = interp66(E.mu_hat, hp.src[m], hp.pitch[m], w);
        }
    }
}
FCSG_HD void unpack_body(Thr t, int block, int nblocks, const EngineDev& E, int which, long n, const double* buf) {
    const long step = static_cast<long>(nblocks) * t.nthr;
    for (long k = static_cast<long>(block) * t.nthr + t.tid; k < n; k += step) {
        const long p = E.npts + k;
        if (which == 0)
            for (int c = 0; c < 4; ++c) E.e[c][p] = buf[4 * k + c];
        else
            E.mu_hat[p] = buf[k];
    }
}

// ---------------------------------------------------------------------------
// kernels and launchers

#if FCSG_CUDA
template <int LB, class Pass, int NE, int NT>
__global__ void __launch_bounds__(NT, (NE > 0 ? 768 : 512) / NT)
    line_pass_kernel(const __grid_constant__ EngineDev E, const __grid_constant__ FcPlanDev pl, int scr_cap, int arg,
                     const LineDesc* desc) {
    extern __shared__ double2 smem[];
    const Pass P(E, arg);
    line_pass<LB, Pass, NE, NT>(Thr{static_cast<int>(threadIdx.x), NT}, blockIdx.x, smem, P, E, pl, scr_cap, desc);
}
__global__ void __launch_bounds__(kThreads) proxy_kernel(const __grid_constant__ EngineDev E) {
    proxy_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, E);
}
constexpr int kClsThreads = 256;
__global__ void __launch_bounds__(kClsThreads) classify_kernel(const __grid_constant__ EngineDev E, bool step0) {
    __shared__ double tab[kTanhTable];
    classify_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, MlpW{}, tab, E,
                  step0);
}
__global__ void __launch_bounds__(kThreads) dilate_kernel(const __grid_constant__ EngineDev E) {
    dilate_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, E);
}
__global__ void __launch_bounds__(kThreads) blend_kernel(const __grid_constant__ EngineDev E) {
    blend_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, E);
}
__global__ void __launch_bounds__(kThreads)
    pack_kernel(const __grid_constant__ EngineDev E, int which, const long* idx, long n, HaloPackDev hp, double* buf) {
    pack_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, E, which, idx, n,
              hp, buf);
}
__global__ void __launch_bounds__(kThreads)
    unpack_kernel(const __grid_constant__ EngineDev E, int which, long n, const double* buf) {
    unpack_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, E, which, n,
                buf);
}
__global__ void finalize_dt_kernel(const __grid_constant__ EngineDev E) { finalize_dt_body(E); }
__global__ void advance_kernel(const __grid_constant__ EngineDev E) { advance_body(E); }
__global__ void __launch_bounds__(kThreads) bc_kernel(const __grid_constant__ EngineDev E) {
    bc_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, E);
}
__global__ void __launch_bounds__(kThreads) exchange_kernel(const __grid_constant__ EngineDev E) {
    exchange_body(Thr{static_cast<int>(threadIdx.x), static_cast<int>(blockDim.x)}, blockIdx.x, gridDim.x, E);
}
#endif

namespace {

constexpr int kLB = 8;  // lines per CTA in the step passes

// CTA size of a pass's compile-time-plan kernel (Pass::kNT if set, else 256)
template <class P, class = void>
struct NtOf {
    static constexpr int v = kThreads;
};
template <class P>
struct NtOf<P, std::void_t<decltype(P::kNT)>> {
    static constexpr int v = P::kNT;
};

int grid_for(long n) {
    long g = (n + kThreads - 1) / kThreads;
    if (g > 148 * 16) g = 148 * 16;
    return static_cast<int>(g < 1 ? 1 : g);
}

#if FCSG_CUDA
template <class Pass, int NE, int NT, int LB>
void launch_line_pass(int nblk, size_t smem, int arg, const EngineDev& E, const FcPlanDev& pl, int scr_cap,
                      const LineDesc* desc, cudaStream_t s) {
    auto k = line_pass_kernel<LB, Pass, NE, NT>;
    static unsigned long long done = 0;  // once per instantiation and device
    if (dev::first_on_device(&done)) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    k<<<nblk, NT, smem, s>>>(E, pl, scr_cap, arg, desc);
}
#endif

bool use_warp_passes() {
    static const bool on = std::getenv("FCSG_NO_WARP_PASSES") == nullptr;
    return on;
}

}  // namespace

size_t line_pass_smem(const FcPlanDev& pl, int scr_cap, int slots, int lb) {
    return (static_cast<size_t>(pl.n_ext) * lb + scr_cap + table_slots_host(pl)) * sizeof(double2) +
           static_cast<size_t>(slots) * pl.n * lb * sizeof(double);
}

bool line_pass_smem_fits(const FcPlanDev& pl, int scr_cap) {
    // the widest staging area of any pass (PassB, PassGB: 7 slots), 2 lines per CTA
    return line_pass_smem(pl, scr_cap, 7, 2) <= kMaxLinePassSmem;
}

namespace {

// One line set of one group view. Lines per CTA: Pass::kLB for the
// compile-time plans (4 where a large staging area would otherwise cost
// occupancy: three 256-thread CTAs per SM fit in shared memory), kLB for the
// generic plan.
template <class Pass>
void run_line_pass(int arg, const EngineDev& E, const LineSet& L, void* stream) {
    constexpr int kSlots = Pass::kStage + Pass::kStash;
    const FcPlanDev& pl = L.pl;
    int scr_cap = L.scr;
    const int nlines = Pass::kRows ? E.nj : E.ni;
    // the compile-time plans assume the reference operator (n_cont 25, degree 2)
    const bool ref_op = pl.n_gap == 24 && pl.dp1 == 3;
    // compile-time plans: 280 (N = 256), 536 (512), 171 (147, the config-3
    // annulus), and the config-4 C1 patch's lengths 94 (N = 70), 102 (78),
    // 103 (79), 163 (139); prime last radices (17, 19, 47, 67, 103, 163) on DMMA
    auto is_ct = [](int ne) {
        return ne == 280 || ne == 536 || ne == 171 || ne == 94 || ne == 102 || ne == 103 || ne == 163;
    };
    const bool ct = ref_op && is_ct(pl.n_ext);
    // the emulation runs the same lines-per-CTA as the GPU (one emulated
    // thread), so it covers the line ownership of every launch shape
    constexpr int kCtLB = Pass::kLB;
    static_assert(kCtLB == 2 || kCtLB == 4 || kCtLB == 8, "descriptor lists exist for 2, 4, 8 lines per CTA");
    // generic plan: 8 lines per CTA, or 2 when 8 would not fit the shared
    // memory of one SM (long lines; Engine::finalize rejects lines for which
    // even 2 do not fit, line_pass_smem_fits)
    const bool narrow = !ct && line_pass_smem(pl, scr_cap, kSlots, kLB) > kMaxLinePassSmem;
    const int lb = ct ? kCtLB : (narrow ? 2 : kLB);
    const LineDesc* desc = L.desc[desc_index(lb)];
    if (ct) scr_cap = std::max(scr_cap, ct_scratch_slots(pl.n_ext, lb));  // prime middles: full scratch
    const int nblk = desc ? L.n[desc_index(lb)] : E.S * ((nlines + lb - 1) / lb);
    if (nblk == 0) return;
    const size_t smem = line_pass_smem(pl, scr_cap, kSlots, lb);
#if FCSG_CUDA
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    constexpr int kNT = NtOf<Pass>::v;
    if (ct && pl.n_ext == 280) launch_line_pass<Pass, 280, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (ct && pl.n_ext == 536) launch_line_pass<Pass, 536, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (ct && pl.n_ext == 171) launch_line_pass<Pass, 171, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (ct && pl.n_ext == 94) launch_line_pass<Pass, 94, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (ct && pl.n_ext == 102) launch_line_pass<Pass, 102, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (ct && pl.n_ext == 103) launch_line_pass<Pass, 103, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (ct) launch_line_pass<Pass, 163, kNT, kCtLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else if (narrow) launch_line_pass<Pass, 0, kThreads, 2>(nblk, smem, arg, E, pl, scr_cap, desc, s);
    else launch_line_pass<Pass, 0, kThreads, kLB>(nblk, smem, arg, E, pl, scr_cap, desc, s);
#else
    (void)stream;
    const Pass P(E, arg);
    std::vector<double2> sm(smem / sizeof(double2) + 1);
    for (int b = 0; b < nblk; ++b) {
        if (ct && pl.n_ext == 280) line_pass<kCtLB, Pass, 280, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (ct && pl.n_ext == 536) line_pass<kCtLB, Pass, 536, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (ct && pl.n_ext == 171) line_pass<kCtLB, Pass, 171, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (ct && pl.n_ext == 94) line_pass<kCtLB, Pass, 94, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (ct && pl.n_ext == 102) line_pass<kCtLB, Pass, 102, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (ct && pl.n_ext == 103) line_pass<kCtLB, Pass, 103, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (ct) line_pass<kCtLB, Pass, 163, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else if (narrow) line_pass<2, Pass, 0, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
        else line_pass<kLB, Pass, 0, 1>(Thr{0, 1}, b, sm.data(), P, E, pl, scr_cap, desc);
    }
#endif
}

template <class Pass>
void run_rows(int arg, const GroupLaunch& g, void* stream) {
    for (const LineSet& L : g.rows) run_line_pass<Pass>(arg, g.E, L, stream);
}
template <class Pass>
void run_cols(int arg, const GroupLaunch& g, void* stream) {
    for (const LineSet& L : g.cols) run_line_pass<Pass>(arg, g.E, L, stream);
}

}  // namespace

int step_scr_cap(const FcPlanDev& pl) {
    int cap = 0;
    for (int s = 0; s < pl.nstages; ++s) {
        const int p = pl.radix[s];
        if (!radix_in_registers(p)) {
            const int per = p * 16;  // largest LB of any instantiation
            const int k = kThreads / per > 1 ? kThreads / per : 1;
            cap = cap > per * k ? cap : per * k;
        }
    }
    return cap;
}

void launch_proxy(const EngineDev& Eall, void* stream) {
#if FCSG_CUDA
    proxy_kernel<<<grid_for(Eall.npts), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(Eall);
#else
    (void)stream;
    proxy_body(Thr{0, 1}, 0, 1, Eall);
#endif
}

#if FCSG_CUDA
constexpr int kSpecThreads = 128;
__global__ void __launch_bounds__(kSpecThreads) classify_spectrum_kernel(const __grid_constant__ EngineDev E, bool step0) {
    classify_spectrum_body(Thr{static_cast<int>(threadIdx.x), kSpecThreads}, blockIdx.x, gridDim.x, E, step0);
}
#endif

#if FCSG_CUDA
// The fallback classifier on the FP64 tensor cores, for 32-point windows (the
// default) in groups without L-shaped subpatches and with lines of >= 32
// points: as classify_mma_kernel, a warp takes the row and column windows of
// 4 points (quad g: window g, lane t: window values t, t+4, ..., t+28); the
// window x (8 rows of A per tile) times the 32 x 16 tail matrix (B, held in
// registers for the whole kernel) gives, in lane t's accumulators, Re/Im of
// tail modes t and t + 4 of its window: 16 DMMA.884 per 8 windows instead of
// 512 multiply-adds per window. The fit's sums are reduced over the quad.
constexpr int kSpecMmaThreads = 256;
__global__ void __launch_bounds__(kSpecMmaThreads) classify_spectrum_mma_kernel(const __grid_constant__ EngineDev E,
                                                                                 bool step0) {
    constexpr int W = 32, NK = 8;
    constexpr unsigned kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, q = g & 3;
    const bool col = g >= 4;
    const double* T = E.fb_tab + E.fb_off[W];
    double bf[2][8];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) bf[nt][ks] = ldg1(T + (4 * ks + t) * 2 * NK + 8 * nt + g);
    const double* lx = T + W * 2 * NK;
    const double lx0 = ldg1(lx + t), lx1 = ldg1(lx + 4 + t), sx = ldg1(lx + NK), sxx = ldg1(lx + NK + 1);
    const double n_ext = static_cast<double>(W + E.fb_ncont - 1);
    const double ln_ext = log(n_ext);
    const double kLogFloor = log(1e-300);
    const long sz = static_cast<long>(E.ni) * E.nj;
    const long ngroups = (E.npts + 3) / 4;
    const long wstep = static_cast<long>(gridDim.x) * (kSpecMmaThreads / 32);
    for (long grp = static_cast<long>(blockIdx.x) * (kSpecMmaThreads / 32) + (threadIdx.x >> 5); grp < ngroups;
         grp += wstep) {
        const long p = 4 * grp + q;
        const bool valid = p < E.npts;
        const unsigned pp = valid ? static_cast<unsigned>(p) : 0u;
        const unsigned sub = fdiv(E.div_sz, pp);
        const unsigned loc = pp - sub * E.div_sz.d;
        const int j = static_cast<int>(fdiv(E.div_ni, loc));
        const int i = static_cast<int>(loc) - j * E.ni;
        const long base = static_cast<long>(sub) * sz;
        const int n = col ? E.nj : E.ni, pos = col ? j : i;
        int st = pos - W / 2;
        st = st < 0 ? 0 : (st > n - W ? n - W : st);
        const long stride = col ? E.ni : 1;
        const long p0 = col ? base + static_cast<long>(st) * E.ni + i : base + static_cast<long>(j) * E.ni + st;
        int cls[2] = {4, 4};
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            if (f == 1 && !step0) break;
            const double* src = f == 0 ? E.proxy : E.e[0];
            double v[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) v[ks] = valid ? src[p0 + (4 * ks + t) * stride] : 0.0;
            double lo = v[0], hi = v[0];
#pragma unroll
            for (int ks = 1; ks < 8; ++ks) {
                lo = v[ks] < lo ? v[ks] : lo;
                hi = hi < v[ks] ? v[ks] : hi;
            }
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                const double l2 = __shfl_xor_sync(kAll, lo, o), h2 = __shfl_xor_sync(kAll, hi, o);
                lo = l2 < lo ? l2 : lo;
                hi = hi < h2 ? h2 : hi;
            }
            const double span = hi - lo;
            double scale = fabs(lo);
            scale = scale < fabs(hi) ? fabs(hi) : scale;
            scale = scale < 1e-100 ? 1e-100 : scale;
            const bool guard = !valid || span <= 1e-13 * scale || span <= E.abs_floor;
            // 2 (v - lo) / span - 1 as (v - lo) (2 / span) - 1: one division per
            // window (<= 1 ulp per value against normalize_stencil, far below
            // the spectrum's own round-off)
            const double r2 = 2.0 / (guard ? 1.0 : span);
            double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const double a = guard ? 0.0 : fma(v[ks] - lo, r2, -1.0);
                dmma(d[0][0], d[0][1], a, bf[0][ks]);
                dmma(d[1][0], d[1][1], a, bf[1][ks]);
            }
            // log(|c_k| / n_ext) = 0.5 log(|c_k|^2) - log(n_ext); |c_k| = 0
            // takes the reference's floor log(1e-300); the tail peak needs one
            // square root (of the largest |c_k|^2 of the window)
            const double s0 = fma(d[0][0], d[0][0], d[0][1] * d[0][1]);
            const double s1 = fma(d[1][0], d[1][0], d[1][1] * d[1][1]);
            const double ly0 = s0 > 0.0 ? fma(0.5, log(s0), -ln_ext) : kLogFloor;
            const double ly1 = s1 > 0.0 ? fma(0.5, log(s1), -ln_ext) : kLogFloor;
            double sy = ly0 + ly1, sxy = lx0 * ly0 + lx1 * ly1, smax = s0 < s1 ? s1 : s0;
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                sy += __shfl_xor_sync(kAll, sy, o);
                sxy += __shfl_xor_sync(kAll, sxy, o);
                const double p2 = __shfl_xor_sync(kAll, smax, o);
                smax = smax < p2 ? p2 : smax;
            }
            const double pk = sqrt(smax) / n_ext;
            const double sd = -((NK * sxy - sx * sy) / (NK * sxx - sx * sx));
            int c = 4;
            if (!(pk < 2e-4)) c = sd < 1.6 ? 1 : (sd < 2.6 ? 2 : (sd < 3.6 ? 3 : 4));
            cls[f] = guard ? 4 : c;
        }
        // min of the row window (quad g) and the column window (quad g + 4)
        const int tau = min(cls[0], __shfl_xor_sync(kAll, cls[0], 16));
        const int tr = min(cls[1], __shfl_xor_sync(kAll, cls[1], 16));
        if (valid && !col && t == 0) {
            E.tau[p] = tau;
            E.mu_hat[p] = (E.mask[p] == 1) ? E.visc_c[tau - 1] * E.h_max[p] * E.speed[p] : 0.0;
            if (step0) E.seed[p] = (E.mask[p] != 0 && (tau <= 2 || tr <= 2)) ? 1.0 : 0.0;
        }
    }
}
#endif

void launch_classify(const EngineDev& Eall, const std::vector<GroupLaunch>& G, bool step0, void* stream) {
    if (Eall.cls_variant == 1) {  // FC-spectrum classifier
#if FCSG_CUDA
        static const bool scalar = [] {
            const char* v = std::getenv("FCSG_CLASSIFIER");
            return v && std::string(v) == "scalar";
        }();
        for (const GroupLaunch& g : G) {
            // tensor-core path: 32-point windows, full lines of >= 32 points
            const bool rect = g.rows.size() == 1 && g.rows[0].desc[0] == nullptr;
            if (!scalar && rect && g.E.fb_window == 32 && g.E.ni >= 32 && g.E.nj >= 32) {
                long n = ((g.E.npts + 3) / 4 + kSpecMmaThreads / 32 - 1) / (kSpecMmaThreads / 32);
                n = n > 148 * 8 ? 148 * 8 : (n < 1 ? 1 : n);
                classify_spectrum_mma_kernel<<<static_cast<int>(n), kSpecMmaThreads, 0,
                                               static_cast<cudaStream_t>(stream)>>>(g.E, step0);
                continue;
            }
            long n = (g.E.npts + kSpecThreads - 1) / kSpecThreads;
            n = n > 148 * 32 ? 148 * 32 : (n < 1 ? 1 : n);
            classify_spectrum_kernel<<<static_cast<int>(n), kSpecThreads, 0, static_cast<cudaStream_t>(stream)>>>(g.E,
                                                                                                                  step0);
        }
#else
        (void)stream;
        for (const GroupLaunch& g : G) classify_spectrum_body(Thr{0, 1}, 0, 1, g.E, step0);
#endif
        return;
    }
#if FCSG_CUDA
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static const bool scalar = [] {
        const char* v = std::getenv("FCSG_CLASSIFIER");
        return v && std::string(v) == "scalar";
    }();
    if (scalar) cudaMemcpyToSymbolAsync(c_mlp, Eall.mlp, kMlpWeights * sizeof(double), 0, cudaMemcpyDeviceToDevice, s);
    static const bool no_f32 = std::getenv("FCSG_CLASSIFIER") != nullptr || std::getenv("FCSG_EXACT_TANH") != nullptr;
    for (const GroupLaunch& g : G) {
        const EngineDev& E = g.E;
        if (!step0 && g.w32 && !no_f32) {  // steady steps: FP32 screen + exact FP64 where it is not conclusive
            launch_classify_f32(E, *g.w32, stream);
            continue;
        }
        if (scalar) {  // CUDA-core classifier (constant-bank weights), for comparison
            long n = (E.npts + kClsThreads - 1) / kClsThreads;
            n = n > 148 * 24 ? 148 * 24 : n;
            classify_kernel<<<static_cast<int>(n), kClsThreads, 0, s>>>(E, step0);
        } else {
            long n = ((E.npts + 3) / 4 + kMmaThreads / 32 - 1) / (kMmaThreads / 32);
            n = n > 148 * 16 ? 148 * 16 : n;  // 4 waves of 4 x 148: -2% against 2 (tail)
            classify_mma_kernel<<<static_cast<int>(n < 1 ? 1 : n), kMmaThreads, 0, s>>>(E, step0);
        }
    }
#else
    (void)stream;
    (void)Eall;
    std::vector<double> tab(kTanhTable);
    for (const GroupLaunch& g : G) classify_body(Thr{0, 1}, 0, 1, MlpW{g.E.mlp}, tab.data(), g.E, step0);
#endif
}

void launch_phase0(const EngineDev& Eall, const std::vector<GroupLaunch>& G, bool step0, void* stream) {
    launch_proxy(Eall, stream);
    launch_classify(Eall, G, step0, stream);
}

void launch_phase1(const EngineDev& Eall, void* stream) {
#if FCSG_CUDA
    blend_kernel<<<grid_for(Eall.npts), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(Eall);
#else
    (void)stream;
    blend_body(Thr{0, 1}, 0, 1, Eall);
#endif
}

void launch_phase2(const std::vector<GroupLaunch>& G, bool step0, void* stream) {
    for (const GroupLaunch& g : G) {
        if (step0) {
#if FCSG_CUDA
            dilate_kernel<<<grid_for(g.E.npts), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(g.E);
#else
            dilate_body(Thr{0, 1}, 0, 1, g.E);
#endif
        }
        // steady steps on whole 256-point lines: the warp transform
        const bool full = g.rows.size() == 1 && g.cols.size() == 1 && g.rows[0].desc[0] == nullptr;
        if (!step0 && full && wpass_applies(g.E, g.rows[0].pl, true) && wpass_applies(g.E, g.cols[0].pl, false) &&
            use_warp_passes()) {
            launch_wfilter(g.E, g.rows[0].pl, true, stream);
            launch_wfilter(g.E, g.cols[0].pl, false, stream);
            continue;
        }
        run_rows<PassFR>(step0 ? 1 : 0, g, stream);
        run_cols<PassFC>(step0 ? 1 : 0, g, stream);
    }
}

void launch_stage(const std::vector<GroupLaunch>& G, int stage, void* stream) {
    launch_pass_a(G, stream);
    launch_pass_b(G, stage, stream);
    launch_pass_c(G, stage, stream);
}

// Groups of whole 256 x 256-point Cartesian subpatches in the flux form run
// the warp passes on the prime-factor transform (wpass.cu): pass Y first
// (columns, tA = iq2y D2 Phi_y), then pass X (rows: rhs and the SSPRK update)
static bool warp_group(const GroupLaunch& g) {
    return g.E.cartesian && !g.E.reference_order && g.rows.size() == 1 && g.cols.size() == 1 &&
           g.rows[0].desc[0] == nullptr && wpass_applies(g.E, g.rows[0].pl, true) &&
           wpass_applies(g.E, g.cols[0].pl, false) && use_warp_passes();
}

// flux form: Cartesian X, Y (no third pass) -- warp groups: Y, X; general
// GA, GB, C. reference order: A', B', C' / A, B, C.
void launch_pass_a(const std::vector<GroupLaunch>& G, void* stream) {
    for (const GroupLaunch& g : G) {
        if (warp_group(g)) {
            launch_wpass(g.E, g.cols[0].pl, false, 0, stream);
            continue;
        }
        if (g.E.reference_order) {
            if (g.E.cartesian) run_rows<PassAc>(0, g, stream);
            else run_rows<PassA>(0, g, stream);
        } else {
            if (g.E.cartesian) run_rows<PassXc>(0, g, stream);
            else run_rows<PassGA>(0, g, stream);
        }
    }
}
void launch_pass_b(const std::vector<GroupLaunch>& G, int stage, void* stream) {
    for (const GroupLaunch& g : G) {
        if (warp_group(g)) {
            launch_wpass(g.E, g.rows[0].pl, true, stage, stream);
            continue;
        }
        if (g.E.reference_order) {
            if (g.E.cartesian) run_cols<PassBc>(0, g, stream);
            else run_cols<PassB>(0, g, stream);
        } else {
            if (g.E.cartesian) run_cols<PassYc>(stage, g, stream);
            else run_cols<PassGB>(0, g, stream);
        }
    }
}
void launch_pass_c(const std::vector<GroupLaunch>& G, int stage, void* stream) {
    for (const GroupLaunch& g : G) {
        if (g.E.reference_order) {
            if (g.E.cartesian) run_rows<PassCc>(stage, g, stream);
            else run_rows<PassC>(stage, g, stream);
        } else if (!g.E.cartesian) {
            run_rows<PassC>(stage, g, stream);
        }
    }
}

void launch_gradient(const std::vector<GroupLaunch>& G, int comp, void* stream) {
    for (const GroupLaunch& g : G) {
        run_rows<PassDiagR>(comp, g, stream);
        run_cols<PassDiagC>(comp, g, stream);
    }
}

// window_quadrature (src/workbench.cpp:187-210), one block per storage slot
FCSG_HD double integrand(const EngineDev& E, int comp, long p) { return comp < 0 ? 1.0 : E.e[comp][p]; }
#if FCSG_CUDA
constexpr int kQuadThreads = 256;
__global__ void __launch_bounds__(kQuadThreads) integrals_kernel(const __grid_constant__ EngineDev E, int comp,
                                                                  const long* slot_off, double* out) {
    __shared__ double red[kQuadThreads];
    const long p0 = slot_off[blockIdx.x], p1 = slot_off[blockIdx.x + 1];
    double acc = 0.0;
    for (long p = p0 + threadIdx.x; p < p1; p += kQuadThreads) acc += E.wq[p] * integrand(E, comp, p);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int h = kQuadThreads / 2; h > 0; h >>= 1) {
        if (static_cast<int>(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}
__global__ void sample_kernel(const double* f, long n, const long* base, const int* pitch, const double* fu,
                              const double* fv, double* out) {
    for (long k = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<long>(gridDim.x) * blockDim.x) {
        const long b = base[k];
        if (b < 0) {
            out[k] = 0.0;
            continue;
        }
        const long w = pitch[k];
        const double u = fu[k], v = fv[k];
        // src/workbench.cpp:293-294, same expression order
        out[k] = (1 - u) * (1 - v) * f[b] + u * (1 - v) * f[b + 1] + (1 - u) * v * f[b + w] + u * v * f[b + w + 1];
    }
}
#endif

void launch_integrals(const EngineDev& Eall, int comp, const long* slot_off, int S, double* out, void* stream) {
#if FCSG_CUDA
    integrals_kernel<<<S, kQuadThreads, 0, static_cast<cudaStream_t>(stream)>>>(Eall, comp, slot_off, out);
#else
    (void)stream;
    for (int s = 0; s < S; ++s) {
        double acc = 0.0;
        for (long p = slot_off[s]; p < slot_off[s + 1]; ++p) acc += Eall.wq[p] * integrand(Eall, comp, p);
        out[s] = acc;
    }
#endif
}

void launch_sample(const double* f, long n, const long* base, const int* pitch, const double* fu, const double* fv,
                   double* out, void* stream) {
    if (n <= 0) return;
#if FCSG_CUDA
    long g = (n + 255) / 256;
    g = g > 148 * 16 ? 148 * 16 : g;
    sample_kernel<<<static_cast<int>(g), 256, 0, static_cast<cudaStream_t>(stream)>>>(f, n, base, pitch, fu, fv, out);
#else
    (void)stream;
    for (long k = 0; k < n; ++k) {
        const long b = base[k];
        if (b < 0) {
            out[k] = 0.0;
            continue;
        }
        const long w = pitch[k];
        const double u = fu[k], v = fv[k];
        out[k] = (1 - u) * (1 - v) * f[b] + u * (1 - v) * f[b + 1] + (1 - u) * v * f[b + w] + u * v * f[b + w + 1];
    }
#endif
}

int stage_launches(const std::vector<GroupLaunch>& G) {
    int n = 0;
    for (const GroupLaunch& g : G) {
        const int nr = static_cast<int>(g.rows.size()), nc = static_cast<int>(g.cols.size());
        n += (g.E.cartesian && !g.E.reference_order) ? nr + nc : 2 * nr + nc;
    }
    return n;
}

int launches_per_step(const std::vector<GroupLaunch>& G) {
    // proxy, blend, dt, advance; per group classify, bc x 6, filter rows + cols;
    // per stage the passes and one exchange
    int n = 4 + 5;
    for (const GroupLaunch& g : G) n += 1 + 6 + static_cast<int>(g.rows.size() + g.cols.size());
    return n + 5 * stage_launches(G);
}

void launch_bc(const std::vector<GroupLaunch>& G, void* stream) {
    for (const GroupLaunch& g : G) {
#if FCSG_CUDA
        bc_kernel<<<g.E.S, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(g.E);
#else
        (void)stream;
        for (int s = 0; s < g.E.S; ++s) bc_body(Thr{0, 1}, s, g.E);
#endif
    }
}

void launch_exchange(const EngineDev& E, void* stream) {
    if (E.n_x + E.n_xi == 0) return;
#if FCSG_CUDA
    exchange_kernel<<<grid_for(E.n_x + E.n_xi), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(E);
#else
    (void)stream;
    exchange_body(Thr{0, 1}, 0, 1, E);
#endif
}

void launch_finalize_dt(const EngineDev& E, void* stream) {
#if FCSG_CUDA
    finalize_dt_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(E);
#else
    (void)stream;
    finalize_dt_body(E);
#endif
}

void launch_advance(const EngineDev& E, void* stream) {
#if FCSG_CUDA
    advance_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(E);
#else
    (void)stream;
    advance_body(E);
#endif
}

void launch_pack(const EngineDev& E, int which, const long* idx, long n, const HaloPackDev& hp, double* buf,
                 void* stream) {
    if (n <= 0) return;
#if FCSG_CUDA
    pack_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(E, which, idx, n, hp, buf);
#else
    (void)stream;
    pack_body(Thr{0, 1}, 0, 1, E, which, idx, n, hp, buf);
#endif
}

void launch_unpack(const EngineDev& E, int which, long n, const double* buf, void* stream) {
    if (n <= 0) return;
#if FCSG_CUDA
    unpack_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(E, which, n, buf);
#else
    (void)stream;
    unpack_body(Thr{0, 1}, 0, 1, E, which, n, buf);
#endif
}

}  // namespace fcsg
