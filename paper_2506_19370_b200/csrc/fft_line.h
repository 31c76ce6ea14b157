// Shared-memory FC line transform: continuation -> mixed-radix FFT -> spectral
// multiplier -> inverse FFT, for a batch of LB complex lines held in shared
// memory as buf[pos * LB + line] (line index fastest, no padding: every pass
// maps thread w to (line w % LB, position or butterfly w / LB), so 8
// consecutive lanes -- one 128-byte shared-memory wavefront of 16-byte
// accesses -- touch 8 consecutive slots: conflict-free, and one twiddle per
// butterfly is a broadcast).
//
// Restates FcOperator::derivative / apply_profile (src/fc_core.cpp:221-238,
// 257-297) for TWO real lines at once: the complex line z = a + i b is
// transformed with a full complex DFT of length n_ext; because every
// multiplier used by the reference is Hermitian-consistent (i*w*k_signed with
// the even-n Nyquist bin zeroed for odd derivatives; real-even for the second
// derivative and both filter profiles), Re/Im of the result are exactly the
// reference's c2r outputs for a and b.
//
// Forward: in-place decimation-in-frequency (natural order in, digit-reversed
// out); the multiplier table is stored in that digit-reversed order; inverse:
// in-place decimation-in-time (digit-reversed in, natural out, unnormalised,
// as FFTW's c2r). No permutation pass is needed.
#pragma once

#include "fcsg_common.h"

namespace fcsg {

// operator tables are read through plain loads: in the kernels they live in
// shared memory (stage_tables), elsewhere in global memory
FCSG_HD double2 ld2(const double2* p) { return *p; }
FCSG_HD double ld1(const double* p) { return *p; }

// read-only global data through the non-coherent path
FCSG_HD double ldg1(const double* p) {
#if FCSG_CUDA && defined(__CUDA_ARCH__)
    return __ldg(p);
#else
    return *p;
#endif
}

FCSG_HD double2 ldg2(const double2* p) {
#if FCSG_CUDA && defined(__CUDA_ARCH__)
    return __ldg(p);
#else
    return *p;
#endif
}

// shared-memory slots (double2) for the staged tables of one operator
FCSG_HD int table_slots(const FcPlanDev& pl) { return 2 * pl.n_ext + (pl.n_gap * pl.dp1 + 1) / 2; }
#if FCSG_CUDA
__host__
#endif
inline int table_slots_host(const FcPlanDev& pl) { return 2 * pl.n_ext + (pl.n_gap * pl.dp1 + 1) / 2; }

// Copy the twiddles, the multiplier table of `mode` and the blend matrix into
// shared memory (tab, table_slots() slots) once per CTA, so no stage waits on
// a first-touch global load; returns a plan pointing at the copies (mult is
// offset so that plan.mult + (mode-1)*n_ext is the staged table). The caller
// synchronises before the first transform.
FCSG_HD FcPlanDev stage_tables(Thr t, const FcPlanDev& pl, int mode, double2* tab) {
    const int n = pl.n_ext;
    const double2* msrc = pl.mult + (mode - 1) * n;
    for (int k = t.tid; k < n; k += t.nthr) {
        tab[k] = pl.tw[k];
        tab[n + k] = msrc[k];
    }
    double* sb = reinterpret_cast<double*>(tab + 2 * n);
    for (int k = t.tid; k < pl.n_gap * pl.dp1; k += t.nthr) sb[k] = pl.blend[k];
    FcPlanDev q = pl;
    q.tw = tab;
    q.mult = tab + n - (mode - 1) * n;
    q.blend = sb;
    return q;
}

// ---------------------------------------------------------------------------
// small DFTs in registers: y_q = sum_r x_r exp(-+ 2 pi i r q / P)

template <bool INV>
FCSG_HD void dft2(double2* x) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
}

// multiply by -i (forward) or +i (inverse)
template <bool INV>
FCSG_HD double2 mul_mi(double2 v) {
    return INV ? mk2(-v.y, v.x) : mk2(v.y, -v.x);
}

template <bool INV>
FCSG_HD void dft4v(double2& x0, double2& x1, double2& x2, double2& x3) {
    const double2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_mi<INV>(csub(x1, x3));
    x0 = cadd(t0, t2);
    x2 = csub(t0, t2);
    x1 = cadd(t1, t3);
    x3 = csub(t1, t3);
}

template <bool INV>
FCSG_HD void dft4(double2* x) {
    dft4v<INV>(x[0], x[1], x[2], x[3]);
}

template <bool INV>
FCSG_HD void dft8(double2* x) {
    double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
    double2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
    dft4v<INV>(e0, e1, e2, e3);
    dft4v<INV>(o0, o1, o2, o3);
    const double h = 0.70710678118654752440;
    // w8^q = exp(-+ i pi q / 4)
    const double2 w1o = INV ? mk2(h * (o1.x - o1.y), h * (o1.x + o1.y)) : mk2(h * (o1.x + o1.y), h * (o1.y - o1.x));
    const double2 w2o = mul_mi<INV>(o2);
    const double2 w3o = INV ? mk2(-h * (o3.x + o3.y), h * (o3.x - o3.y)) : mk2(h * (o3.y - o3.x), -h * (o3.x + o3.y));
    x[0] = cadd(e0, o0);
    x[4] = csub(e0, o0);
    x[1] = cadd(e1, w1o);
    x[5] = csub(e1, w1o);
    x[2] = cadd(e2, w2o);
    x[6] = csub(e2, w2o);
    x[3] = cadd(e3, w3o);
    x[7] = csub(e3, w3o);
}

// cos / sin (2 pi k / P) for the odd radices in registers, the quad-precision
// values rounded to double (the same values the twiddle table holds at
// tw[k n / P], fc_tables.cpp): constants folded into the instructions instead
// of shared-memory loads
FCSG_HD constexpr double root_cos(int P, int k) {
    switch (P * 16 + k) {
        case 3 * 16 + 1: return -0.5;
        case 5 * 16 + 1: return 0.30901699437494745;
        case 5 * 16 + 2: return -0.80901699437494745;
        case 7 * 16 + 1: return 0.62348980185873348;
        case 7 * 16 + 2: return -0.22252093395631439;
        case 7 * 16 + 3: return -0.90096886790241915;
        case 9 * 16 + 1: return 0.76604444311897801;
        case 9 * 16 + 2: return 0.17364817766693036;
        case 9 * 16 + 3: return -0.5;
        case 9 * 16 + 4: return -0.93969262078590843;
        case 11 * 16 + 1: return 0.84125353283118121;
        case 11 * 16 + 2: return 0.41541501300188644;
        case 11 * 16 + 3: return -0.14231483827328514;
        case 11 * 16 + 4: return -0.6548607339452851;
        case 11 * 16 + 5: return -0.95949297361449737;
        case 13 * 16 + 1: return 0.88545602565320991;
        case 13 * 16 + 2: return 0.56806474673115581;
        case 13 * 16 + 3: return 0.12053668025532305;
        case 13 * 16 + 4: return -0.35460488704253562;
        case 13 * 16 + 5: return -0.74851074817110108;
        case 13 * 16 + 6: return -0.97094181742605201;
        default: return 0.0;
    }
}
FCSG_HD constexpr double root_sin(int P, int k) {
    switch (P * 16 + k) {
        case 3 * 16 + 1: return 0.8660254037844386;
        case 5 * 16 + 1: return 0.95105651629515353;
        case 5 * 16 + 2: return 0.58778525229247314;
        case 7 * 16 + 1: return 0.7818314824680298;
        case 7 * 16 + 2: return 0.97492791218182362;
        case 7 * 16 + 3: return 0.43388373911755812;
        case 9 * 16 + 1: return 0.64278760968653936;
        case 9 * 16 + 2: return 0.98480775301220802;
        case 9 * 16 + 3: return 0.8660254037844386;
        case 9 * 16 + 4: return 0.34202014332566871;
        case 11 * 16 + 1: return 0.54064081745559756;
        case 11 * 16 + 2: return 0.90963199535451833;
        case 11 * 16 + 3: return 0.98982144188093268;
        case 11 * 16 + 4: return 0.75574957435425827;
        case 11 * 16 + 5: return 0.28173255684142967;
        case 13 * 16 + 1: return 0.46472317204376856;
        case 13 * 16 + 2: return 0.82298386589365635;
        case 13 * 16 + 3: return 0.99270887409805397;
        case 13 * 16 + 4: return 0.93501624268541483;
        case 13 * 16 + 5: return 0.66312265824079519;
        case 13 * 16 + 6: return 0.23931566428755777;
        default: return 0.0;
    }
}

// odd P: symmetric-pair form. cos/sin(2 pi k / P): compile-time constants for
// P <= 13, else from the n-point twiddle table (P divides n):
// tw[k n / P] = (cos, -sin).
template <int P, bool INV>
FCSG_HD void dft_odd(double2* x, const double2* tw, int n) {
    constexpr int H = (P - 1) / 2;
    double2 a[H], b[H];
    double2 y0 = x[0];
    for (int k = 1; k <= H; ++k) {
        a[k - 1] = cadd(x[k], x[P - k]);
        b[k - 1] = csub(x[k], x[P - k]);
        y0 = cadd(y0, a[k - 1]);
    }
    const int st = n / P;
    double2 y[P];
    y[0] = y0;
#pragma unroll
    for (int q = 1; q <= H; ++q) {
        double2 re = x[0];
        double2 im = mk2(0.0, 0.0);
        int idx = 0;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
            idx += q;
            if (idx >= P) idx -= P;
            double2 w;
            if constexpr (P <= 13) {
                // idx and P - idx share cos, sin flips sign; idx = 0 when P
                // is composite (9)
                const int ii = idx <= H ? idx : P - idx;
                w = idx == 0 ? mk2(1.0, 0.0) : mk2(root_cos(P, ii), idx <= H ? -root_sin(P, ii) : root_sin(P, ii));
            } else {
                w = ld2(tw + idx * st);
            }
            re = mk2(re.x + a[k - 1].x * w.x, re.y + a[k - 1].y * w.x);
            im = mk2(im.x - b[k - 1].x * w.y, im.y - b[k - 1].y * w.y);
        }
        // forward: y_q = re - i im, y_{P-q} = re + i im
        const double2 mi = mul_mi<INV>(im);
        y[q] = cadd(re, mi);
        y[P - q] = csub(re, mi);
    }
    for (int q = 0; q < P; ++q) x[q] = y[q];
}

template <int P, bool INV>
FCSG_HD void dft_reg(double2* x, const double2* tw, int n) {
    if constexpr (P == 2) dft2<INV>(x);
    else if constexpr (P == 4) dft4<INV>(x);
    else if constexpr (P == 8) dft8<INV>(x);
    else dft_odd<P, INV>(x, tw, n);
}

// x[q] *= w^q (CONJ: conj(w)^q), q = 1 .. P-1, for the butterfly's twiddle
// w = w_n^(j tstep): one table load, the powers by products in two chains
// (odd and even exponents, each advanced by w^2: at most 4 products deep, a
// few ulp against the table, far below the transform's round-off), three
// complex registers live instead of P - 1
template <int P, bool CONJ>
FCSG_HD void apply_twiddles(double2* x, double2 w) {
    if (CONJ) w.y = -w.y;
    const double2 w2 = cmul(w, w);
    double2 odd = w, even = w2;
#pragma unroll
    for (int q = 1; q < P; ++q) {
        if (q & 1) {
            x[q] = cmul(x[q], odd);
            odd = cmul(odd, w2);
        } else {
            x[q] = cmul(x[q], even);
            even = cmul(even, w2);
        }
    }
}

// ---------------------------------------------------------------------------
// one radix-P stage over all LB lines. Stage span L, m = L / P; butterfly
// (block, j) works on positions block*L + j + q*m, q < P.

template <int P>
FCSG_HD void stage_reg(Thr t, double2* buf, int pitch, int LB, int n, int L, const double2* tw, bool inv) {
    const int m = L / P;
    const int total = (n / P) * LB;
    const int tstep = n / L;
    for (int w = t.tid; w < total; w += t.nthr) {
        const int line = w % LB;
        const int b = w / LB;
        const int blk = b / m;
        const int j = b - blk * m;
        double2* p = buf + (blk * L + j) * pitch + line;
        const int ms = m * pitch;
        double2 x[P];
        for (int q = 0; q < P; ++q) x[q] = p[q * ms];
        if (!inv) {
            dft_reg<P, false>(x, tw, n);
            if (j) apply_twiddles<P, false>(x, ld2(tw + j * tstep));
        } else {
            if (j) apply_twiddles<P, true>(x, ld2(tw + j * tstep));
            dft_reg<P, true>(x, tw, n);
        }
        for (int q = 0; q < P; ++q) p[q * ms] = x[q];
    }
}

// generic radix (large primes): direct DFT with outputs staged in scr
// (scr_cap complex slots) so the stage stays in place. Contains syncs.
FCSG_HD void stage_generic(Thr t, double2* buf, int pitch, int LB, int n, int L, int P,
                           const double2* tw, bool inv, double2* scr, int scr_cap) {
    const int m = L / P;
    const int nb = n / P;
    const int tstep = n / L;
    const int pstep = n / P;
    const int ms = m * pitch;
    if (inv) {  // DIT: twiddle the inputs once, in place
        const int total = n * LB;
        for (int w = t.tid; w < total; w += t.nthr) {
            const int line = w % LB;
            const int pos = w / LB;
            const int blk = pos / L;
            const int rem = pos - blk * L;
            const int q = rem / m;
            const int j = rem - q * m;
            if (j && q) {
                double2* p = buf + pos * pitch + line;
                *p = cmulc(*p, ld2(tw + j * q * tstep));
            }
        }
        FCSG_SYNC();
    }
    const int per_b = P * LB;
    int K = scr_cap / per_b;
    if (K < 1) K = 1;
    for (int b0 = 0; b0 < nb; b0 += K) {
        const int kk = (nb - b0 < K) ? nb - b0 : K;
        const int total = kk * per_b;
        for (int w = t.tid; w < total; w += t.nthr) {
            const int line = w % LB;
            const int rest = w / LB;
            const int q = rest % P;
            const int bb = b0 + rest / P;
            const int blk = bb / m;
            const int j = bb - blk * m;
            const double2* p = buf + (blk * L + j) * pitch + line;
            double2 step = ld2(tw + q * pstep);
            if (inv) step.y = -step.y;
            double2 cur = mk2(1.0, 0.0);
            double2 acc = mk2(0.0, 0.0);
            int idx = 0;
            for (int r = 0; r < P; ++r) {
                const double2 xr = p[r * ms];
                acc = cadd(acc, cmul(xr, cur));
                idx += q;
                if (idx >= P) idx -= P;
                if ((r & 7) == 7) {  // refresh the rotation from the table
                    cur = ld2(tw + idx * pstep);
                    if (inv) cur.y = -cur.y;
                } else {
                    cur = cmul(cur, step);
                }
            }
            if (!inv && j && q) acc = cmul(acc, ld2(tw + j * q * tstep));
            scr[w] = acc;
        }
        FCSG_SYNC();
        for (int w = t.tid; w < total; w += t.nthr) {
            const int line = w % LB;
            const int rest = w / LB;
            const int q = rest % P;
            const int bb = b0 + rest / P;
            const int blk = bb / m;
            const int j = bb - blk * m;
            buf[(blk * L + j) * pitch + line + q * ms] = scr[w];
        }
        FCSG_SYNC();
    }
}

#if FCSG_CUDA
__host__ __device__
#endif
constexpr bool radix_in_registers(int p) {
    return p == 2 || p == 3 || p == 4 || p == 5 || p == 7 || p == 8 || p == 9 || p == 11 || p == 13;
}

FCSG_HD void run_stage(Thr t, double2* buf, int pitch, int LB, int n, int L, int P, const double2* tw,
                       bool inv, double2* scr, int scr_cap) {
    switch (P) {
        case 2: stage_reg<2>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 3: stage_reg<3>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 4: stage_reg<4>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 5: stage_reg<5>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 7: stage_reg<7>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 8: stage_reg<8>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 9: stage_reg<9>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 11: stage_reg<11>(t, buf, pitch, LB, n, L, tw, inv); break;
        case 13: stage_reg<13>(t, buf, pitch, LB, n, L, tw, inv); break;
        default: stage_generic(t, buf, pitch, LB, n, L, P, tw, inv, scr, scr_cap); break;
    }
}

// FcOperator::continuation (src/fc_core.cpp:221-238) for LB complex lines:
// gap[j] = sum_i A[j,i] f[N-dp1+i]  +  sum_i A[g-1-j,i] f[dp1-1-i], written
// at positions N..N+g-1.
FCSG_HD void continuation(Thr t, double2* buf, int pitch, int LB, const FcPlanDev& pl) {
    const int N = pl.n, g = pl.n_gap, d1 = pl.dp1;
    const int total = g * LB;
    for (int w = t.tid; w < total; w += t.nthr) {
        const int line = w % LB;
        const int jj = w / LB;
        double2 a = mk2(0.0, 0.0), b = mk2(0.0, 0.0);
        const double* Ar = pl.blend + jj * d1;
        const double* Al = pl.blend + (g - 1 - jj) * d1;
        for (int i = 0; i < d1; ++i) {
            const double2 fr = buf[(N - d1 + i) * pitch + line];
            const double2 fl = buf[(d1 - 1 - i) * pitch + line];
            const double cr = ld1(Ar + i), cl = ld1(Al + i);
            a = mk2(a.x + cr * fr.x, a.y + cr * fr.y);
            b = mk2(b.x + cl * fl.x, b.y + cl * fl.y);
        }
        buf[(N + jj) * pitch + line] = cadd(a, b);
    }
}

// modes (match include/fcsg.h): 1 = d/dq, 2 = d2/dq2, 3 = filter, 4 = smear filter
FCSG_HD void spec_mult(Thr t, double2* buf, int pitch, int LB, int n, const double2* mult) {
    const int total = n * LB;
    for (int w = t.tid; w < total; w += t.nthr) {
        const int line = w % LB;
        const int pos = w / LB;
        double2* p = buf + pos * pitch + line;
        *p = cmul(*p, ld2(mult + pos));
    }
}

// Full unit-span operator on the LB complex lines already loaded at
// positions 0..N-1. Ends with a sync; result at positions 0..N-1.
FCSG_HD void fc_transform(Thr t, double2* buf, int pitch, int LB, const FcPlanDev& pl, int mode,
                          double2* scr, int scr_cap) {
    continuation(t, buf, pitch, LB, pl);
    FCSG_SYNC();
    const int n = pl.n_ext;
    for (int s = 0; s < pl.nstages; ++s) {
        run_stage(t, buf, pitch, LB, n, pl.span[s], pl.radix[s], pl.tw, false, scr, scr_cap);
        FCSG_SYNC();
    }
    spec_mult(t, buf, pitch, LB, n, pl.mult + (mode - 1) * n);
    FCSG_SYNC();
    for (int s = pl.nstages - 1; s >= 0; --s) {
        run_stage(t, buf, pitch, LB, n, pl.span[s], pl.radix[s], pl.tw, true, scr, scr_cap);
        FCSG_SYNC();
    }
}

// ---------------------------------------------------------------------------
// compile-time plans for the hot lengths: every index computation below uses
// constants (no runtime integer division), stages are unrolled at compile time

template <int P, int L, int NE, int LB, int NTHR, bool INV>
FCSG_HD void stage_reg_ct(int tid, double2* buf, const double2* tw) {
    constexpr int m = L / P;
    constexpr int total = (NE / P) * LB;
    constexpr int tstep = NE / L;
    constexpr int pitch = LB;
    constexpr int ms = m * pitch;
#pragma unroll 2
    for (int w = tid; w < total; w += NTHR) {
        const int line = w % LB;
        const int b = w / LB;
        const int blk = b / m;
        const int j = b - blk * m;
        double2* p = buf + (blk * L + j) * pitch + line;
        double2 x[P];
#pragma unroll
        for (int q = 0; q < P; ++q) x[q] = p[q * ms];
        if (!INV) {
            dft_reg<P, false>(x, tw, NE);
            if (m > 1 && j) apply_twiddles<P, false>(x, ld2(tw + j * tstep));
        } else {
            if (m > 1 && j) apply_twiddles<P, true>(x, ld2(tw + j * tstep));
            dft_reg<P, true>(x, tw, NE);
        }
#pragma unroll
        for (int q = 0; q < P; ++q) p[q * ms] = x[q];
    }
}

template <int NE, int S, int LB, int NTHR, bool INV>
FCSG_HD void stage_ct(int tid, double2* buf, const double2* tw, double2* scr, int scr_cap) {
    constexpr Factors F = factor_stages(NE);
    constexpr int P = F.r[S];
    constexpr int L = F.span[S];
    if constexpr (radix_in_registers(P)) {
        stage_reg_ct<P, L, NE, LB, NTHR, INV>(tid, buf, tw);
    } else {
        stage_generic(Thr{tid, NTHR}, buf, LB, LB, NE, L, P, tw, INV, scr, scr_cap);
    }
}

// DIF stages S .. END-1
template <int NE, int S, int LB, int NTHR, int END>
FCSG_HD void dif_stages_ct(int tid, double2* buf, const double2* tw, double2* scr, int scr_cap) {
    if constexpr (S < END) {
        stage_ct<NE, S, LB, NTHR, false>(tid, buf, tw, scr, scr_cap);
        FCSG_SYNC();
        dif_stages_ct<NE, S + 1, LB, NTHR, END>(tid, buf, tw, scr, scr_cap);
    }
}

template <int NE, int S, int LB, int NTHR>
FCSG_HD void dit_stages_ct(int tid, double2* buf, const double2* tw, double2* scr, int scr_cap) {
    if constexpr (S >= 0) {
        stage_ct<NE, S, LB, NTHR, true>(tid, buf, tw, scr, scr_cap);
        FCSG_SYNC();
        dit_stages_ct<NE, S - 1, LB, NTHR>(tid, buf, tw, scr, scr_cap);
    }
}

// gap length (n_cont - 1) and boundary points (degree + 1) of the operator a
// compile-time plan of length NE is built for
#if FCSG_CUDA
__host__ __device__
#endif
constexpr int ct_gap(int ne) {
    return ne == 282 ? 26 : 24;
}
#if FCSG_CUDA
__host__ __device__
#endif
constexpr int ct_dp1(int ne) {
    return ne == 282 ? 5 : 3;
}

// compile-time continuation (gap G, D1 boundary points)
template <int N, int G, int D1, int LB, int NTHR>
FCSG_HD void continuation_ct(int tid, double2* buf, const double* blend) {
    constexpr int pitch = LB;
    for (int w = tid; w < G * LB; w += NTHR) {
        const int line = w % LB;
        const int jj = w / LB;
        double2 a = mk2(0.0, 0.0), b = mk2(0.0, 0.0);
        const double* Ar = blend + jj * D1;
        const double* Al = blend + (G - 1 - jj) * D1;
#pragma unroll
        for (int i = 0; i < D1; ++i) {
            const double2 fr = buf[(N - D1 + i) * pitch + line];
            const double2 fl = buf[(D1 - 1 - i) * pitch + line];
            const double cr = ld1(Ar + i), cl = ld1(Al + i);
            a = mk2(a.x + cr * fr.x, a.y + cr * fr.y);
            b = mk2(b.x + cl * fl.x, b.y + cl * fl.y);
        }
        buf[(N + jj) * pitch + line] = cadd(a, b);
    }
}

template <int NE, int LB, int NTHR>
FCSG_HD void spec_mult_ct(int tid, double2* buf, const double2* mult) {
    constexpr int pitch = LB;
    for (int w = tid; w < NE * LB; w += NTHR) {
        const int line = w % LB;
        const int pos = w / LB;
        double2* p = buf + pos * pitch + line;
        *p = cmul(*p, ld2(mult + pos));
    }
}

// Last DIF stage (span P, m = 1: butterflies on P contiguous positions, no
// twiddles), the spectral multiplier and the first DIT stage touch the same P
// positions, so one thread does all three in registers: two shared-memory
// round trips and two barriers fewer per transform.
template <int NE, int LB, int NTHR>
FCSG_HD void middle_fused_ct(int tid, double2* buf, const double2* tw, const double2* mult) {
    constexpr Factors F = factor_stages(NE);
    constexpr int P = F.r[F.n - 1];
    constexpr int total = (NE / P) * LB;
    constexpr int pitch = LB;
#pragma unroll 2
    for (int w = tid; w < total; w += NTHR) {
        const int line = w % LB;
        const int blk = w / LB;
        double2* p = buf + blk * P * pitch + line;
        const double2* mm = mult + blk * P;
        double2 x[P];
#pragma unroll
        for (int q = 0; q < P; ++q) x[q] = p[q * pitch];
        dft_reg<P, false>(x, tw, NE);
#pragma unroll
        for (int q = 0; q < P; ++q) x[q] = cmul(x[q], ld2(mm + q));
        dft_reg<P, true>(x, tw, NE);
#pragma unroll
        for (int q = 0; q < P; ++q) p[q * pitch] = x[q];
    }
}

// Large prime last radix P, symmetric-pair form: with s_r = x_r + x_{P-r},
// d_r = x_r - x_{P-r} (r = 1..H, H = (P-1)/2) and t = 2 pi r q / P,
//   Y_q     = x_0 + sum_r (s_r cos t - i d_r sin t),
//   Y_{P-q} = x_0 + sum_r (s_r cos t + i d_r sin t),
// so one pass over H terms gives two outputs (a quarter of the direct DFT's
// complex multiply-adds). Forward DFT + multiplier into the scratch as the
// sums/differences of the multiplied pairs, then the inverse the same way
// back into buf. scr holds NE * LB complex values (scr[pos * LB + line]).
template <int NE, int LB, int NTHR>
FCSG_HD void middle_sym_ct(int tid, double2* buf, const double2* tw, const double2* mult, double2* scr) {
    constexpr Factors F = factor_stages(NE);
    constexpr int P = F.r[F.n - 1];
    constexpr int H = (P - 1) / 2;
    constexpr int pstep = NE / P;
    constexpr int nblk = NE / P;
    constexpr int pitch = LB;
    // 1: s/d in place
    for (int w = tid; w < nblk * H * LB; w += NTHR) {
        const int line = w % LB;
        const int u = w / LB;
        const int blk = u / H, r = 1 + (u - blk * H);
        double2* xb = buf + blk * P * pitch + line;
        const double2 a = xb[r * pitch], b = xb[(P - r) * pitch];
        xb[r * pitch] = cadd(a, b);
        xb[(P - r) * pitch] = csub(a, b);
    }
    FCSG_SYNC();
    // 2: Y_q, Y_{P-q}, times the multiplier, stored as their sum / difference
    for (int w = tid; w < nblk * (H + 1) * LB; w += NTHR) {
        const int line = w % LB;
        const int u = w / LB;
        const int blk = u / (H + 1), q = u - blk * (H + 1);
        const double2* xb = buf + blk * P * pitch + line;
        const double2 x0 = xb[0];
        double2* sb = scr + blk * P * LB + line;
        const double2* mb = mult + blk * P;
        if (q == 0) {
            double2 y = x0;
            for (int r = 1; r <= H; ++r) y = cadd(y, xb[r * pitch]);
            sb[0] = cmul(y, ld2(mb));
            continue;
        }
        double2 A = x0, B = mk2(0.0, 0.0);
        int k = 0;
        for (int r = 1; r <= H; ++r) {
            k += q;
            if (k >= P) k -= P;
            const double2 c = ld2(tw + k * pstep);  // (cos t, -sin t)
            const double2 sr = xb[r * pitch], dr = xb[(P - r) * pitch];
            A = mk2(A.x + sr.x * c.x, A.y + sr.y * c.x);
            B = mk2(B.x - dr.x * c.y, B.y - dr.y * c.y);  // + d_r sin t
        }
        const double2 yq = cmul(mk2(A.x + B.y, A.y - B.x), ld2(mb + q));          // A - iB
        const double2 yp = cmul(mk2(A.x - B.y, A.y + B.x), ld2(mb + P - q));      // A + iB
        sb[q * LB] = cadd(yq, yp);
        sb[(P - q) * LB] = csub(yq, yp);
    }
    FCSG_SYNC();
    // 3: inverse, z_r = y_0 + sum_q (S_q cos t + i D_q sin t), z_{P-r} with -i
    for (int w = tid; w < nblk * (H + 1) * LB; w += NTHR) {
        const int line = w % LB;
        const int u = w / LB;
        const int blk = u / (H + 1), r = u - blk * (H + 1);
        const double2* sb = scr + blk * P * LB + line;
        double2* zb = buf + blk * P * pitch + line;
        const double2 y0 = sb[0];
        if (r == 0) {
            double2 z = y0;
            for (int q = 1; q <= H; ++q) z = cadd(z, sb[q * LB]);
            zb[0] = z;
            continue;
        }
        double2 A = y0, B = mk2(0.0, 0.0);
        int k = 0;
        for (int q = 1; q <= H; ++q) {
            k += r;
            if (k >= P) k -= P;
            const double2 c = ld2(tw + k * pstep);
            const double2 Sq = sb[q * LB], Dq = sb[(P - q) * LB];
            A = mk2(A.x + Sq.x * c.x, A.y + Sq.y * c.x);
            B = mk2(B.x - Dq.x * c.y, B.y - Dq.y * c.y);
        }
        zb[r * pitch] = mk2(A.x - B.y, A.y + B.x);        // A + iB
        zb[(P - r) * pitch] = mk2(A.x + B.y, A.y - B.x);  // A - iB
    }
}

#if FCSG_CUDA
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// middle_sym_ct on the FP64 tensor cores. The sums over r of the symmetric
// form are real matrix products: with the columns j = (block, line, re/im),
//   A[q][j] = sum_r cos(2 pi q r / P) s_r[j],   B[q][j] = sum_r sin(2 pi q r / P) d_r[j]
// (q = 0..H rows, r = 1..H), so one warp computes them for 4 block-lines
// (8 real columns) per mma.m8n8k4 tile: A operand = the cos / sin matrices
// (rows q, columns r, read from the twiddle table), B operand = s_r / d_r
// straight from the line buffer. A lane's D fragment holds the real and
// imaginary column of one block-line, so Y_q = A - iB and Y_{P-q} = A + iB
// are formed in registers. The inverse is the same product over the sums /
// differences of the multiplied outputs.
template <int NE, int LB, int NTHR>
__device__ void middle_dmma_ct(int tid, double2* buf, const double2* tw, const double2* mult, double2* scr,
                               const double2* frag) {
    constexpr Factors F = factor_stages(NE);
    constexpr int P = F.r[F.n - 1];
    constexpr int H = (P - 1) / 2;
    constexpr int pstep = NE / P;
    constexpr int nblk = NE / P;
    constexpr int MT = (H + 1 + 7) / 8;  // m-tiles over q = 0..H
    constexpr int KS = (H + 3) / 4;      // k-steps over r = 1..H
    constexpr int NBL = nblk * LB;       // block-lines
    constexpr int NTILE = (NBL + 3) / 4;
    constexpr int NW = NTHR / 32;
    constexpr int MC = MT <= 3 ? MT : 1;
    static_assert(NTHR % 32 == 0, "whole warps");
    const int lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    // 1: s_r, d_r in place
    for (int w = tid; w < nblk * H * LB; w += NTHR) {
        const int line = w % LB;
        const int u = w / LB;
        const int blk = u / H, r = 1 + (u - blk * H);
        double2* xb = buf + blk * P * LB + line;
        const double2 a = xb[r * LB], b = xb[(P - r) * LB];
        xb[r * LB] = cadd(a, b);
        xb[(P - r) * LB] = csub(a, b);
    }
    __syncthreads();
    // cos / sin (2 pi q r / P) of this lane's A fragment (row q = 8 mt + g,
    // column r = 1 + 4 ks + t): one 16-byte load per (m-tile, k-step) from the
    // plan's fragment table (FcPlanDev::prime_frag, L1 / L2 resident; zero
    // outside q, r <= H) -- reducing q r mod P and gathering the root from the
    // staged twiddles cost a quarter of the pass's issue slots and most of
    // its shared-memory bank conflicts
    auto cs = [&](int mt, int ks, double& c, double& sn) {
        const double2 w = ldg2(frag + (mt * KS + ks) * 32 + lane);
        c = w.x;
        sn = w.y;
    };
    // 2: forward DFT + multiplier; src = buf (s at r, d at P - r), dst = scr
    // 3: inverse; src = scr (S at q, D at P - q), dst = buf
    for (int ph = 0; ph < 2; ++ph) {
        const double2* src = ph == 0 ? buf : scr;
        double2* dst = ph == 0 ? scr : buf;
        // work items = (tile of 4 block-lines, chunk of MC m-tiles) over the
        // warps: with few block-lines (one 139-point line set: a single tile)
        // the m-tiles are what spreads the product over the CTA
        constexpr int NMC = (MT + MC - 1) / MC;
        for (int item = warp; item < NTILE * NMC; item += NW) {
            const int nt = item / NMC, mt_begin = (item - nt * NMC) * MC;
            const int blB = nt * 4 + (g >> 1);  // B column n = g: block-line, real/imaginary part
            const bool vB = blB < NBL;
            const double* colB =
                reinterpret_cast<const double*>(src + (vB ? (blB / LB) * P * LB + blB % LB : 0)) + (g & 1);
            const int blD = nt * 4 + t;  // D columns 2t, 2t + 1: block-line blD, re / im
            const bool vD = blD < NBL;
            const int blk = vD ? blD / LB : 0, line = vD ? blD % LB : 0;
            const double2 x0 = src[blk * P * LB + line];
            double2* db = dst + blk * P * LB + line;
            const double2* mb = mult + blk * P;
            // m-tiles in chunks of MC (all at once for P = 47; one at a time
            // for P = 67, whose 5 x 4 accumulators would not fit 80 registers)
            {
                const int mt0 = mt_begin;
                double aA[MC][2], aB[MC][2];
#pragma unroll
                for (int m = 0; m < MC; ++m) aA[m][0] = aA[m][1] = aB[m][0] = aB[m][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int r = 1 + 4 * ks + t;
                    const bool vr = vB && r <= H;
                    const double sv = vr ? colB[2 * r * LB] : 0.0;
                    const double dv = vr ? colB[2 * (P - r) * LB] : 0.0;
#pragma unroll
                    for (int m = 0; m < MC; ++m) {
                        double c, sn;
                        cs(mt0 + m, ks, c, sn);
                        dmma884(aA[m][0], aA[m][1], c, sv);
                        dmma884(aB[m][0], aB[m][1], sn, dv);
                    }
                }
                if (!vD) continue;
#pragma unroll
                for (int m = 0; m < MC; ++m) {
                    const int q = 8 * (mt0 + m) + g;
                    if (q > H) continue;
                    const double ax = aA[m][0] + x0.x, ay = aA[m][1] + x0.y, bx = aB[m][0], by = aB[m][1];
                    if (ph == 0) {
                        const double2 yq = cmul(mk2(ax + by, ay - bx), ld2(mb + q));  // A - iB
                        if (q == 0) {
                            db[0] = yq;
                        } else {
                            const double2 yp = cmul(mk2(ax - by, ay + bx), ld2(mb + P - q));  // A + iB
                            db[q * LB] = cadd(yq, yp);
                            db[(P - q) * LB] = csub(yq, yp);
                        }
                    } else {
                        db[q * LB] = mk2(ax - by, ay + bx);  // A + iB
                        if (q > 0) db[(P - q) * LB] = mk2(ax + by, ay - bx);
                    }
                }
            }
        }
        if (ph == 0) __syncthreads();  // the caller syncs after the inverse
    }
}
#endif

// fc_transform for n_ext = NE with the reference continuation (n_cont = 25,
// degree 2): N = NE - 24. When the last radix is a large prime, scr must hold
// NE * LB complex values (see middle_sym_ct).
template <int NE, int LB, int NTHR>
FCSG_HD void fc_transform_ct(int tid, double2* buf, const FcPlanDev& pl, int mode, double2* scr, int scr_cap) {
    constexpr Factors F = factor_stages(NE);
    continuation_ct<NE - ct_gap(NE), ct_gap(NE), ct_dp1(NE), LB, NTHR>(tid, buf, pl.blend);
    FCSG_SYNC();
    dif_stages_ct<NE, 0, LB, NTHR, F.n - 1>(tid, buf, pl.tw, scr, scr_cap);
    if constexpr (radix_in_registers(F.r[F.n - 1])) {
        middle_fused_ct<NE, LB, NTHR>(tid, buf, pl.tw, pl.mult + (mode - 1) * NE);
    } else {
#if FCSG_CUDA
        middle_dmma_ct<NE, LB, NTHR>(tid, buf, pl.tw, pl.mult + (mode - 1) * NE, scr, pl.prime_frag);
#else
        middle_sym_ct<NE, LB, NTHR>(tid, buf, pl.tw, pl.mult + (mode - 1) * NE, scr);
#endif
    }
    FCSG_SYNC();
    dit_stages_ct<NE, F.n - 2, LB, NTHR>(tid, buf, pl.tw, scr, scr_cap);
}

// scratch (complex slots) fc_transform_ct<NE, LB> needs
#if FCSG_CUDA
__host__ __device__
#endif
constexpr int ct_scratch_slots(int ne, int lb) {
    const Factors f = factor_stages(ne);
    return radix_in_registers(f.r[f.n - 1]) ? 0 : ne * lb;
}

// the lengths with a compile-time plan: the reference operator (degree 2,
// n_cont = 25) at N = 256, 512 and 147 (config 3's annulus subpatches), and
// BASELINE config 1's operator (degree 4, n_cont = 27) at N = 256
#if FCSG_CUDA
__host__ __device__
#endif
constexpr bool has_ct_plan(int n_ext) {
    return n_ext == 280 || n_ext == 536 || n_ext == 282 || n_ext == 171;
}
// true when plan pl is the operator a compile-time plan of its length was built for
inline bool ct_plan_for(const FcPlanDev& pl) {
    return has_ct_plan(pl.n_ext) && pl.n_gap == ct_gap(pl.n_ext) && pl.dp1 == ct_dp1(pl.n_ext);
}

}  // namespace fcsg
