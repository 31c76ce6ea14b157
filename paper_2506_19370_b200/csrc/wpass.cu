// Warp-per-line kernels on the n_ext = 280 prime-factor transform (wline.h):
// the N = 256 lines of the reference operator (every subpatch of BASELINE
// configs 1 and 5, and the Cartesian I / S patches of configs 3 and 4).
//
//  * fc_lines (FcOperator::derivative / filter / strong_filter over a batch
//    of lines, src/fc_core.cpp:257-306): one complex line = two real lines
//    per warp.
//  * pass X / pass Y of the Cartesian flux form (step_kernels.cu PassXc /
//    PassYc, euler_rhs src/euler.cpp:25-101 as div(mu grad w - f), and the
//    SSPRK(5,4) stage update src/euler.cpp:182-221): one row (X) or column
//    (Y) of one subpatch per warp, 4 transform rounds, the per-point values a
//    later round needs kept in the lane's registers.
//
// A CTA is kWarps independent warps; the only block barrier orders the copy
// of the multiplier table into shared memory before the first transform.
// Each warp's lane l owns the points i = l + 32 m (m < 8) of its line for
// loads and epilogues (coalesced along rows), and the butterflies of the
// transform (wline.h).
#include <algorithm>
#include <cstdlib>

#include "dev.h"
#include "fc_lines.h"
#include "pass_common.h"
#include "step_kernels.h"
#include "wct280.h"
#include "wline.h"
#include "wpass_common.h"

namespace fcsg {

namespace {
constexpr int kWarps = 8;  // warps per CTA
constexpr int kWThreads = kWarps * 32;
}  // namespace

// tuning knobs of the passes (A/B variant builds: scripts/build_variant.sh)
#ifndef FCSG_X_MINB
#define FCSG_X_MINB 5  // pass X: CTAs per SM the register budget is sized for
#endif
#ifndef FCSG_Y_MINB
#define FCSG_Y_MINB 5
#endif
#ifndef FCSG_X_KC
#define FCSG_X_KC 1  // pass X update epilogue: points per load chunk
#endif
#ifndef FCSG_X_KL
#define FCSG_X_KL 4  // pass X other phases: points per load chunk
#endif
#ifndef FCSG_Y_KC
#define FCSG_Y_KC 4  // pass Y: points per load chunk
#endif


// the operator tables a CTA keeps in shared memory: the multiplier (280
// double2, prime-factor order), the 24 x 3 blend matrix and the slot of each
// natural position i < 256 (slot_of: ~12 integer instructions, which the
// loads and epilogues would otherwise spend per point -- a quarter of the
// passes' instructions were integer before the table)
constexpr int kBlendSlots = (w280::kGap * w280::kD1 + 1) / 2;
constexpr int kSlotTabSlots = w280::kN * 2 / 16;  // 256 ushort
constexpr int kTabSlots = w280::kNE + kBlendSlots + kSlotTabSlots;
FCSG_HD void stage_w280_tables(int tid, int nthr, const double2* mult_src, const double* blend_src, double2* mult,
                               double* blend) {
    for (int k = tid; k < w280::kNE; k += nthr) mult[k] = ldg2(mult_src + k);
    for (int k = tid; k < w280::kGap * w280::kD1; k += nthr) blend[k] = ldg1(blend_src + k);
    unsigned short* st = reinterpret_cast<unsigned short*>(mult + w280::kNE + kBlendSlots);
    for (int k = tid; k < w280::kN; k += nthr) st[k] = static_cast<unsigned short>(w280::slot_of(k));
}
FCSG_HD const unsigned short* slot_table(const double2* mult) {
    return reinterpret_cast<const unsigned short*>(mult + w280::kNE + kBlendSlots);
}
#if !FCSG_CUDA
// the emulation build's copy (its tables are not staged)
inline const unsigned short* host_slot_table() {
    static const std::vector<unsigned short> t = [] {
        std::vector<unsigned short> v(w280::kN);
        for (int k = 0; k < w280::kN; ++k) v[k] = static_cast<unsigned short>(w280::slot_of(k));
        return v;
    }();
    return t.data();
}
#endif

// ---------------------------------------------------------------------------
// FC line batch
//
// One complex line (two real lines) per warp, one pass over the batch: a
// single wave for config 1 (2048 pairs). The kernel is latency-bound (16 MB
// moved in a few microseconds), so every lane issues all 16 of its loads at
// once, before the CTA stages the operator tables. Measured (graph-timed,
// config 1): 2 lines per warp in 4-warp CTAs 9.9 us, 2-warp CTAs 10.1,
// 1-warp 11.1; one real line per warp (twice the warps, the imaginary half
// idle) 14.5-16.3.

// RPW real lines per warp: 2 (one complex transform carries two lines, the
// default) or 1 (the imaginary half idle: twice the warps for the same lines,
// more latency hiding for the same single wave -- an A/B variant)
template <int NL, int RPW>
FCSG_HD void w280_load(int lane, long unit, const FcLinesArgs& a, double* v0, double* v1) {
    using namespace w280;
    const long l = RPW * unit;
    const long ls = a.line_stride, st = a.stride;
    const bool have1 = RPW == 2 && l + 1 < a.n_lines;
    constexpr int PPL = kN / NL;
#pragma unroll
    for (int m = 0; m < PPL; ++m) {
        const int i = lane + NL * m;
        v0[m] = ldg1(a.in + l * ls + i * st);
        v1[m] = have1 ? ldg1(a.in + (l + 1) * ls + i * st) : 0.0;
    }
}

template <int NL, int RPW>
FCSG_HD void w280_finish(int lane, long unit, double2* buf, const double2* mult, const double* blend,
                         const unsigned short* st, const FcLinesArgs& a, const double* v0, const double* v1) {
    using namespace w280;
    const long l = RPW * unit;
    const long ols = a.out_line_stride, ost = a.out_stride;
    const bool have1 = RPW == 2 && l + 1 < a.n_lines;
    constexpr int PPL = kN / NL;
#pragma unroll
    for (int m = 0; m < PPL; ++m) buf[st[lane + NL * m]] = mk2(v0[m], v1[m]);
    FCSG_SYNCWARP();
    transform<NL, 1>(lane, buf, kSlots, mult, blend);
#pragma unroll 4
    for (int m = 0; m < PPL; ++m) {
        const int i = lane + NL * m;
        const double2 v = buf[st[i]];
        a.out[l * ols + i * ost] = v.x * a.scale;
        if (have1) a.out[(l + 1) * ols + i * ost] = v.y * a.scale;
    }
}

#if FCSG_CUDA
template <int RPW, int WPC>
__global__ void __launch_bounds__(WPC * 32) w280_lines_kernel(const __grid_constant__ FcLinesArgs a) {
    extern __shared__ double2 wsm[];
    double2* mult = wsm;
    double* blend = reinterpret_cast<double*>(wsm + w280::kNE);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + kTabSlots + warp * w280::kSlots;
    const long nunits = (a.n_lines + RPW - 1) / RPW;
    long unit = static_cast<long>(blockIdx.x) * WPC + warp;
    double v0[w280::kN / 32], v1[w280::kN / 32];
    if (unit < nunits) w280_load<32, RPW>(lane, unit, a, v0, v1);  // in flight while the tables are staged
    stage_w280_tables(threadIdx.x, WPC * 32, a.pl.mult_pfa + (a.mode - 1) * w280::kNE, a.pl.blend, mult, blend);
    __syncthreads();
    for (; unit < nunits; unit += static_cast<long>(gridDim.x) * WPC) {
        w280_finish<32, RPW>(lane, unit, buf, mult, blend, slot_table(mult), a, v0, v1);
        const long nxt = unit + static_cast<long>(gridDim.x) * WPC;
        if (nxt < nunits) {
            FCSG_SYNCWARP();
            w280_load<32, RPW>(lane, nxt, a, v0, v1);
        }
    }
}

template <int RPW, int WPC>
void launch_w280_variant(const FcLinesArgs& a, cudaStream_t s) {
    const long nunits = (a.n_lines + RPW - 1) / RPW;
    const size_t smem = (kTabSlots + WPC * w280::kSlots) * sizeof(double2);
    const long nblk = (nunits + WPC - 1) / WPC;
    const int grid = static_cast<int>(std::min<long>(nblk, 148L * 64));
    w280_lines_kernel<RPW, WPC><<<grid, WPC * 32, smem, s>>>(a);
}
#endif

// ---------------------------------------------------------------------------
// FC line batch, register-resident 8 x 35 transform (wct280.h): eight real
// lines (four complex) per warp, rows only (stride 1 in and out: lane (c, r)
// reads and writes positions r + 8 t of its lines straight from and to
// global memory). Three warp phases separated by __syncwarp: P1 loads,
// continuation, DFT-35 -> shared memory; P2 the 140 DFT-8 groups with the
// multiplier; P3 shared memory -> inverse DFT-35 -> stores.

FCSG_HD void wct_load(int lane, long unit, const FcLinesArgs& a, double2 (&z)[wct::kT]) {
    using namespace wct;
    const int c = lane >> 3, r = lane & 7;
    const long l0 = 8 * unit + 2 * c;
    const bool h0 = l0 < a.n_lines, h1 = l0 + 1 < a.n_lines;
    const double* p0 = a.in + l0 * a.line_stride + r;
    const double* p1 = p0 + a.line_stride;
#pragma unroll
    for (int t = 0; t < 32; ++t) z[t] = mk2(h0 ? ldg1(p0 + 8 * t) : 0.0, h1 ? ldg1(p1 + 8 * t) : 0.0);
}

FCSG_HD void wct_p1(int lane, long unit, const FcLinesArgs& a, double2 (&z)[wct::kT], double2* buf,
                    const double* blend) {
    using namespace wct;
    const int c = lane >> 3, r = lane & 7;
    double2 fr[kD1], fl[kD1];
#if FCSG_CUDA
    (void)unit;
    (void)a;
    // f[253 + i] sits in lane 5 + i of the line's lane group (t = 31),
    // f[2 - i] in lane 2 - i (t = 0)
    const int g = lane & ~7;
#pragma unroll
    for (int i = 0; i < kD1; ++i) {
        fr[i] = mk2(__shfl_sync(0xffffffffu, z[31].x, g + 5 + i), __shfl_sync(0xffffffffu, z[31].y, g + 5 + i));
        fl[i] = mk2(__shfl_sync(0xffffffffu, z[0].x, g + 2 - i), __shfl_sync(0xffffffffu, z[0].y, g + 2 - i));
    }
#else
    const long l0 = 8 * unit + 2 * c;
    const bool h0 = l0 < a.n_lines, h1 = l0 + 1 < a.n_lines;
    const double* q0 = a.in + l0 * a.line_stride;
    const double* q1 = q0 + a.line_stride;
    for (int i = 0; i < kD1; ++i) {
        fr[i] = mk2(h0 ? q0[kN - kD1 + i] : 0.0, h1 ? q1[kN - kD1 + i] : 0.0);
        fl[i] = mk2(h0 ? q0[kD1 - 1 - i] : 0.0, h1 ? q1[kD1 - 1 - i] : 0.0);
    }
#endif
    continuation(r, z, fr, fl, blend);
    dft35<false>(z);
    put35(buf, c, r, z);
}

FCSG_HD void wct_p3(int lane, long unit, const FcLinesArgs& a, const double2* buf) {
    using namespace wct;
    const int c = lane >> 3, r = lane & 7;
    const long l0 = 8 * unit + 2 * c;
    const bool h0 = l0 < a.n_lines, h1 = l0 + 1 < a.n_lines;
    double2 z[kT];
    get35(buf, c, r, z);
    dft35<true>(z);
    double* q0 = a.out + l0 * a.out_line_stride + r;
    double* q1 = q0 + a.out_line_stride;
    const double s = a.scale;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
        if (h0) q0[8 * t] = z[t].x * s;
        if (h1) q1[8 * t] = z[t].y * s;
    }
}

#if FCSG_CUDA
// programmatic dependent launch: the kernel is launched with the
// programmatic-stream-serialization attribute, so its CTAs may start while
// the previous kernel of the stream finishes; everything before
// griddepcontrol.wait reads only the operator tables (written once at
// operator creation, never by a kernel), everything after it sees the
// previous kernel's results
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int WPC>
__global__ void __launch_bounds__(WPC * 32) wct_lines_kernel(const __grid_constant__ FcLinesArgs a) {
    extern __shared__ double2 wsm[];
    double2* tabs = wsm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + wct::kTabSlots + warp * wct::kBufSlots;
    const long nunits = (a.n_lines + 7) / 8;
    const double* blend = reinterpret_cast<const double*>(tabs + wct::kNE + wct::kTwSlots);
    const long stride = static_cast<long>(gridDim.x) * WPC;
    long unit = static_cast<long>(blockIdx.x) * WPC + warp;
    double2 z[wct::kT];
    {
        wct::TableRegs<WPC * 32> tr;
        tr.load(threadIdx.x, a.pl.mult_pfa + (a.mode - 1) * wct::kNE, a.pl.tw, a.pl.blend);
        griddep_wait();
        if (unit < nunits) wct_load(lane, unit, a, z);
        griddep_launch_dependents();
        tr.store(threadIdx.x, tabs);
    }
    __syncthreads();
    // the first unit peeled (its loads were issued above, before the table
    // stores); later units (batches beyond one wave) load at the top
    auto body = [&](long u) {
        wct_p1(lane, u, a, z, buf, blend);
        __syncwarp();
        wct::middle<32>(lane, buf, tabs + wct::kNE, tabs);
        __syncwarp();
        wct_p3(lane, u, a, buf);
        __syncwarp();
    };
    // batches beyond one wave: the next unit's eight rows into L2 (one bulk
    // prefetch of 2 KB per real line, by the line pair's first lane) while
    // this unit is transformed
    auto prefetch_next = [&](long u) {
        const long nxt = u + stride;
        if (nxt < nunits && (lane & 7) == 0) {
            const long l0 = 8 * nxt + 2 * (lane >> 3);
            if (l0 < a.n_lines) pf_l2_bulk(a.in + l0 * a.line_stride, wct::kN * sizeof(double));
            if (l0 + 1 < a.n_lines) pf_l2_bulk(a.in + (l0 + 1) * a.line_stride, wct::kN * sizeof(double));
        }
    };
    if (unit < nunits) {
        prefetch_next(unit);
        body(unit);
    }
    for (unit += stride; unit < nunits; unit += stride) {
        wct_load(lane, unit, a, z);
        prefetch_next(unit);
        body(unit);
    }
}

// ---------------------------------------------------------------------------
// The same kernel with the rows staged by the TMA unit (FCSG_LINES_TMA=1, an
// A/B variant): one lane arms the warp's mbarrier with the byte count and
// issues one 2 KB bulk copy per real line (cp.async.bulk global -> shared,
// SASS UBLKCP) into the warp's transform buffer -- which is free until the
// DFT-35 results are stored -- in natural order with a row pitch of 2080 bytes
// (lane groups of consecutive complex lines land on the two halves of the
// bank row); the lanes read their positions r + 8 t from shared memory. The
// results go back the same way: registers -> rows in shared memory ->
// fence.proxy.async -> one bulk store per line. 64 LDG + 64 STG per lane
// become 16 bulk copies per warp and 64 LDS + 64 STS per lane. Needs 16-byte
// aligned rows (base pointers and even line strides), else the direct kernel.
constexpr int kTmaRowPitch = 2080;  // bytes
static_assert(8 * kTmaRowPitch <= wct::kBufSlots * 16, "the staged rows fit the transform buffer");

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

template <int WPC>
__global__ void __launch_bounds__(WPC * 32) wct_lines_tma_kernel(const __grid_constant__ FcLinesArgs a) {
    extern __shared__ double2 wsm[];
    double2* tabs = wsm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + wct::kTabSlots + warp * wct::kBufSlots;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + wct::kTabSlots + WPC * wct::kBufSlots) + warp;
    char* rows = reinterpret_cast<char*>(buf);
    const long nunits = (a.n_lines + 7) / 8;
    const double* blend = reinterpret_cast<const double*>(tabs + wct::kNE + wct::kTwSlots);
    const long stride = static_cast<long>(gridDim.x) * WPC;
    const int c = lane >> 3, r = lane & 7;
    constexpr unsigned kRowBytes = wct::kN * sizeof(double);
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    // lane 0: arm the barrier and request the unit's rows
    auto request = [&](long u) {
        if (lane == 0) {
            const long l0 = 8 * u;
            const int nrows = static_cast<int>(a.n_lines - l0 < 8 ? a.n_lines - l0 : 8);
            mbar_expect_tx(bar, nrows * kRowBytes);
            for (int k = 0; k < nrows; ++k)
                bulk_load(rows + k * kTmaRowPitch, a.in + (l0 + k) * a.line_stride, kRowBytes, bar);
        }
    };
    long unit = static_cast<long>(blockIdx.x) * WPC + warp;
    {
        wct::TableRegs<WPC * 32> tr;
        tr.load(threadIdx.x, a.pl.mult_pfa + (a.mode - 1) * wct::kNE, a.pl.tw, a.pl.blend);
        griddep_wait();
        if (unit < nunits) request(unit);
        griddep_launch_dependents();
        tr.store(threadIdx.x, tabs);
    }
    __syncthreads();
    unsigned parity = 0;
    for (; unit < nunits; unit += stride) {
        const long l0 = 8 * unit + 2 * c;
        const bool h0 = l0 < a.n_lines, h1 = l0 + 1 < a.n_lines;
        mbar_wait(bar, parity);
        parity ^= 1;
        double2 z[wct::kT];
        {
            const double* x0 = reinterpret_cast<const double*>(rows + (2 * c) * kTmaRowPitch) + r;
            const double* x1 = reinterpret_cast<const double*>(rows + (2 * c + 1) * kTmaRowPitch) + r;
#pragma unroll
            for (int t = 0; t < 32; ++t) z[t] = mk2(h0 ? x0[8 * t] : 0.0, h1 ? x1[8 * t] : 0.0);
        }
        __syncwarp();  // every lane has read its rows: the buffer may take the DFT-35 results
        wct_p1(lane, unit, a, z, buf, blend);
        __syncwarp();
        wct::middle<32>(lane, buf, tabs + wct::kNE, tabs);
        __syncwarp();
        wct::get35(buf, c, r, z);
        wct::dft35<true>(z);
        __syncwarp();  // every lane has read the buffer: it may take the result rows
        {
            double* y0 = reinterpret_cast<double*>(rows + (2 * c) * kTmaRowPitch) + r;
            double* y1 = reinterpret_cast<double*>(rows + (2 * c + 1) * kTmaRowPitch) + r;
            const double sc = a.scale;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
                y0[8 * t] = z[t].x * sc;
                y1[8 * t] = z[t].y * sc;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> the bulk store's reads
        __syncwarp();
        if (lane == 0) {
            const long b0 = 8 * unit;
            const int nrows = static_cast<int>(a.n_lines - b0 < 8 ? a.n_lines - b0 : 8);
            for (int k = 0; k < nrows; ++k)
                bulk_store(a.out + (b0 + k) * a.out_line_stride, rows + k * kTmaRowPitch, kRowBytes);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the rows have been read out
        }
        __syncwarp();
        if (unit + stride < nunits) request(unit + stride);
    }
}

template <int WPC>
void launch_wct_tma_variant(const FcLinesArgs& a, cudaStream_t s, bool pdl) {
    static unsigned long long done = 0;
    constexpr size_t smem = (wct::kTabSlots + WPC * wct::kBufSlots) * sizeof(double2) + WPC * sizeof(unsigned long long);
    if (dev::first_on_device(&done))
        cudaFuncSetAttribute(wct_lines_tma_kernel<WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const long nunits = (a.n_lines + 7) / 8;
    const long nblk = (nunits + WPC - 1) / WPC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<long>(nblk, 148L * 16)));
    cfg.blockDim = dim3(WPC * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, wct_lines_tma_kernel<WPC>, a);
}

template <int WPC>
void launch_wct_variant(const FcLinesArgs& a, cudaStream_t s, bool pdl) {
    static unsigned long long done = 0;
    constexpr size_t smem = (wct::kTabSlots + WPC * wct::kBufSlots) * sizeof(double2);
    if (dev::first_on_device(&done))
        cudaFuncSetAttribute(wct_lines_kernel<WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const long nunits = (a.n_lines + 7) / 8;
    const long nblk = (nunits + WPC - 1) / WPC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<long>(nblk, 148L * 16)));
    cfg.blockDim = dim3(WPC * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, wct_lines_kernel<WPC>, a);
}
#endif

bool wct_lines_applies(const FcLinesArgs& a) {
    return w280_lines_applies(a.pl) && a.stride == 1 && a.out_stride == 1;
}

void launch_wct_lines(const FcLinesArgs& a, void* stream) {
    if (a.n_lines == 0) return;
#if FCSG_CUDA
    // A/B experiments: FCSG_WCT_WPC = warps per CTA (4: two CTAs of 244 registers per SM; five-warp CTAs
    // capped at 168 registers for 10 warps per SM measured 3455 against 4321 GB/s on 262144 lines)
    static const int wpc = [] {
        const char* v = std::getenv("FCSG_WCT_WPC");
        return v ? std::atoi(v) : 4;
    }();
    static const bool pdl = !std::getenv("FCSG_NO_PDL");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    // A/B: FCSG_LINES_TMA=1 stages the rows with TMA bulk copies (needs 16-byte aligned rows)
    static const bool tma = [] {
        const char* v = std::getenv("FCSG_LINES_TMA");
        return v && v[0] == '1';
    }();
    const bool aligned = reinterpret_cast<unsigned long long>(a.in) % 16 == 0 &&
                         reinterpret_cast<unsigned long long>(a.out) % 16 == 0 && a.line_stride % 2 == 0 &&
                         a.out_line_stride % 2 == 0;
    if (tma && aligned) {
        switch (wpc) {
            case 2: launch_wct_tma_variant<2>(a, s, pdl); break;
            case 8: launch_wct_tma_variant<8>(a, s, pdl); break;
            default: launch_wct_tma_variant<4>(a, s, pdl); break;
        }
        return;
    }
    switch (wpc) {
        case 2: launch_wct_variant<2>(a, s, pdl); break;
        case 8: launch_wct_variant<8>(a, s, pdl); break;
        default: launch_wct_variant<4>(a, s, pdl); break;
    }
#else
    (void)stream;
    std::vector<double2> tabs(wct::kTabSlots), buf(wct::kBufSlots);
    wct::stage_tables(0, 1, a.pl.mult_pfa + (a.mode - 1) * wct::kNE, a.pl.tw, a.pl.blend, tabs.data());
    const double* blend = reinterpret_cast<const double*>(tabs.data() + wct::kNE + wct::kTwSlots);
    const long nunits = (a.n_lines + 7) / 8;
    double2 z[wct::kT];
    for (long unit = 0; unit < nunits; ++unit) {
        for (int lane = 0; lane < 32; ++lane) {
            wct_load(lane, unit, a, z);
            wct_p1(lane, unit, a, z, buf.data(), blend);
        }
        for (int lane = 0; lane < 32; ++lane) wct::middle<32>(lane, buf.data(), tabs.data() + wct::kNE, tabs.data());
        for (int lane = 0; lane < 32; ++lane) wct_p3(lane, unit, a, buf.data());
    }
#endif
}

bool w280_lines_applies(const FcPlanDev& pl) {
    return pl.n_ext == 280 && pl.n == 256 && pl.n_gap == 24 && pl.dp1 == 3 && pl.mult_pfa != nullptr;
}

void launch_w280_lines(const FcLinesArgs& a, void* stream) {
    if (a.n_lines == 0) return;
#if FCSG_CUDA
    static const int variant = [] {  // A/B experiments: FCSG_W280_VARIANT = RPW * 10 + WPC
        const char* v = std::getenv("FCSG_W280_VARIANT");
        return v ? std::atoi(v) : 24;  // 2 lines per warp, 4-warp CTAs (measured best of 11..24)
    }();
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (variant) {
        case 11: launch_w280_variant<1, 1>(a, s); break;
        case 12: launch_w280_variant<1, 2>(a, s); break;
        case 14: launch_w280_variant<1, 4>(a, s); break;
        case 21: launch_w280_variant<2, 1>(a, s); break;
        case 22: launch_w280_variant<2, 2>(a, s); break;
        default: launch_w280_variant<2, 4>(a, s); break;
    }
#else
    (void)stream;
    const long npairs = (a.n_lines + 1) / 2;
    std::vector<double2> buf(w280::kSlots);
    const double2* mult = a.pl.mult_pfa + (a.mode - 1) * w280::kNE;
    double v0[w280::kN], v1[w280::kN];
    for (long pair = 0; pair < npairs; ++pair) {
        w280_load<1, 2>(0, pair, a, v0, v1);
        w280_finish<1, 2>(0, pair, buf.data(), mult, a.pl.blend, host_slot_table(), a, v0, v1);
    }
#endif
}

// ---------------------------------------------------------------------------
// Cartesian flux-form passes (PassXc / PassYc restated per warp)
//
// Both passes transform two complex lines at once: the pass's rounds come in
// two independent pairs (X: D1 (rho, rho u) and D1 (rho v, theta); Y: D2
// (rho v, theta) and D2 (rho, rho u)), so a pass is two "double rounds":
// load -> transform both -> epilogue (Phi = mu grad w - f for both pairs) ->
// transform both -> epilogue (tA, or rhs + SSPRK update of all four
// components). The per-point values the second epilogue needs are re-read
// (L1 / L2 hits) instead of kept: pass Y updates e only in its last
// epilogue, so the state it reads there is still the stage's input.

// pitch between line buffers (double2): 313 = 1 (mod 8) spreads the quad's
// buffers over the banks (309 and 311, which would fit a fifth CTA per SM,
// measured 5-9% slower passes at either 4 or 5 CTAs)
constexpr int kBP = w280::kSlots + 1;

// Pass X (rows, second pass of the stage): D1 (rho, rho u) and D1 (rho v,
// theta) -> Phi_x = mu iq1x D1 w - F_c -> D1 Phi_x -> rhs_c = tA_c + iq1x
// D1 Phi_x_c (tA = iq2y D2 Phi_y from pass Y) -> SSPRK(5,4) update of the
// four components. One row per warp; lane l owns the points l + 32 m
// (coalesced).
template <int NL>
FCSG_HD void wpass_x_body(int lane, int line, double2* buf, const double2* mult, const EngineDev& E,
                          const double* blend, const unsigned short* st, int stage) {
    using namespace w280;
    constexpr int PPL = kN / NL;
    constexpr int KC = PPL >= FCSG_X_KC ? FCSG_X_KC : 1;  // points per load chunk of the update epilogue (13 loads per point)
    constexpr int KL = PPL >= FCSG_X_KL ? FCSG_X_KL : 1;  // points per load chunk of the other phases
    const int ni = E.ni, nj = E.nj;
    const int sub = line / nj, row = line - sub * nj;
    const long rb = static_cast<long>(sub) * ni * nj + static_cast<long>(row) * ni;
    const double inv_len = 1.0 / ((kN - 1) * E.h1[sub]);  // LineInfo::inv_len (src/subpatch_data.cpp:134)
    const bool uq = E.uniform_q != 0;
    const double qc = uq ? E.iq1x_c[sub] : 0.0;
    const double dt = E.sc->dt;
    const bool e0r = stage >= 1 && stage <= 3;  // stages whose update reads the register e0
    double2* bA = buf;
    double2* bB = buf + kBP;
    // load: e -> (rho, rho u) | (rho v, theta)
#pragma unroll 1
    for (int m0 = 0; m0 < PPL; m0 += KL) {
        double v[KL][4];
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const long p = rb + lane + NL * (m0 + k);
#pragma unroll
            for (int c = 0; c < 4; ++c) v[k][c] = ldg1(E.e[c] + p);
        }
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const int i = lane + NL * (m0 + k);
            const PrimR q = prim_r(v[k][0], v[k][1], v[k][2], v[k][3]);
            w_check_positive(E, q.rho, q.theta, rb + i, sub, i, row);
            const int s = st[i];
            bA[s] = mk2(q.rho, q.mx);
            bB[s] = mk2(q.my, q.theta);
        }
    }
    if (lane == 0) {  // the epilogue's row of mu (and iq1x) into L2 behind the transform
        pf_l2_bulk(E.mu + rb, kN * sizeof(double));
        if (!uq) pf_l2_bulk(E.iq1x + rb, kN * sizeof(double));
    }
    FCSG_SYNCWARP();
    transform<NL, 2>(lane, buf, kBP, mult, blend);
    // epilogue: s4 = mu (iq1x D1 w); the next input Phi_x = s4 - F
#pragma unroll 1
    for (int m0 = 0; m0 < PPL; m0 += KL) {
        double v[KL][4], mu[KL], a[KL];
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const long p = rb + lane + NL * (m0 + k);
#pragma unroll
            for (int c = 0; c < 4; ++c) v[k][c] = ldg1(E.e[c] + p);
            mu[k] = ldg1(E.mu + p);
            a[k] = uq ? qc : ldg1(E.iq1x + p);
        }
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const int s = st[lane + NL * (m0 + k)];
            const PrimR q = prim_r(v[k][0], v[k][1], v[k][2], v[k][3]);
            const double2 wa = bA[s], wb = bB[s];
            // mu iq1x inv_len once per point, then one FMA per component
            const double ms = mu[k] * (a[k] * inv_len);
            bA[s] = mk2(fma(ms, wa.x, -flux_x(q, 0)), fma(ms, wa.y, -flux_x(q, 1)));
            bB[s] = mk2(fma(ms, wb.x, -flux_x(q, 2)), fma(ms, wb.y, -flux_x(q, 3)));
        }
    }
    if (lane == 0) {  // the update's inputs into L2 behind the transform
        for (int c = 0; c < 4; ++c) {
            pf_l2_bulk(E.tA[c] + rb, kN * sizeof(double));
            if (e0r) pf_l2_bulk(E.e0[c] + rb, kN * sizeof(double));
            if (stage == 4) {
                pf_l2_bulk(E.e2[c] + rb, kN * sizeof(double));
                pf_l2_bulk(E.e3[c] + rb, kN * sizeof(double));
                pf_l2_bulk(E.rhs3[c] + rb, kN * sizeof(double));
            }
        }
    }
    FCSG_SYNCWARP();
    transform<NL, 2>(lane, buf, kBP, mult, blend);
    // epilogue: rhs = tA + iq1x D1 Phi_x, SSPRK update; u = the stage's input
    // state (pass Y does not write e)
#pragma unroll 1
    for (int m0 = 0; m0 < PPL; m0 += KC) {
        double u[KC][4], ta[KC][4], z[KC][4], a[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const long p = rb + lane + NL * (m0 + k);
            a[k] = uq ? qc : ldg1(E.iq1x + p);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                u[k][c] = ldg1(E.e[c] + p);
                ta[k][c] = ldg1(E.tA[c] + p);
                z[k][c] = e0r ? ldg1(E.e0[c] + p) : 0.0;
            }
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const long p = rb + lane + NL * (m0 + k);
            const int s = st[lane + NL * (m0 + k)];
            const double2 wa = bA[s], wb = bB[s];
            const double sa = a[k] * inv_len;
            ssprk_update_e0(E, stage, 0, p, u[k][0], fma(sa, wa.x, ta[k][0]), z[k][0], dt);
            ssprk_update_e0(E, stage, 1, p, u[k][1], fma(sa, wa.y, ta[k][1]), z[k][1], dt);
            ssprk_update_e0(E, stage, 2, p, u[k][2], fma(sa, wb.x, ta[k][2]), z[k][2], dt);
            ssprk_update_e0(E, stage, 3, p, u[k][3], fma(sa, wb.y, ta[k][3]), z[k][3], dt);
        }
    }
}

// Pass Y (columns, first pass of the stage): D2 (rho v, theta) and D2 (rho,
// rho u) -> Phi_y = mu iq2y D2 w - G_c -> D2 Phi_y -> tA_c = iq2y D2 Phi_y_c
// (pass X adds iq1x D1 Phi_x and updates: the terms of rhs_c commute, so
// this order only changes which partial is rounded first).
//
// Columns are strided in memory (pitch ni), so a CTA takes a quad of 4
// adjacent columns: thread t of NT handles column c = t % 4 at rows
// i = t / 4 + (NT / 4) k for the loads and epilogues -- one warp instruction
// reads 8 rows x 32 contiguous bytes -- and writes into the buffers of the
// warp that transforms that column (warp c). Block barriers order the
// loads before the transforms and the transforms before the epilogues; the
// transforms themselves are per warp.
constexpr int kQuad = 4;

template <int NT>
FCSG_HD void wpass_y_quad(int tid, int quad, double2* bufs, const double2* mult, const EngineDev& E,
                          const double* blend, const unsigned short* st) {
    using namespace w280;
    constexpr int PPT = kQuad * kN / NT;  // points per thread
    constexpr int KC = PPT >= FCSG_Y_KC ? FCSG_Y_KC : 1;  // points per load chunk
    const int ni = E.ni, nj = E.nj;
    const int qps = (ni + kQuad - 1) / kQuad;
    const int sub = quad / qps, c0 = (quad - sub * qps) * kQuad;
    const long gb = static_cast<long>(sub) * ni * nj + c0;
    const double inv_len = 1.0 / ((kN - 1) * E.h2[sub]);
    const bool uq = E.uniform_q != 0;
    const double qc = uq ? E.iq2y_c[sub] : 0.0;
    const int ncol = ni - c0 < kQuad ? ni - c0 : kQuad;
    // point k of this thread: w = tid + NT k, column w % 4, row w / 4
    auto col = [&](int k) { return (tid + NT * k) & (kQuad - 1); };
    auto row = [&](int k) { return (tid + NT * k) >> 2; };
    auto pt = [&](int k) { return gb + static_cast<long>(row(k)) * ni + col(k); };
    // line buffers: column c, line A (rho v, theta) at c * 2 kBP, line B (rho, rho u) at + kBP
    auto bA = [&](int k) -> double2& { return bufs[col(k) * 2 * kBP + st[row(k)]]; };
    auto bB = [&](int k) -> double2& { return bufs[col(k) * 2 * kBP + kBP + st[row(k)]]; };
    // the next epilogue's inputs into L2 behind the transforms: one thread per
    // 32-byte sector (the quad's 4 columns of one row)
    auto prefetch = [&](const double* const* f, int nf) {
        if (col(0) != 0) return;
        for (int k = 0; k < PPT; ++k)
            for (int q = 0; q < nf; ++q) pf_l2(f[q] + pt(k));
    };
    auto transform_all = [&]() {
        FCSG_SYNC();
#if FCSG_CUDA
        const int warp = tid >> 5;
        if (warp < kQuad) transform<32, 2>(tid & 31, bufs + warp * 2 * kBP, kBP, mult, blend);
#else
        for (int c = 0; c < kQuad; ++c) transform<1, 2>(0, bufs + c * 2 * kBP, kBP, mult, blend);
#endif
        FCSG_SYNC();
    };
    auto load_e = [&](int k, double* v) {
        const bool ok = col(k) < ncol;
        const long p = ok ? pt(k) : gb;
        v[0] = ok ? ldg1(E.e[0] + p) : 1.0;
        v[1] = ok ? ldg1(E.e[1] + p) : 0.0;
        v[2] = ok ? ldg1(E.e[2] + p) : 0.0;
        v[3] = ok ? ldg1(E.e[3] + p) : 1.0;
    };
    // load: (rho v, theta) | (rho, rho u)
#pragma unroll 1
    for (int k0 = 0; k0 < PPT; k0 += KC) {
        double v[KC][4];
#pragma unroll
        for (int k = 0; k < KC; ++k) load_e(k0 + k, v[k]);
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const PrimR q = prim_r(v[k][0], v[k][1], v[k][2], v[k][3]);
            bA(k0 + k) = mk2(q.my, q.theta);
            bB(k0 + k) = mk2(q.rho, q.mx);
        }
    }
    {
        const double* f[2] = {E.mu, E.iq2y};
        prefetch(f, uq ? 1 : 2);
    }
    transform_all();
    // epilogue: Phi_y = mu iq2y D2 w - (G_2, G_3) | - (G_0, G_1)
#pragma unroll 1
    for (int k0 = 0; k0 < PPT; k0 += KC) {
        double v[KC][4], mu[KC], d[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            load_e(k0 + k, v[k]);
            const bool ok = col(k0 + k) < ncol;
            const long p = ok ? pt(k0 + k) : gb;
            mu[k] = ok ? ldg1(E.mu + p) : 0.0;
            d[k] = uq ? qc : (ok ? ldg1(E.iq2y + p) : 0.0);
        }
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const PrimR q = prim_r(v[k][0], v[k][1], v[k][2], v[k][3]);
            double2& a = bA(k0 + k);
            double2& b = bB(k0 + k);
            const double2 wa = a, wb = b;
            const double ms = mu[k] * (d[k] * inv_len);
            a = mk2(fma(ms, wa.x, -flux_y(q, 2)), fma(ms, wa.y, -flux_y(q, 3)));
            b = mk2(fma(ms, wb.x, -flux_y(q, 0)), fma(ms, wb.y, -flux_y(q, 1)));
        }
    }
    transform_all();
    // epilogue: tA = iq2y D2 Phi_y (components 2, 3 from line A, 0, 1 from B)
#pragma unroll 2
    for (int k = 0; k < PPT; ++k) {
        if (col(k) >= ncol) continue;
        const long p = pt(k);
        const double d = (uq ? qc : ldg1(E.iq2y + p)) * inv_len;
        const double2 wa = bA(k), wb = bB(k);
        E.tA[2][p] = d * wa.x;
        E.tA[3][p] = d * wa.y;
        E.tA[0][p] = d * wb.x;
        E.tA[1][p] = d * wb.y;
    }
}

// ---------------------------------------------------------------------------
// Phase-2 filter of steady steps on the warp transform (filter_field,
// src/subpatch_data.cpp:30-44, src/runtime.cpp:403-421: rows then columns of
// rho, rho u, rho v, theta, then E rebuilt), the PassFR / PassFC pair of
// step_kernels.cu restated per warp. Rows: one row per warp, the conserved
// state -> (rho, rho u) | (rho v, theta) -> filter -> tF. Columns: one
// column quad per CTA, tF -> filter -> e, E = rho theta / (gamma - 1) +
// |m|^2 / (2 rho).

template <int NL>
FCSG_HD void wfilter_x_body(int lane, int line, double2* buf, const double2* mult, const EngineDev& E,
                            const double* blend, const unsigned short* st) {
    using namespace w280;
    constexpr int PPL = kN / NL;
    constexpr int KL = PPL >= 4 ? 4 : 1;
    const int ni = E.ni, nj = E.nj;
    const int sub = line / nj, row = line - sub * nj;
    const long rb = static_cast<long>(sub) * ni * nj + static_cast<long>(row) * ni;
    double2* bA = buf;
    double2* bB = buf + kBP;
#pragma unroll 1
    for (int m0 = 0; m0 < PPL; m0 += KL) {
        double v[KL][4];
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const long p = rb + lane + NL * (m0 + k);
#pragma unroll
            for (int c = 0; c < 4; ++c) v[k][c] = ldg1(E.e[c] + p);
        }
#pragma unroll
        for (int k = 0; k < KL; ++k) {
            const double rho = v[k][0], mx = v[k][1], my = v[k][2], En = v[k][3];
            const int s = st[lane + NL * (m0 + k)];
            bA[s] = mk2(rho, mx);
            bB[s] = mk2(my, kGm1 * (En - 0.5 * (mx * mx + my * my) / rho) / rho);
        }
    }
    FCSG_SYNCWARP();
    transform<NL, 2>(lane, buf, kBP, mult, blend);
#pragma unroll 4
    for (int m = 0; m < PPL; ++m) {
        const int i = lane + NL * m;
        const long p = rb + i;
        const int s = st[i];
        const double2 a = bA[s], b = bB[s];
        E.tF[0][p] = a.x;
        E.tF[1][p] = a.y;
        E.tF[2][p] = b.x;
        E.tF[3][p] = b.y;
    }
}

template <int NT>
FCSG_HD void wfilter_y_quad(int tid, int quad, double2* bufs, const double2* mult, const EngineDev& E,
                            const double* blend, const unsigned short* st) {
    using namespace w280;
    constexpr int PPT = kQuad * kN / NT;
    const int ni = E.ni, nj = E.nj;
    const int qps = (ni + kQuad - 1) / kQuad;
    const int sub = quad / qps, c0 = (quad - sub * qps) * kQuad;
    const long gb = static_cast<long>(sub) * ni * nj + c0;
    const int ncol = ni - c0 < kQuad ? ni - c0 : kQuad;
    auto col = [&](int k) { return (tid + NT * k) & (kQuad - 1); };
    auto row = [&](int k) { return (tid + NT * k) >> 2; };
    auto pt = [&](int k) { return gb + static_cast<long>(row(k)) * ni + col(k); };
    auto bA = [&](int k) -> double2& { return bufs[col(k) * 2 * kBP + st[row(k)]]; };
    auto bB = [&](int k) -> double2& { return bufs[col(k) * 2 * kBP + kBP + st[row(k)]]; };
#pragma unroll 4
    for (int k = 0; k < PPT; ++k) {
        const bool ok = col(k) < ncol;
        const long p = ok ? pt(k) : gb;
        bA(k) = ok ? mk2(ldg1(E.tF[0] + p), ldg1(E.tF[1] + p)) : mk2(1.0, 0.0);
        bB(k) = ok ? mk2(ldg1(E.tF[2] + p), ldg1(E.tF[3] + p)) : mk2(0.0, 1.0);
    }
    FCSG_SYNC();
#if FCSG_CUDA
    const int warp = tid >> 5;
    if (warp < kQuad) transform<32, 2>(tid & 31, bufs + warp * 2 * kBP, kBP, mult, blend);
#else
    for (int c = 0; c < kQuad; ++c) transform<1, 2>(0, bufs + c * 2 * kBP, kBP, mult, blend);
#endif
    FCSG_SYNC();
#pragma unroll 4
    for (int k = 0; k < PPT; ++k) {
        if (col(k) >= ncol) continue;
        const long p = pt(k);
        const double2 a = bA(k), b = bB(k);
        const double rho = a.x, mx = a.y, my = b.x;
        E.e[0][p] = rho;
        E.e[1][p] = mx;
        E.e[2][p] = my;
        E.e[3][p] = rho * b.y / kGm1 + 0.5 * (mx * mx + my * my) / rho;
    }
}

#if FCSG_CUDA
// pass X: CTA of kXWarps independent warps, each with two line buffers
constexpr int kXWarps = 4;
constexpr int kXThreads = kXWarps * 32;
constexpr size_t kXSmem = (kTabSlots + kXWarps * 2 * kBP) * sizeof(double2);
// pass Y: CTA = one column quad (4 warps), 8 line buffers
constexpr int kYThreads = kQuad * 32;
constexpr size_t kYSmem = (kTabSlots + kQuad * 2 * kBP) * sizeof(double2);

// Both kernels are persistent (grid = resident CTAs): a CTA stages the
// operator tables once and walks its work items, prefetching the next
// item's state into L2 before it starts on the current one.
__global__ void __launch_bounds__(kXThreads, FCSG_X_MINB) wpass_x_kernel(const __grid_constant__ EngineDev E,
                                                               const double2* __restrict__ mult_src,
                                                               const double* __restrict__ blend_src, int stage) {
    extern __shared__ double2 wsm[];
    double2* mult = wsm;
    double* blend = reinterpret_cast<double*>(wsm + w280::kNE);
    stage_w280_tables(threadIdx.x, kXThreads, mult_src, blend_src, mult, blend);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + kTabSlots + warp * 2 * kBP;
    const int nlines = E.S * E.nj;
    const int stride = gridDim.x * kXWarps;
    for (int line = blockIdx.x * kXWarps + warp; line < nlines; line += stride) {
        const int nxt = line + stride;
        if (nxt < nlines && lane < 4) {  // the next row's state (4 x 2 KB)
            const int sub = nxt / E.nj, row = nxt - sub * E.nj;
            pf_l2_bulk(E.e[lane] + static_cast<long>(sub) * E.ni * E.nj + static_cast<long>(row) * E.ni,
                       w280::kN * sizeof(double));
        }
        wpass_x_body<32>(lane, line, buf, mult, E, blend, slot_table(mult), stage);
    }
}

__global__ void __launch_bounds__(kYThreads, FCSG_Y_MINB) wpass_y_kernel(const __grid_constant__ EngineDev E,
                                                               const double2* __restrict__ mult_src,
                                                               const double* __restrict__ blend_src) {
    extern __shared__ double2 wsm[];
    double2* mult = wsm;
    double* blend = reinterpret_cast<double*>(wsm + w280::kNE);
    stage_w280_tables(threadIdx.x, kYThreads, mult_src, blend_src, mult, blend);
    const int qps = (E.ni + kQuad - 1) / kQuad;
    const int nquads = E.S * qps;
    for (int quad = blockIdx.x; quad < nquads; quad += gridDim.x) {
        const int nxt = quad + gridDim.x;
        if (nxt < nquads) {  // the next quad's state: one 32-byte sector per row and component
            const int sub = nxt / qps, c0 = (nxt - sub * qps) * kQuad;
            const long gb = static_cast<long>(sub) * E.ni * E.nj + c0;
            for (int r = threadIdx.x; r < 4 * w280::kN; r += kYThreads)
                pf_l2(E.e[r >> 8] + gb + static_cast<long>(r & (w280::kN - 1)) * E.ni);
        }
        __syncthreads();  // tables staged; the previous quad's buffers consumed
        wpass_y_quad<kYThreads>(threadIdx.x, quad, wsm + kTabSlots, mult, E, blend, slot_table(mult));
    }
}

__global__ void __launch_bounds__(kXThreads, 5) wfilter_x_kernel(const __grid_constant__ EngineDev E,
                                                                 const double2* __restrict__ mult_src,
                                                                 const double* __restrict__ blend_src) {
    extern __shared__ double2 wsm[];
    double2* mult = wsm;
    double* blend = reinterpret_cast<double*>(wsm + w280::kNE);
    stage_w280_tables(threadIdx.x, kXThreads, mult_src, blend_src, mult, blend);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + kTabSlots + warp * 2 * kBP;
    const int nlines = E.S * E.nj;
    for (int line = blockIdx.x * kXWarps + warp; line < nlines; line += gridDim.x * kXWarps)
        wfilter_x_body<32>(lane, line, buf, mult, E, blend, slot_table(mult));
}

__global__ void __launch_bounds__(kYThreads, 5) wfilter_y_kernel(const __grid_constant__ EngineDev E,
                                                                 const double2* __restrict__ mult_src,
                                                                 const double* __restrict__ blend_src) {
    extern __shared__ double2 wsm[];
    double2* mult = wsm;
    double* blend = reinterpret_cast<double*>(wsm + w280::kNE);
    stage_w280_tables(threadIdx.x, kYThreads, mult_src, blend_src, mult, blend);
    const int nquads = E.S * ((E.ni + kQuad - 1) / kQuad);
    for (int quad = blockIdx.x; quad < nquads; quad += gridDim.x) {
        __syncthreads();
        wfilter_y_quad<kYThreads>(threadIdx.x, quad, wsm + kTabSlots, mult, E, blend, slot_table(mult));
    }
}

// resident CTAs of a kernel (grid of the persistent launches), per device
template <class K>
int resident_ctas(K kernel, int threads, size_t smem, unsigned long long* done, int* cache) {
    int d = 0;
    cudaGetDevice(&d);
    if (dev::first_on_device(done)) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
        if (const char* v = std::getenv("FCSG_WPASS_MAX_CTAS")) per = std::min(per, std::atoi(v));  // experiments
        cache[d & 63] = sms * (per > 0 ? per : 1);
    }
    return cache[d & 63];
}
// the persistent grid under a view's cap of CTAs per SM
inline int capped_grid(int resident, int cap) {
    if (cap <= 0) return resident;
    int d = 0, sms = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    return std::min(resident, cap * sms);
}
#endif

bool wpass_applies(const EngineDev& E, const FcPlanDev& pl, bool rows) {
    return pl.n_ext == 280 && pl.n == 256 && pl.n_gap == 24 && pl.dp1 == 3 && pl.mult_pfa != nullptr &&
           (rows ? E.ni : E.nj) == 256;
}

void launch_wpass(const EngineDev& E, const FcPlanDev& pl, bool rows, int stage, void* stream) {
    const int nlines = E.S * (rows ? E.nj : E.ni);
    if (nlines == 0) return;
    // A/B: FCSG_WPASS_CT=1 runs the passes on the register-resident 8 x 35
    // transform (wctpass.cu). Measured slower on the B200 (config 5: pass Y
    // 0.36 ms, pass X 0.32 ms against 0.22 / 0.21 ms here): 35 complex values
    // per lane leave 8 warps per SM, too few to cover the FP64 dependency
    // chains -- so the prime-factor kernels stay the default.
    static const bool ct = [] {
        const char* v = std::getenv("FCSG_WPASS_CT");
        return v && v[0] == '1';
    }();
    if (ct) {
        launch_wctpass(E, pl, rows, stage, stream);
        return;
    }
    const double2* mult = pl.mult_pfa;  // mode 1: d/dq
    const int nquads = E.S * ((E.ni + kQuad - 1) / kQuad);
#if FCSG_CUDA
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static unsigned long long done = 0, occ_x = 0, occ_y = 0;
    static int res_x[64], res_y[64];
    if (dev::first_on_device(&done)) {
        cudaFuncSetAttribute(wpass_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kXSmem));
        cudaFuncSetAttribute(wpass_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kYSmem));
    }
    if (rows) {
        const int need = (nlines + kXWarps - 1) / kXWarps;
        const int grid = std::min(need, capped_grid(resident_ctas(wpass_x_kernel, kXThreads, kXSmem, &occ_x, res_x), E.wpass_cap));
        wpass_x_kernel<<<grid, kXThreads, kXSmem, s>>>(E, mult, pl.blend, stage);
    } else {
        const int grid = std::min(nquads, capped_grid(resident_ctas(wpass_y_kernel, kYThreads, kYSmem, &occ_y, res_y), E.wpass_cap));
        wpass_y_kernel<<<grid, kYThreads, kYSmem, s>>>(E, mult, pl.blend);
    }
#else
    (void)stream;
    if (rows) {
        std::vector<double2> buf(2 * kBP);
        for (int line = 0; line < nlines; ++line)
            wpass_x_body<1>(0, line, buf.data(), mult, E, pl.blend, host_slot_table(), stage);
    } else {
        std::vector<double2> bufs(kQuad * 2 * kBP);
        for (int q = 0; q < nquads; ++q) wpass_y_quad<1>(0, q, bufs.data(), mult, E, pl.blend, host_slot_table());
    }
#endif
}

void launch_wfilter(const EngineDev& E, const FcPlanDev& pl, bool rows, void* stream) {
    const int nlines = E.S * (rows ? E.nj : E.ni);
    if (nlines == 0) return;
    const double2* mult = pl.mult_pfa + 2 * w280::kNE;  // mode 3: the per-step filter
    const int nquads = E.S * ((E.ni + kQuad - 1) / kQuad);
#if FCSG_CUDA
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static unsigned long long done = 0, occ_x = 0, occ_y = 0;
    static int res_x[64], res_y[64];
    if (dev::first_on_device(&done)) {
        cudaFuncSetAttribute(wfilter_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kXSmem));
        cudaFuncSetAttribute(wfilter_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kYSmem));
    }
    if (rows) {
        const int need = (nlines + kXWarps - 1) / kXWarps;
        const int grid = std::min(need, capped_grid(resident_ctas(wfilter_x_kernel, kXThreads, kXSmem, &occ_x, res_x), E.wpass_cap));
        wfilter_x_kernel<<<grid, kXThreads, kXSmem, s>>>(E, mult, pl.blend);
    } else {
        const int grid = std::min(nquads, capped_grid(resident_ctas(wfilter_y_kernel, kYThreads, kYSmem, &occ_y, res_y), E.wpass_cap));
        wfilter_y_kernel<<<grid, kYThreads, kYSmem, s>>>(E, mult, pl.blend);
    }
#else
    (void)stream;
    if (rows) {
        std::vector<double2> buf(2 * kBP);
        for (int line = 0; line < nlines; ++line)
            wfilter_x_body<1>(0, line, buf.data(), mult, E, pl.blend, host_slot_table());
    } else {
        std::vector<double2> bufs(kQuad * 2 * kBP);
        for (int q = 0; q < nquads; ++q) wfilter_y_quad<1>(0, q, bufs.data(), mult, E, pl.blend, host_slot_table());
    }
#endif
}

}  // namespace fcsg
