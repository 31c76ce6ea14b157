// FC line batch on the register-resident 14 x 20 transform (wct20.h): four
// real lines (two complex) per warp, rows only (stride 1 in and out: lane
// (l, q) reads and writes positions q + 14 t of its lines straight from and to
// global memory). FcOperator::derivative / filter / strong_filter over a batch
// of lines, src/fc_core.cpp:257-306. Three warp phases separated by
// __syncwarp: P1 loads, continuation, DFT-20 -> shared memory; P2 the 40
// DFT-14 groups with the multiplier; P3 shared memory -> inverse DFT-20 ->
// stores. Against the 8 x 35 kernel (wpass.cu: wct_lines_kernel): half the
// registers and half the work per warp, twice the warps -- built to shorten
// config 1's per-warp latency chain, and measured SLOWER at every batch size
// (config 1: 10.4 against 8.3 us per call; 262144 lines: 3785 against 4299
// GB/s): 4 of 32 lanes idle, the second DFT-14 iteration a quarter full, and
// config 1 is bound by launch ramp + first DRAM access + table staging, not
// by the chain. Kept as an A/B variant (FCSG_LINES_KERNEL=20), parity-tested.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dev.h"
#include "fc_lines.h"
#include "wct20.h"
#include "wpass_common.h"

namespace fcsg {

namespace {

struct W20Lane {
    int l, q;
    bool active, h0, h1;
    long l0;
};
FCSG_HD W20Lane w20_lane(int lane, long unit, const FcLinesArgs& a) {
    W20Lane L;
    L.active = lane < w20::kActive;
    L.l = L.active ? lane / w20::kQ : 0;
    L.q = lane - w20::kQ * (lane / w20::kQ);
    L.l0 = 4 * unit + 2 * L.l;
    L.h0 = L.active && L.l0 < a.n_lines;
    L.h1 = L.active && L.l0 + 1 < a.n_lines;
    return L;
}

// the line's own points of lane (l, q): t < 18, and t = 18 for q < 4
FCSG_HD void w20_load(const W20Lane& L, const FcLinesArgs& a, double2 (&z)[w20::kT]) {
    const double* p0 = a.in + (L.h0 ? L.l0 : 0) * a.line_stride + L.q;
    const double* p1 = a.in + (L.h1 ? L.l0 + 1 : 0) * a.line_stride + L.q;
#pragma unroll
    for (int t = 0; t < 18; ++t) z[t] = mk2(L.h0 ? ldg1(p0 + 14 * t) : 0.0, L.h1 ? ldg1(p1 + 14 * t) : 0.0);
    const bool tail = L.q < 4;
    z[18] = mk2(L.h0 && tail ? ldg1(p0 + 252) : 0.0, L.h1 && tail ? ldg1(p1 + 252) : 0.0);
    z[19] = mk2(0.0, 0.0);
}

// boundary samples of the lane's line: f[253 + i] = z[18] of lane q = 1 + i,
// f[2 - i] = z[0] of lane q = 2 - i (of the line's lane group)
#if FCSG_CUDA
__device__ __forceinline__ void w20_ends(int lane, const double2 (&z)[w20::kT], double2 (&fr)[w20::kD1],
                                         double2 (&fl)[w20::kD1]) {
    const int g = (lane / w20::kQ) * w20::kQ;  // lanes 28-31: g = 28 (their values are unused)
#pragma unroll
    for (int i = 0; i < w20::kD1; ++i) {
        const int sr = (g + 1 + i) & 31, sl = (g + 2 - i) & 31;
        fr[i] = mk2(__shfl_sync(0xffffffffu, z[18].x, sr), __shfl_sync(0xffffffffu, z[18].y, sr));
        fl[i] = mk2(__shfl_sync(0xffffffffu, z[0].x, sl), __shfl_sync(0xffffffffu, z[0].y, sl));
    }
}
#endif

FCSG_HD void w20_p1(const W20Lane& L, double2 (&z)[w20::kT], const double2 (&fr)[w20::kD1],
                    const double2 (&fl)[w20::kD1], const double* blend, double2* buf) {
    w20::continuation(L.q, z, fr, fl, blend);
    w20::dft20<false>(z);
    if (L.active) w20::put20(buf, L.l, L.q, z);
}

FCSG_HD void w20_p3(const W20Lane& L, const FcLinesArgs& a, const double2* buf) {
    if (!L.active) return;
    double2 z[w20::kT];
    w20::get20(buf, L.l, L.q, z);
    w20::dft20<true>(z);
    double* q0 = a.out + L.l0 * a.out_line_stride + L.q;
    double* q1 = q0 + a.out_line_stride;
    const double s = a.scale;
#pragma unroll
    for (int t = 0; t < 19; ++t) {
        if (t == 18 && L.q >= 4) break;
        if (L.h0) q0[14 * t] = z[t].x * s;
        if (L.h1) q1[14 * t] = z[t].y * s;
    }
}

#if FCSG_CUDA
__device__ __forceinline__ void w20_griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void w20_griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <int WPC>
__global__ void __launch_bounds__(WPC * 32) w20_lines_kernel(const __grid_constant__ FcLinesArgs a) {
    extern __shared__ double2 wsm[];
    double2* tabs = wsm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* buf = wsm + w20::kTabSlots + warp * w20::kBufSlots;
    const long nunits = (a.n_lines + 3) / 4;
    const double* blend = reinterpret_cast<const double*>(tabs + w20::kNE + w20::kTwSlots);
    const long stride = static_cast<long>(gridDim.x) * WPC;
    long unit = static_cast<long>(blockIdx.x) * WPC + warp;
    double2 z[w20::kT];
    W20Lane L = w20_lane(lane, unit, a);
    {
        // programmatic dependent launch: everything before the wait reads only
        // the operator tables (written once at operator creation)
        w20::TableRegs<WPC * 32> tr;
        tr.load(threadIdx.x, a.pl.mult_pfa + (a.mode - 1) * w20::kNE, a.pl.tw, a.pl.blend);
        w20_griddep_wait();
        if (unit < nunits) w20_load(L, a, z);
        w20_griddep_launch();
        tr.store(threadIdx.x, tabs);
    }
    __syncthreads();
    auto body = [&]() {
        double2 fr[w20::kD1], fl[w20::kD1];
        w20_ends(lane, z, fr, fl);
        w20_p1(L, z, fr, fl, blend, buf);
        __syncwarp();
        w20::middle(lane, buf, tabs + w20::kNE, tabs);
        __syncwarp();
        w20_p3(L, a, buf);
        __syncwarp();
    };
    auto prefetch_next = [&](long u) {  // batches beyond one wave: the next unit's four rows into L2
        const long nxt = u + stride;
        if (nxt < nunits && L.active && L.q == 0) {
            const long l0 = 4 * nxt + 2 * L.l;
            if (l0 < a.n_lines) pf_l2_bulk(a.in + l0 * a.line_stride, w20::kN * sizeof(double));
            if (l0 + 1 < a.n_lines) pf_l2_bulk(a.in + (l0 + 1) * a.line_stride, w20::kN * sizeof(double));
        }
    };
    if (unit < nunits) {
        prefetch_next(unit);
        body();
    }
    for (unit += stride; unit < nunits; unit += stride) {
        L = w20_lane(lane, unit, a);
        w20_load(L, a, z);
        prefetch_next(unit);
        body();
    }
}

template <int WPC>
void launch_w20_variant(const FcLinesArgs& a, cudaStream_t s, bool pdl) {
    static unsigned long long done = 0;
    static int resident[64];
    constexpr size_t smem = (w20::kTabSlots + WPC * w20::kBufSlots) * sizeof(double2);
    int d = 0;
    cudaGetDevice(&d);
    if (dev::first_on_device(&done)) {
        cudaFuncSetAttribute(w20_lines_kernel<WPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, w20_lines_kernel<WPC>, WPC * 32, smem);
        resident[d & 63] = sms * (per > 0 ? per : 1);
    }
    const long nunits = (a.n_lines + 3) / 4;
    const long nblk = (nunits + WPC - 1) / WPC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<long>(nblk, resident[d & 63])));
    cfg.blockDim = dim3(WPC * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, w20_lines_kernel<WPC>, a);
}
#endif

}  // namespace

void launch_w20_lines(const FcLinesArgs& a, void* stream) {
    if (a.n_lines == 0) return;
#if FCSG_CUDA
    static const int wpc = [] {  // A/B experiments: FCSG_W20_WPC = warps per CTA
        const char* v = std::getenv("FCSG_W20_WPC");
        return v ? std::atoi(v) : 4;
    }();
    static const bool pdl = !std::getenv("FCSG_NO_PDL");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (wpc) {
        case 2: launch_w20_variant<2>(a, s, pdl); break;
        case 8: launch_w20_variant<8>(a, s, pdl); break;
        default: launch_w20_variant<4>(a, s, pdl); break;
    }
#else
    (void)stream;
    std::vector<double2> tabs(w20::kTabSlots), buf(w20::kBufSlots);
    w20::stage_tables(0, 1, a.pl.mult_pfa + (a.mode - 1) * w20::kNE, a.pl.tw, a.pl.blend, tabs.data());
    const double* blend = reinterpret_cast<const double*>(tabs.data() + w20::kNE + w20::kTwSlots);
    const long nunits = (a.n_lines + 3) / 4;
    std::vector<double2> zz(32 * w20::kT);
    struct Ends {
        double2 fr[w20::kD1], fl[w20::kD1];
    };
    Ends ends_[32];
    auto Z = [&](int lane) -> double2(&)[w20::kT] { return *reinterpret_cast<double2(*)[w20::kT]>(&zz[lane * w20::kT]); };
    for (long unit = 0; unit < nunits; ++unit) {
        W20Lane L[32];
        for (int lane = 0; lane < 32; ++lane) {
            L[lane] = w20_lane(lane, unit, a);
            w20_load(L[lane], a, Z(lane));
        }
        for (int lane = 0; lane < w20::kActive; ++lane) {  // ends from the lane group's registers, as the shuffles do
            const int g = (lane / w20::kQ) * w20::kQ;
            double2 fr[w20::kD1], fl[w20::kD1];
            for (int i = 0; i < w20::kD1; ++i) {
                fr[i] = Z(g + 1 + i)[18];
                fl[i] = Z(g + 2 - i)[0];
            }
            // the ends read z[18] (q = 1..3) and z[0], which no lane's continuation rewrites (q >= 4 only),
            // but the DFT rewrites all of z: gather first, transform in a second loop
            ends_[lane] = {{fr[0], fr[1], fr[2]}, {fl[0], fl[1], fl[2]}};
        }
        for (int lane = 0; lane < w20::kActive; ++lane) {
            double2 fr[w20::kD1], fl[w20::kD1];
            for (int i = 0; i < w20::kD1; ++i) {
                fr[i] = ends_[lane].fr[i];
                fl[i] = ends_[lane].fl[i];
            }
            w20_p1(L[lane], Z(lane), fr, fl, blend, buf.data());
        }
        for (int lane = 0; lane < 32; ++lane) w20::middle(lane, buf.data(), tabs.data() + w20::kNE, tabs.data());
        for (int lane = 0; lane < w20::kActive; ++lane) w20_p3(L[lane], a, buf.data());
    }
#endif
}

}  // namespace fcsg
