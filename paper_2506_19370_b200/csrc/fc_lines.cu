// Batched FC line operator: the drop-in for FcOperator::derivative / filter /
// strong_filter (src/fc_core.cpp:257-306) applied over many lines at once.
// One CTA owns LB complex lines = 2*LB real lines; real lines (2a, 2a+1) are
// packed as one complex line, transformed with fc_transform (fft_line.h), and
// unpacked. Loads/stores are coalesced along whichever axis is contiguous:
// along the line for stride==1 (rows), across lines when line_stride==1
// (columns of a row-major field; then thread w takes point w / LB of line
// w % LB, the shared-memory order).
#include <cstdlib>

#include "dev.h"
#include "fc_lines.h"
#include "fft_line.h"

namespace fcsg {

template <int LB, int NE, int NTHR>
FCSG_HD void fc_lines_body(Thr t, int block, double2* smem, const FcLinesArgs& a) {
    const FcPlanDev& pl = a.pl;
    constexpr int pitch = LB;  // line index fastest, no padding: see fft_line.h
    double2* buf = smem;
    double2* scr = smem + (NE > 0 ? NE : pl.n_ext) * pitch;
    const FcPlanDev spl = stage_tables(Thr{t.tid, NTHR}, pl, a.mode, scr + a.scr_cap);
    const int N = NE > 0 ? NE - ct_gap(NE) : pl.n;
    const long l0 = static_cast<long>(block) * 2 * LB;
    const long ls = a.line_stride, st = a.stride;
    const long ols = a.out_line_stride, ost = a.out_stride;
    const int total = N * LB;
    const bool rows = (st == 1), orows = (ost == 1);
#pragma unroll 4
    for (int w = t.tid; w < total; w += NTHR) {
        const int c = rows ? w / N : w % LB, i = rows ? w % N : w / LB;
        const long l = l0 + 2 * c;
        double v0 = 0.0, v1 = 0.0;
        if (l < a.n_lines) v0 = ldg1(a.in + l * ls + i * st);
        if (l + 1 < a.n_lines) v1 = ldg1(a.in + (l + 1) * ls + i * st);
        buf[i * pitch + c] = mk2(v0, v1);
    }
    FCSG_SYNC();
    if constexpr (NE > 0) fc_transform_ct<NE, LB, NTHR>(t.tid, buf, spl, a.mode, scr, a.scr_cap);
    else fc_transform(Thr{t.tid, NTHR}, buf, pitch, LB, spl, a.mode, scr, a.scr_cap);
#pragma unroll 4
    for (int w = t.tid; w < total; w += NTHR) {
        const int c = orows ? w / N : w % LB, i = orows ? w % N : w / LB;
        const long l = l0 + 2 * c;
        const double2 v = buf[i * pitch + c];
        if (l < a.n_lines) a.out[l * ols + i * ost] = v.x * a.scale;
        if (l + 1 < a.n_lines) a.out[(l + 1) * ols + i * ost] = v.y * a.scale;
    }
}

#if FCSG_CUDA
template <int LB, int NE>
__global__ void __launch_bounds__(256, NE > 0 ? 3 : 2) fc_lines_kernel(const __grid_constant__ FcLinesArgs a) {
    extern __shared__ double2 smem[];
    fc_lines_body<LB, NE, 256>(Thr{static_cast<int>(threadIdx.x), 256}, blockIdx.x, smem, a);
}

template <int LB, int NE>
void launch_fc_lines_t(const FcLinesArgs& a, int nblk, size_t smem, cudaStream_t s) {
    static unsigned long long done = 0;  // per device (function attributes are per device)
    if (dev::first_on_device(&done)) {
        cudaFuncSetAttribute(fc_lines_kernel<LB, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(fc_lines_kernel<LB, NE>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    fc_lines_kernel<LB, NE><<<nblk, 256, smem, s>>>(a);
}

template <int LB>
void launch_fc_lines_lb(const FcLinesArgs& a, int nblk, size_t smem, cudaStream_t s) {
    const bool ct = ct_plan_for(a.pl);
    if (ct && a.pl.n_ext == 280) launch_fc_lines_t<LB, 280>(a, nblk, smem, s);
    else if (ct && a.pl.n_ext == 536) launch_fc_lines_t<LB, 536>(a, nblk, smem, s);
    else if (ct && a.pl.n_ext == 282) launch_fc_lines_t<LB, 282>(a, nblk, smem, s);
    else if (ct && a.pl.n_ext == 171) launch_fc_lines_t<LB, 171>(a, nblk, smem, s);
    else launch_fc_lines_t<LB, 0>(a, nblk, smem, s);
}
#endif

size_t fc_lines_smem_bytes(const FcPlanDev& pl, int LB, int scr_cap) {
    return (static_cast<size_t>(pl.n_ext) * LB + scr_cap + table_slots_host(pl)) * sizeof(double2);
}

int fc_lines_scr_cap(const FcPlanDev& pl, int LB) {
    int cap = 0;
    for (int s = 0; s < pl.nstages; ++s) {
        const int p = pl.radix[s];
        const bool reg = p == 2 || p == 3 || p == 4 || p == 5 || p == 7 || p == 8 || p == 9 || p == 11 || p == 13;
        if (!reg) cap = std::max(cap, p * LB * std::max(1, 256 / (p * LB)));
    }
    return cap;
}

constexpr long kW20MaxLines = 0;

void launch_fc_lines(FcLinesArgs a, int LB, void* stream) {
    if (wct_lines_applies(a) && !std::getenv("FCSG_NO_WCT_LINES") && !std::getenv("FCSG_NO_WARP_LINES")) {
        // register-resident transforms: 8 x 35 (eight lines per warp), or
        // 14 x 20 (four lines per warp, half the registers) with
        // FCSG_LINES_KERNEL=20 -- an A/B variant, measured slower at every
        // batch size (config 1: 10.4 against 8.3 us per call; 262144 lines:
        // 3785 against 4299 GB/s), so kW20MaxLines = 0
        static const int pick = [] {
            const char* v = std::getenv("FCSG_LINES_KERNEL");
            return v ? std::atoi(v) : 0;
        }();
        if (pick == 20 || (pick == 0 && a.n_lines <= kW20MaxLines)) launch_w20_lines(a, stream);
        else launch_wct_lines(a, stream);
        return;
    }
    if (w280_lines_applies(a.pl) && !std::getenv("FCSG_NO_WARP_LINES")) {
        launch_w280_lines(a, stream);
        return;
    }
#if !FCSG_CUDA
    LB = 4;  // the emulation runs one block shape
#endif
    const int lines_per_block = 2 * LB;
    const int nblk = static_cast<int>((a.n_lines + lines_per_block - 1) / lines_per_block);
    if (nblk == 0) return;
    a.scr_cap = fc_lines_scr_cap(a.pl, LB);
    if (ct_plan_for(a.pl)) a.scr_cap = std::max(a.scr_cap, ct_scratch_slots(a.pl.n_ext, LB));
    const size_t smem = fc_lines_smem_bytes(a.pl, LB, a.scr_cap);
#if FCSG_CUDA
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (LB) {
        case 4: launch_fc_lines_lb<4>(a, nblk, smem, s); break;
        case 5: launch_fc_lines_lb<5>(a, nblk, smem, s); break;
        case 6: launch_fc_lines_lb<6>(a, nblk, smem, s); break;
        case 8: launch_fc_lines_lb<8>(a, nblk, smem, s); break;
        default: launch_fc_lines_lb<16>(a, nblk, smem, s); break;
    }
#else
    (void)stream;
    std::vector<double2> sm(smem / sizeof(double2));
    // same plan dispatch as the CUDA build, so the emulation covers the
    // compile-time plans too
    const int ne = ct_plan_for(a.pl) ? a.pl.n_ext : 0;
    for (int b = 0; b < nblk; ++b) {
        if (ne == 280) fc_lines_body<4, 280, 1>(Thr{0, 1}, b, sm.data(), a);
        else if (ne == 536) fc_lines_body<4, 536, 1>(Thr{0, 1}, b, sm.data(), a);
        else if (ne == 282) fc_lines_body<4, 282, 1>(Thr{0, 1}, b, sm.data(), a);
        else if (ne == 171) fc_lines_body<4, 171, 1>(Thr{0, 1}, b, sm.data(), a);
        else fc_lines_body<4, 0, 1>(Thr{0, 1}, b, sm.data(), a);
    }
#endif
}

}  // namespace fcsg
