#pragma once

#include <algorithm>
#include <cstddef>
#include <vector>

#include "fcsg_common.h"

namespace fcsg {

struct FcLinesArgs {
    FcPlanDev pl;
    int mode;          // 1 d/dq, 2 d2/dq2, 3 filter, 4 smear filter
    const double* in;  // line l, element i at in[l*line_stride + i*stride]
    double* out;       // line l, element i at out[l*out_line_stride + i*out_stride]; in == out allowed
    long line_stride;
    long stride;
    long out_line_stride;
    long out_stride;
    long n_lines;
    double scale;      // multiplies every output (inv_len^order for derivatives)
    int scr_cap;       // complex scratch slots for generic-radix stages (set by the launcher)
};

size_t fc_lines_smem_bytes(const FcPlanDev& pl, int LB, int scr_cap);
int fc_lines_scr_cap(const FcPlanDev& pl, int LB);
void launch_fc_lines(FcLinesArgs a, int LB, void* stream);
// the warp-per-line prime-factor kernel (wpass.cu) for the N = 256 reference
// operator (n_ext = 280); launch_fc_lines takes it when it applies
bool w280_lines_applies(const FcPlanDev& pl);
void launch_w280_lines(const FcLinesArgs& a, void* stream);
// the register-resident 8 x 35 kernel (wct280.h) for rows (stride 1) of the
// same operator; launch_fc_lines prefers it
bool wct_lines_applies(const FcLinesArgs& a);
void launch_wct_lines(const FcLinesArgs& a, void* stream);
// the same batches on the register-resident 14 x 20 transform (w20lines.cu:
// four real lines per warp, half the registers): FCSG_LINES_KERNEL=20, an A/B
// variant (measured slower than the 8 x 35 kernel at every batch size)
void launch_w20_lines(const FcLinesArgs& a, void* stream);

}  // namespace fcsg
