// FP32-screened steady-step classifier (classify_f32.cu).
#pragma once

#include <vector>

#include "mlp_common.h"
#include "step_kernels.h"

namespace fcsg {

// the MLP weights rounded to float, FCNN order; passed by value as a kernel
// parameter (4 KB: the constant bank)
struct MlpF32 {
    float w[kMlpWeights];
};
MlpF32 mlp_f32_weights(const std::vector<double>& packed);
// logit margin above which the FP32 pass's argmax is exact (2x a rigorous
// error bound); EngineDev::cls_margin32
double mlp_f32_margin(const std::vector<double>& packed);
// tau and mu_hat of every point of E (steady steps, ann variant)
void launch_classify_f32(const EngineDev& E, const MlpF32& W, void* stream);

}  // namespace fcsg
