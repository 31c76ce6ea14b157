// Host-side construction of the FC operator tables (init time only).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "fcsg_common.h"

namespace fcsg {

struct Error : std::runtime_error {
    int kind;
    Error(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

// include/fcs/fc_core.hpp:11-15
struct FilterSpec {
    double alpha = 23.025850929940457;
    int p = 7;
    int p_smear = 2;
};

// Everything one FcOperator needs, in host memory.
struct FcTables {
    int n = 0, n_cont = 0, degree = 2;
    FilterSpec filter;
    int n_ext = 0, n_modes = 0;
    double period = 0.0;
    std::vector<double> blend;           // (n_cont-1) x (degree+1)
    std::vector<double> filter_profile;  // n_modes
    std::vector<double> smear_profile;   // n_modes
    std::vector<int> radix, span;        // FFT stages
    std::vector<int> freq_of_pos;        // DIF output position -> frequency index
    std::vector<double2> tw;             // n_ext
    std::vector<double2> mult;           // 4 x n_ext (d1, d2, filter, smear) in position order
};

// Blend-to-zero matrix for Gram degree d (d = 2 is the reference's
// FcOperator::blend_matrix, src/fc_core.cpp:55-163).
std::vector<double> build_blend_matrix(int n_cont, int degree);

// FcOperator constructor semantics (src/fc_core.cpp:190-217) plus the FFT
// plan and multiplier tables of this implementation.
FcTables build_fc_tables(int n_points, int n_cont, int degree, FilterSpec f);

}  // namespace fcsg
