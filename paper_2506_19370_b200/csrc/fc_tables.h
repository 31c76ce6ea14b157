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
    std::vector<double2> mult_pfa;       // n_ext = 280: 4 x 280 in the (k1, k2, k3) order of wline.h
    std::vector<double2> prime_frag;     // last radix P >= 17: (cos, sin)(2 pi q r / P) per lane of the DMMA A
                                         // fragments, [m-tile][k-step][lane] (fft_line.h middle_dmma_ct)
};

// Blend-to-zero matrix for Gram degree d (d = 2 is the reference's
// FcOperator::blend_matrix, src/fc_core.cpp:55-163).
std::vector<double> build_blend_matrix(int n_cont, int degree);

// FcOperator constructor semantics (src/fc_core.cpp:190-217) plus the FFT
// plan and multiplier tables of this implementation.
FcTables build_fc_tables(int n_points, int n_cont, int degree, FilterSpec f);

// FC-spectrum ("fallback") classifier, one window length w (<= 64):
// Classifier::classify_line's variant (src/viscosity.cpp:161-208) over
// FcOperator::spectrum (src/fc_core.cpp:308-316) of OperatorCache::get(w)
// (n_cont 25, degree 2). Only the top quarter of the modes, k in [k_lo, nb),
// enters the decision, and continuation + DFT restricted to those modes is one
// linear map of the window: T[i][2 (k - k_lo) + {0, 1}] = (Re, Im) of the
// contribution of window value i to c_k (no 1/n_ext; the caller divides |c_k|
// like the reference). Layout of one table (doubles): T (w x 2 nk, i-major),
// then lx[nk] = log(k), then sx, sxx (the fit's constant sums, accumulated in
// the reference's order).
struct SpectrumTail {
    int w = 0, n_ext = 0, nb = 0, k_lo = 0, nk = 0;
    std::vector<double> table;
};
SpectrumTail build_spectrum_tail(int w, int n_cont);

}  // namespace fcsg
