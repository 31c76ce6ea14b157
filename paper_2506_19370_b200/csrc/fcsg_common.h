// Common definitions shared by the sm_100a kernels and their host launchers.
//
// Every kernel body in this directory is written as an FCSG_HD function that
// takes an explicit (tid, nthr) thread context and a shared-memory pointer, so
// the identical source also compiles as plain C++ (FCSG_EMULATE) for the
// CPU unit-test harness (tests/, libfcsg_emu.so). The product library
// libfcsg.so is always the nvcc build; nothing in the package loads the
// emulation build.
#pragma once

#include <cstdint>

#if defined(__CUDACC__) && !defined(FCSG_EMULATE)
// device compile of the product: kernel bodies are device code
#include <cuda_runtime.h>
#define FCSG_HD __device__ __forceinline__
#define FCSG_DEV __device__ __forceinline__
#define FCSG_SYNC() __syncthreads()
#define FCSG_CUDA 1
#else
#include <cmath>
#include <cstring>
#define FCSG_HD inline
#define FCSG_DEV inline
#define FCSG_SYNC() ((void)0)
#define FCSG_CUDA 0
#if !defined(FCSG_EMULATE)
#include <vector_types.h>  // host TU of the product: CUDA's double2
#elif !defined(__CUDACC__)
struct double2 {
    double x, y;
};
#endif
#endif

namespace fcsg {

// error kinds, shared with include/fcsg.h and the reference's exception types
// (include/fcs/errors.hpp:10-43)
enum ErrKind : int {
    kOk = 0,
    kConfig = 1,
    kUsage = 2,
    kGeometry = 3,
    kDecomposition = 4,
    kInvalidState = 5,
    kCuda = 8,
    kOther = 9,
};

// device error word (first failure wins): code and either (storage slot of
// the subpatch, i, j) or, from the kernels over all points, the global point
// index gp (>= 0; the host maps it back to (subpatch, i, j))
struct DevError {
    int code;  // 0 = none; 1 = nonpositive density or pressure (rhs), 2 = proxy/MWSB, 3 = nonfinite wave speed
    int sub;
    int i;
    int j;
    long long gp;
};

struct Thr {
    int tid;
    int nthr;
};

FCSG_HD double2 mk2(double a, double b) {
    double2 r;
    r.x = a;
    r.y = b;
    return r;
}
FCSG_HD double2 cadd(double2 a, double2 b) { return mk2(a.x + b.x, a.y + b.y); }
FCSG_HD double2 csub(double2 a, double2 b) { return mk2(a.x - b.x, a.y - b.y); }
FCSG_HD double2 cmul(double2 a, double2 b) { return mk2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
// a * conj(b)
FCSG_HD double2 cmulc(double2 a, double2 b) { return mk2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }
FCSG_HD double2 cscale(double2 a, double s) { return mk2(a.x * s, a.y * s); }

constexpr int kMaxStages = 12;

// FFT stage radices of length n, largest-first among the register radices
// (8, 4, 2, 9, 3, 5, 7, 11, 13), then the remaining primes (direct DFT).
// Shared by the host tables (digit-reversal order of the multiplier table)
// and the compile-time device plans, so both always agree.
struct Factors {
    int n = 0;
    int r[kMaxStages] = {};
    int span[kMaxStages] = {};
};
#if defined(__CUDACC__)
__host__ __device__
#endif
constexpr Factors factor_stages(int len) {
    Factors f{};
    int m = len;
    while (m % 8 == 0 && f.n < kMaxStages) { f.r[f.n++] = 8; m /= 8; }
    if (m % 4 == 0) { f.r[f.n++] = 4; m /= 4; }
    if (m % 2 == 0) { f.r[f.n++] = 2; m /= 2; }
    while (m % 9 == 0 && f.n < kMaxStages) { f.r[f.n++] = 9; m /= 9; }
    const int small[5] = {3, 5, 7, 11, 13};
    for (int k = 0; k < 5; ++k)
        while (m % small[k] == 0 && f.n < kMaxStages) { f.r[f.n++] = small[k]; m /= small[k]; }
    for (int p = 17; p * p <= m; p += 2)
        while (m % p == 0 && f.n < kMaxStages) { f.r[f.n++] = p; m /= p; }
    if (m > 1 && f.n < kMaxStages) f.r[f.n++] = m;
    if (f.n == 0) f.r[f.n++] = 1;
    int L = len;
    for (int s = 0; s < f.n; ++s) {
        f.span[s] = L;
        L /= f.r[s];
    }
    return f;
}
constexpr int kMaxGap = 64;     // n_cont - 1
constexpr int kFbMinWindow = 12;  // fallback classifier: shorter windows are class 4 (src/viscosity.cpp:164)
constexpr int kFbMaxWindow = 64;  // fallback classifier: longest supported window
constexpr int kMaxDeg = 6;      // degree + 1 <= 7

// Device-side description of one FC operator (n points, n_cont, degree):
// FFT plan over n_ext = n + n_cont - 1 plus the continuation and spectral
// multiplier tables (see fc_tables.cpp for how each table restates
// src/fc_core.cpp).
struct FcPlanDev {
    int n;        // points per line (N)
    int n_ext;    // FFT length
    int n_gap;    // n_cont - 1
    int dp1;      // degree + 1 boundary points used by the continuation
    int nstages;
    int radix[kMaxStages];
    int span[kMaxStages];
    const double2* tw;      // exp(-2 pi i k / n_ext), k < n_ext
    const double* blend;    // n_gap x dp1, row-major (FcOperator::blend_matrix)
    const double2* mult;    // 4 x n_ext multipliers in DIF output order: d1, d2, filter, smear
    const double2* mult_pfa;  // n_ext = 280 only (else null): the same 4 tables in the prime-factor
                              // order (k1, k2, k3) of wline.h, k3 fastest
    const double2* prime_frag;  // last radix P a large prime (else null): the (cos, sin)(2 pi q r / P) operand
                                // fragments of the tensor-core DFT, [m-tile][k-step][lane] (fc_tables.cpp)
};

}  // namespace fcsg
