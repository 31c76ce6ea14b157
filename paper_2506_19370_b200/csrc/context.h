// Host-side context: one CUDA device, one stream, the operator cache and the
// engines built on it.
#pragma once

#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "dev.h"
#include "fc_tables.h"
#include "fcsg_common.h"

namespace fcsg {

// FcOperator on the device: host tables + device copies (OperatorCache entry).
struct DevOp {
    FcTables t;
    FcPlanDev plan{};
    double2* d_tw = nullptr;
    double* d_blend = nullptr;
    double2* d_mult = nullptr;
    double2* d_mult_pfa = nullptr;
    double2* d_prime_frag = nullptr;
    ~DevOp() {
        dev::free(d_prime_frag);
        dev::free(d_mult_pfa);
        dev::free(d_tw);
        dev::free(d_blend);
        dev::free(d_mult);
    }
};

class Engine;

struct Ctx {
    int device = 0;
    void* stream = nullptr;
    std::map<std::tuple<int, int, int, double, int, int>, int> op_index;
    std::vector<std::unique_ptr<DevOp>> ops;

    std::string err;
    int err_kind = 0, err_patch = -1, err_sub = -1, err_i = -1, err_j = -1;
    double err_t = 0.0;

    // OperatorCache::get semantics: one operator per key
    int get_op(int n, int n_cont, int degree, FilterSpec f);
    const DevOp& op(int id) const;
};

}  // namespace fcsg
