// kr_common.cuh — shared internals of libkrcuda.so (engine + solver).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "kr_engine.h"

namespace krb {

// Error carried to the C ABI boundary (mirrors errors.hpp codes).
struct Fail {
    int code;
    std::string msg;
};

void set_error(int code, const std::string& msg);

#define KR_CK(call)                                                                        \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::krb::Fail{KR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

#define KR_CK_LAUNCH() KR_CK(cudaGetLastError())

template <class F>
int guarded(F&& f) {
    try {
        f();
        return KR_OK;
    } catch (const Fail& e) {
        set_error(e.code, e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(KR_CUDA, e.what());
        return KR_CUDA;
    }
}

// One row-ordered compressed matrix in HBM.  Row r's entries are summed in
// storage order by exactly one thread (the reference's accumulation order),
// and `blk` partitions rows into thread blocks of <= kRowsPerBlock rows and
// roughly kNnzPerBlock entries.
struct DevRows {
    int64_t nrows = 0, nnz = 0;
    int64_t* rowptr = nullptr;
    int32_t* col = nullptr;
    double* val = nullptr;
    int32_t* blk = nullptr;
    int32_t nblk = 0;
};

template <class T>
T* dev_alloc(int64_t n) {
    T* p = nullptr;
    if (n > 0) KR_CK(cudaMalloc(&p, sizeof(T) * size_t(n)));
    return p;
}

}  // namespace krb

// Engine state (opaque to C callers).
struct kr_engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t rows = 0, cols = 0, k = 0;
    int64_t nnzA = 0, nnzU = 0, nnzM = 0, nnzV = 0;
    int32_t n1 = 0, n2 = 0;
    // M classification: 0 identity (solve skipped, engine.hpp:74), 1 chains
    // (<=1 off-diagonal per row and per column: Technique B), 2 general
    // level-scheduled, 3 not unit lower triangular (products fail CONTRACT).
    int mkind = 0;
    std::string mfail;
    krb::DevRows VT;  // rows of V^T (= V's CSC columns): t = V^T x            engine.hpp:65-72
    krb::DevRows UA;  // row i = [U row i | Ahat row i] over [z | x]            engine.hpp:81-89
    krb::DevRows UT;  // rows of U^T: s = U^T y                                 engine.hpp:103-110
    krb::DevRows AV;  // row c = [Ahat^T row c | V row c] over [y | z]          engine.hpp:117-130
    // chains (mkind 1): elements in solve order; mul = M(row, previous row)
    int64_t nchains = 0;
    int64_t* chain_ptr = nullptr;
    int32_t* chain_idx = nullptr;
    double* chain_mul = nullptr;
    // levels (mkind 2): forward uses strict-lower CSR(M), backward CSC(M)
    std::vector<int64_t> lvl_fwd_ptr, lvl_bwd_ptr;  // host: level boundaries
    int32_t* lvl_fwd_rows = nullptr;
    int32_t* lvl_bwd_cols = nullptr;
    int64_t* mr_ptr = nullptr;  // CSR strictly lower
    int32_t* mr_col = nullptr;
    double* mr_val = nullptr;
    int64_t* mc_ptr = nullptr;  // CSC strictly lower
    int32_t* mc_row = nullptr;
    double* mc_val = nullptr;
    // scratch
    double* d_tz = nullptr;  // k: t, then z in place (GradientWorkspace::y/z)
    double* d_in = nullptr;  // staging for host-buffer calls
    double* d_out = nullptr;
    int64_t flops_total = 0, flops_last = 0, launches = 0;
    int64_t flops_per_product = 0;
};

namespace krb {
// Enqueue the products on `s` (device pointers); return KR status.
void engine_ax(kr_engine* e, const double* x, double* y, cudaStream_t s);
void engine_atx(kr_engine* e, const double* y, double* x, cudaStream_t s);
}  // namespace krb
