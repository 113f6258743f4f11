// kr_jit.cuh — the DCFR player step compiled for a treeplex (kr_jit.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "kr_engine.h"

namespace krb {

constexpr int kJitHands = 32;    // granule of the hands per CTA (one warp)
constexpr int kJitMaxSeq = 96;   // regrets live in registers: larger trees keep the generic kernels

struct JitStep {
    cudaKernel_t kern = nullptr;
    int n = 0;
    int hands = 128;   // hands per CTA
    int threads = 128; // threads per CTA (two per hand in the two-group kernels)
    int layout = 0;    // 0 hand-major, 1 per-board sequence-major, 2 global sequence-major x
    size_t smem = 0;   // one hands x n tile (+ the two-group exchange slots)
    std::string log;   // NVRTC / ptxas log (registers, spills)
};

// Compile (or fetch from the process cache) the step kernel for tree t and
// update rule (KR_RULE_*).  False, with the reason in `why`, when NVRTC is
// absent, the tree is not level-ordered or too large, or KR_STEP names
// another kernel.
// layout 1: gradients read and strategies written sequence-major per board
// (the implicit engine's kron_product_seq layout; bstart / nb at launch);
// layout 2: strategies written sequence-major over all hands (the
// Kronecker-factored engine's staging layout), gradients hand-major.
// groups > 1: the tree split over that many warp groups per 32-hand set (for
// grids too small to fill the GPU with one thread per hand).
bool jit_step_compile(const kr_treeplex& t, int rule, JitStep& out, std::string& why, int layout = 0,
                      int groups = 1);

// k_player_team's mode-1 arguments (the sweep, sequence form, discount and
// average of one player over H hands).
void jit_step_launch(const JitStep& j, int device, int64_t H, const double* g, int negate, double* regret,
                     double* xout, double* avg, double pos, double neg, double shrink, const double* fac,
                     const int* dt, int noAvg, double* rootOut, const double* extra, cudaStream_t st,
                     const int64_t* bstart = nullptr, int nb = 0, int stagger = 0);

// Start stagger (ns) of the DCFR solver's full-GPU step grids (KR_JIT_STAGGER).
int jit_stagger_ns();

// The generated source (for inspection and tests).
std::string jit_step_source(const kr_treeplex& t, int rule, int layout = 0, int groups = 1);

}  // namespace krb
