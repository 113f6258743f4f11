// kr_common.cuh — shared internals of libkrcuda.so (engine + solver).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
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

#ifdef KR_CHECKED
#include <cstdio>
__device__ __forceinline__ uint32_t kr_dyn_smem() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
#define KR_DCHECK(c)                                                                                       \
    do {                                                                                                   \
        if (!(c)) {                                                                                        \
            printf("KR_CHECKED %s:%d: %s (block %d,%d thread %d)\n", __FILE__, __LINE__, #c, int(blockIdx.x), \
                   int(blockIdx.y), int(threadIdx.x));                                                     \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
// [off, off + bytes) inside the launch's dynamic shared memory
#define KR_SMEM_CHECK(off, bytes) KR_DCHECK(uint64_t(off) + uint64_t(bytes) <= uint64_t(kr_dyn_smem()))
#else
#define KR_DCHECK(c) ((void)0)
#define KR_SMEM_CHECK(off, bytes) ((void)0)
#endif

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

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

// SELL-32-sigma matrix in HBM (sliced ELLPACK, Kreutzer et al.): output rows
// are taken in windows of kSigma, sorted by length inside the window, and cut
// into slices of 32 rows.  Entry j of the row held by lane l of slice s lives
// at slice_ptr[s] + 32*j + l, so a warp streams 32 rows with coalesced loads
// while every row is still folded by ONE lane in its storage order — the
// reference's accumulation order (engine.hpp:67-70, 82-88, 104-108, 118-129).
// Rows longer than kLongRow entries are kept out of the slices and handled
// by one thread block each (cooperative loads, ordered one-thread sum), so a
// few very long rows cannot serialise a warp on memory latency.
constexpr int kSigma = 1024;
constexpr int kLongRow = 256;
constexpr int64_t kLongRowBudget = 4096;  // long rows per matrix the adaptive threshold allows (kr_engine.cu)
struct DevSell {
    int64_t nrows = 0, nslices = 0, nnz = 0, padded = 0;
    int32_t maxLen = 0;            // longest row kept in the slices
    int64_t* slice_ptr = nullptr;  // nslices + 1
    int32_t* lane_row = nullptr;   // nslices * 32; -1 = unused lane
    int32_t* lane_len = nullptr;   // nslices * 32
    int32_t* col = nullptr;        // padded entries
    double* val = nullptr;
    // long rows, plain CSR
    int64_t nlong = 0, nnzLong = 0;
    int64_t* long_ptr = nullptr;   // nlong + 1
    int32_t* long_row = nullptr;   // output row of each long row
    int32_t* long_col = nullptr;
    double* long_val = nullptr;
    // dispatch order (widest slices first): over all slices, and within each
    // board group (entries relative to the group's first slice)
    int32_t* order_all = nullptr;
    int32_t* order_grp = nullptr;
    // Compressed slots (SELL-C), same slot layout as col /
    // val: each row is [segment 0 | segment 1] (the two merged factors, in
    // storage order); 16-bit columns relative to a per-slice base of each
    // segment; the coded segment's values as 16-bit codes into its board's
    // table (exact doubles), the other segment's values in val.
    bool comp = false;
    int codedSeg = 0;                // segment whose values are coded (0 or 1)
    uint16_t* col16 = nullptr;       // padded
    uint16_t* code16 = nullptr;      // padded
    int32_t* lane_len0 = nullptr;    // 32 * nslices: entries of segment 0
    int32_t* base0 = nullptr;        // nslices
    int32_t* base1 = nullptr;        // nslices
    int32_t* tbase = nullptr;        // nslices: table offset (board * kCodeSlab)
    double* table = nullptr;         // nboards * kCodeSlab
};

constexpr int64_t kCodeSlab = 65536;  // table entries per board (16-bit codes)

// Programmatic dependent launch (PDL).  Every engine / solver kernel starts
// with pdl_entry(): it waits until the grid it depends on has completed (its
// memory visible) and then lets its own dependents start launching, so a
// dependent kernel's launch and CTA rasterisation overlap this one instead of
// following it.  Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// KR_PDL=0: plain stream-ordered launches.  KR_PDL_MAXGRID: only grids of at
// most this many CTAs are launched early (multi-wave grids launched early
// measured slower: their waiting CTAs hold SM slots the kernel before them
// still needs).
// afterSmall: launches whose early start only pays after a small kernel
// (the team player step: launched early behind a ~400-CTA SpMV it measured
// 14% slower for the config-2 factored solver, behind a 43-CTA K7 launch 4%
// faster): those also need the previous kernel on the stream to have at most
// KR_PDL_MAXPREV (128) CTAs.
inline bool pdl_enabled(unsigned gridCtas, unsigned prevCtas, bool afterSmall) {
    // read per launch (tens of ns against a launch), so a process can switch
    const char* off = std::getenv("KR_PDL");
    if (off && std::atoi(off) == 0) return false;
    const char* mg = std::getenv("KR_PDL_MAXGRID");
    if (gridCtas > (mg ? unsigned(std::atol(mg)) : 2000u)) return false;
    if (!afterSmall) return true;
    const char* mp = std::getenv("KR_PDL_MAXPREV");
    return prevCtas <= (mp ? unsigned(std::atol(mp)) : 128u);
}

// Grid size of the last kernel this thread launched on each stream (the
// early launch pays after small, latency-bound kernels).
inline unsigned& last_grid(cudaStream_t s) {
    thread_local std::vector<std::pair<cudaStream_t, unsigned>> last;
    for (auto& e : last)
        if (e.first == s) return e.second;
    if (last.size() > 64) last.clear();
    last.emplace_back(s, 0xffffffffu);
    return last.back().second;
}

// KR_CHECKED: the bounds-checked build (build.build_cuda_variant("checked",
// ["KR_CHECKED"]), loaded with KR_CUDA_LIB_VARIANT=checked; the pool's GPUs
// take no compute-sanitizer runs).  Every device allocation gets 4 KB guard
// zones on both sides and its whole extent filled with a poison byte (reads
// of uninitialised or out-of-range data turn into huge / negative values that
// break the bitwise tests or trip an index check); the guards are verified
// when the allocation is freed and by kr_checked_verify().  KR_DCHECK traps
// on a failed device-side index check, printing where.
#ifdef KR_CHECKED
void* checked_alloc(size_t bytes);
void checked_free(void* p);
#endif

template <class T>
T* dev_alloc(int64_t n) {
    T* p = nullptr;
#ifdef KR_CHECKED
    if (n > 0) p = static_cast<T*>(checked_alloc(sizeof(T) * size_t(n)));
#else
    if (n > 0) KR_CK(cudaMalloc(&p, sizeof(T) * size_t(n)));
#endif
    return p;
}

inline void dev_free(void* p) {
#ifdef KR_CHECKED
    checked_free(p);
#else
    cudaFree(p);
#endif
}

// kernel<<<grid, block, smem, stream>>>(args...) with the PDL attribute
// (arguments coerced to the kernel's parameter types, as <<<>>> does).
template <typename... KArgs, typename... Args>
void launch_pdl(bool afterSmall, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    const unsigned ctas = grid.x * grid.y * grid.z;
    unsigned& prev = last_grid(stream);
    cfg.numAttrs = pdl_enabled(ctas, prev, afterSmall) ? 1 : 0;
    prev = ctas;
    KR_CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <typename... KArgs, typename... Args>
void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
    launch_pdl(false, kernel, grid, block, smem, stream, std::forward<Args>(args)...);
}

// Raise (never lower) a kernel's dynamic shared-memory limit: the attribute
// belongs to the kernel, not to the engine or solver that launches it, so a
// smaller later object must not shrink what an earlier one needs.
template <class K>
void raise_smem_limit(K kernel, size_t bytes) {
    cudaFuncAttributes fa;
    KR_CK(cudaFuncGetAttributes(&fa, kernel));
    if (size_t(fa.maxDynamicSharedSizeBytes) < bytes)
        KR_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

struct KronState;  // implicit Kronecker engine (kr_kron.cu)
// Boards [b0, b1) of direction dir (0: A x, 1: Aᵀ y); b1 < 0 = all boards.
void kron_product(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0 = 0, int b1 = -1);
int64_t kron_flops(const kr_engine* e, int dir);
// Sequence-major (per board [seq][hand]) product and layout conversions of
// the implicit engine (kr_kron.cu).
void kron_product_seq(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s);
void kron_transpose(kr_engine* e, int dir, int side, const double* src, double* dst, bool toSeq, cudaStream_t s);
bool kron_seq_major();
int kron_boards(const kr_engine* e);
void kron_destroy(KronState* k);

// NCCL transport (kr_comm.cu)
void comm_allgather(kr_comm* c, const double* send, double* recv, size_t count, cudaStream_t s);
int comm_rank(const kr_comm* c);
int comm_size(const kr_comm* c);
int comm_device(const kr_comm* c);

struct KfState;  // Kronecker-factored engine (kr_kfengine.cu)
void kf_product(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0 = 0, int b1 = -1);
void kf_destroy(KfState* k);
// The Kronecker-factored products on an input already in the engine's
// staging layout (sequence-major over all of the direction's hands), and the
// conversion into that layout.
void kf_product_staged(kr_engine* e, int dir, const double* inT, double* out, cudaStream_t s);
void kf_stage_all(kr_engine* e, int dir, const double* in, double* inT, cudaStream_t s);

}  // namespace krb

namespace krb {
// Resources of one pipelined host-buffer product (kr_engine_ax / _atx, and
// each direction of kr_engine_pair): the stream it is forked from and joined
// into, copy and stage streams, per-group events, device staging buffers.
struct HostPipe {
    cudaStream_t main = nullptr, copyIn = nullptr, copyOut = nullptr, stage2 = nullptr, stage3 = nullptr;
    std::vector<cudaEvent_t> evIn, evOut, evMid, evSolve;
    cudaEvent_t evStart = nullptr, evEnd = nullptr;
    double* d_in = nullptr;   // owned by the pipe only for pipe[1]
    double* d_out = nullptr;
    bool made = false;
};

// kr_engine_pair_queue: a queue of independent pairs.  Each direction has two
// device slots (input, output); pair i uses slot i % 2, so the input copy of
// pair i + 1 and the output copy of pair i - 1 run while pair i computes.
// One H2D stream and one D2H stream carry both directions (one whole-vector
// copy each: the bus runs at its duplex rate, profiles/r02/zc_probe_r02z.log),
// one compute stream per direction.
struct QueuePipe {
    cudaStream_t cin = nullptr, cout = nullptr, comp[2] = {nullptr, nullptr};
    cudaEvent_t evIn[2][2] = {}, evDone[2][2] = {}, evOut[2][2] = {};  // [dir][slot]
    cudaEvent_t evStart = nullptr, evEnd[4] = {};
    double* in[2][2] = {};
    double* out[2][2] = {};
    bool made = false;
};
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
    // Internal layouts: the k coordinates are relabelled chain-major (mkind
    // 1) so every chain is a contiguous range, and V^T x gathers from a
    // sequence-major copy of x (x'[s*M2 + J] = x[J*n2 + s]) when n2 is known.
    bool xseq = false;
    int64_t M2 = 0;  // hands of the column player over all boards
    krb::DevSell VT;  // t = V^T x'                     engine.hpp:65-72
    krb::DevSell UA;  // y = [U | Ahat] [z ; x]         engine.hpp:81-89
    krb::DevSell UT;  // s = U^T y                      engine.hpp:103-110
    krb::DevSell AV;  // x = [Ahat^T | V] [y ; z]       engine.hpp:117-130
    // chains (mkind 1), chain-sliced: slice s holds 32 chains, element j of
    // lane l's chain at position chain_ptr[s] + 32 j + l (j < chain_len);
    // chain_mul[p] = M(t, previous t of the chain); chain_neg1 = all -1.
    int64_t kpad = 0;       // internal k positions (>= k; padding never touched)
    int64_t nchains = 0;    // number of chain slices
    bool chain_tma = true;  // TMA bulk-copy pipeline (else register pipeline)
    bool lean = true;       // lean SELL variant for one-entry-row matrices (KR_NO_LEAN=1: off)
    int chain_withmul = 0;  // some chain has a multiplier other than -1
    int64_t* chain_ptr = nullptr;
    std::vector<int64_t> bCh;  // host: first chain slice of each board (+ total)
    int32_t* chain_len = nullptr;
    double* chain_mul = nullptr;
    uint8_t* chain_neg1 = nullptr;
    // levels (mkind 2): forward uses strict-lower CSR(M), backward CSC(M)
    std::vector<int64_t> lvl_fwd_ptr, lvl_bwd_ptr;  // host: level boundaries
    int32_t* lvl_fwd_rows = nullptr;
    int32_t* lvl_bwd_cols = nullptr;
    int64_t* mr_ptr = nullptr;
    int32_t* mr_col = nullptr;
    double* mr_val = nullptr;
    int64_t* mc_ptr = nullptr;
    int32_t* mc_row = nullptr;
    double* mc_val = nullptr;
    // scratch
    double* d_tz = nullptr;   // k: t, then z in place (GradientWorkspace::y/z), A x
    double* d_tz2 = nullptr;  // the same for A^T y, so the two may run concurrently
    double* d_xp = nullptr;  // cols: sequence-major copy of x
    double* d_in = nullptr;  // staging for host-buffer calls
    double* d_out = nullptr;
    int64_t flops_total = 0, flops_last = 0, launches = 0;
    int64_t flops_per_product = 0;
    // optional per-kernel event timing (kr_engine_set_timing)
    bool timing = false;
    int timingMask = 0xF;  // matrices bracketed when timing (bit w: VT, UA, UT, AV)
    struct Pending {
        int which;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> eventPool;
    int64_t tLaunches[4] = {0, 0, 0, 0};
    double tMs[4] = {0, 0, 0, 0};
    // implicit Kronecker mode (kr_engine_create_kron): no factors at all
    krb::KronState* kron = nullptr;
    // Kronecker-factored mode (kr_engine_create_kfactored): Technique B post
    // from its hand-space factors, products bitwise the factored engine's
    krb::KfState* kf = nullptr;
    int pf = 0;  // SELL slice L2 prefetch distance in batches (KR_PF)
    // Board groups.  Host-buffer calls pipeline over them: input copies,
    // per-group kernels and output copies run concurrently (copyIn / stream /
    // copyOut).  grpBoard: board ranges; grpRow / grpCol: row / column
    // offsets; bSl / bNl: first slice / long row of each board per matrix.
    std::vector<int64_t> grpRow{0}, grpCol{0};
    std::vector<int64_t> bSl[4], bNl[4];
    std::vector<int32_t> grpBoard{0};
    // pipe[0]: the host-buffer products (main = `stream`); pipe[1]: the
    // second direction of kr_engine_pair (its own streams and staging
    // buffers, created on first use)
    krb::HostPipe pipe[2];
    krb::QueuePipe queue;
    // captured host-buffer pipelines, keyed by (direction, host input,
    // host output[, second input, second output]); pinned buffers only
    // (kr_engine_ax / kr_engine_atx: dir 0 / 1; kr_engine_pair: dir 2)
    struct PipeGraph {
        int dir;
        const double* in;
        double* out;
        cudaGraphExec_t exec;
        int64_t launches;
        const double* in2 = nullptr;
        double* out2 = nullptr;
    };
    std::vector<PipeGraph> pipeGraphs;
    std::vector<PipeGraph> pipeSeen;  // first calls (exec unused): captured on the second
    // SelfCheck mode (kr_engine_set_selfcheck, SelfCheckEngine solver.hpp:67-99):
    // every scEvery-th product is replayed through scRef (the block formula
    // restated: the implicit engine) and compared normwise on the device;
    // a violation is sticky (scStat[4] = 1) and surfaces as KR_CONTRACT.
    kr_engine* scRef = nullptr;
    int scEvery = 0;
    double scTol = 0;
    int64_t scCalls = 0, scChecks = 0;
    double* scBuf[2] = {nullptr, nullptr};  // expected outputs per direction
    double* scStat = nullptr;               // [2 dirs][2] (max |got-exp|, max |exp|) bits, [4] flag, [5] worst ratio
    // kr_engine_pair_device: A^T y forks onto `side` (created on first use)
    cudaStream_t side = nullptr;
    cudaEvent_t evFork = nullptr, evJoin = nullptr;
    int ngroups() const { return int(grpRow.size()) - 1; }
};

namespace krb {
// Enqueue the products on `s` (device pointers).
void engine_ax(kr_engine* e, const double* x, double* y, cudaStream_t s);
// Boards [b0, b1) of one product (direction dir), for the board-block
// engines (implicit, Kronecker-factored); no flop accounting (the caller
// accounts the whole product once with engine_account).  False for engines
// whose products do not split by board range (the factored engine).
bool engine_product_boards(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0, int b1);
void engine_account(kr_engine* e, int dir);
int engine_boards(const kr_engine* e);
// SelfCheck: compare out with the reference engine's product of in (every
// scEvery-th call; no-op when off or while s is being captured); and raise
// KR_CONTRACT if a check has failed (synchronises the engine's stream).
void engine_selfcheck(kr_engine* e, int dir, const double* in, const double* out, cudaStream_t s);
void engine_selfcheck_raise(kr_engine* e);
void engine_atx(kr_engine* e, const double* y, double* x, cudaStream_t s);
// Copy streams and events for the pipelined host-buffer calls (>= 2 groups).
void engine_make_pipeline(kr_engine* e);
std::vector<int> group_ends(int nb, uint32_t flags);
// Shared-memory limits of the chain-solve kernels (engines built elsewhere).
void engine_chain_setup(kr_engine* e);
}  // namespace krb
