// kr_engine.cu — B200 factored gradient oracle: y = A x and x = A^T y with
// A = Ahat + U M^-1 V^T (arXiv 2112.03804; reference engine.hpp:58-133).
//
// Design:
//  * Every product is "ordered": each output row is accumulated by ONE lane
//    in the reference's storage order (engine.hpp:67-70, 82-88, 104-108,
//    118-129), so results are bitwise equal to the reference (compiled with
//    -fmad=false: no contraction, as in the reference's x86-64 build).
//  * matvecTranspose's scatters become gathers over transposed layouts built
//    once at create time (no atomics, deterministic).
//  * Ax  = [V^T x'] -> [M solve] -> [[U|Ahat] over [z|x]]   (3 launches + x')
//    ATx = [U^T y]  -> [M^T solve] -> [[Ahat^T|V] over [y|z]]  (3 launches)
//    U and Ahat rows are merged so one pass reproduces the single accumulator
//    of engine.hpp:83-89 (and likewise engine.hpp:117-130).
//  * Matrices are stored SELL-32-sigma (kr_common.cuh): one warp streams 32
//    rows with coalesced 128/256-byte loads, no shared memory, no barriers.
//  * Technique B's M is a set of chains over strength-sorted hands; k is
//    relabelled chain-major so each chain is contiguous, and one warp walks
//    a chain with a shuffle-fed serial recurrence (the exact reference
//    recurrence z_r = t_r - M(r,p) z_p, engine.hpp:38-39).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <thread>
#include <unordered_map>

#include <cooperative_groups.h>

#include "kr_common.cuh"

namespace cg = cooperative_groups;

#ifdef KR_CHECKED
namespace krb {
namespace {
constexpr size_t kGuard = 4096;
constexpr unsigned char kPoison = 0xF7;  // double -1.4e270-ish, int32 < 0, uint16 0xF7F7
struct CheckedAlloc {
    char* base;
    size_t bytes, total;
};
std::mutex g_checked_mu;
std::unordered_map<void*, CheckedAlloc>& checked_allocs() {
    static std::unordered_map<void*, CheckedAlloc> m;
    return m;
}
int64_t g_checked_bad = 0;

// the two guard zones and the rounding tail after the caller's bytes
bool guards_intact(void* p, const CheckedAlloc& a) {
    const size_t lo = kGuard, tail = a.total - kGuard - a.bytes;
    std::vector<unsigned char> h(std::max(lo, tail));
    auto all_poison = [&](const char* d, size_t n) {
        if (cudaMemcpy(h.data(), d, n, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
        for (size_t i = 0; i < n; ++i)
            if (h[i] != kPoison) return false;
        return true;
    };
    const bool ok = all_poison(a.base, lo) && all_poison(static_cast<char*>(p) + a.bytes, tail);
    if (!ok)
        std::fprintf(stderr, "KR_CHECKED: guard zone of a %zu-byte device allocation was overwritten\n", a.bytes);
    return ok;
}
}  // namespace

void* checked_alloc(size_t bytes) {
    const size_t total = ((bytes + 255) & ~size_t(255)) + 2 * kGuard;
    char* base = nullptr;
    KR_CK(cudaMalloc(&base, total));
    KR_CK(cudaMemset(base, kPoison, total));
    KR_CK(cudaDeviceSynchronize());
    void* p = base + kGuard;
    std::lock_guard<std::mutex> g(g_checked_mu);
    checked_allocs()[p] = {base, bytes, total};
    return p;
}

void checked_free(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_checked_mu);
    auto it = checked_allocs().find(p);
    if (it == checked_allocs().end()) {
        std::fprintf(stderr, "KR_CHECKED: free of a pointer the library did not allocate\n");
        ++g_checked_bad;
        return;
    }
    cudaDeviceSynchronize();
    if (!guards_intact(p, it->second)) ++g_checked_bad;
    cudaFree(it->second.base);
    checked_allocs().erase(it);
}
}  // namespace krb
#endif

namespace krb {

namespace {
thread_local int g_code = 0;
thread_local std::string g_msg;
}  // namespace

void set_error(int code, const std::string& msg) {
    g_code = code;
    g_msg = msg;
}

namespace {

#ifndef KR_WARPS_PER_BLOCK
#define KR_WARPS_PER_BLOCK 4
#endif
constexpr int kWarpsPerBlock = KR_WARPS_PER_BLOCK;  // SELL slices (warps) per block

// ------------------------------------------------------------- kernels ----

struct SellView {
    const int64_t* slice_ptr;
    const int32_t* lane_row;
    const int32_t* lane_len;
    const int32_t* col;
    const double* val;
    int64_t nslices;
    const int64_t* long_ptr;
    const int32_t* long_row;
    const int32_t* long_col;
    const double* long_val;
    int64_t nlong;
    const int32_t* order;  // slice dispatch order (nullptr: storage order)
    int32_t pf;            // L2 prefetch distance of the slice rows, in batches of KU (0: none)
    int64_t nsrc, ndst;    // gather-index and output-row bounds (checked build)
};

// One bulk prefetch of [p, p + bytes) into L2 (bytes a multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

constexpr int kChunk = 256;  // long-row entries staged per warp
#ifndef KR_KU
#define KR_KU 8
#endif
constexpr int kU = KR_KU;  // entries per lane per pipeline stage

// COH bit 0 / bit 1: xa / xb was written earlier in the same kernel (the
// fused small-engine product, behind a cluster barrier's acquire): plain
// coherent loads (ld.global.ca) instead of the read-only path.
template <int COH>
__device__ __forceinline__ double src_load(const double* p) {
    return COH ? __ldca(p) : __ldg(p);
}
template <bool TWO, int COH = 0>
__device__ __forceinline__ double gather(const double* __restrict__ xa, const double* __restrict__ xb, int32_t split,
                                         int32_t c) {
    KR_DCHECK(c >= 0);
    if (TWO) return c < split ? src_load<COH & 1>(xa + c) : src_load<COH & 2>(xb + (c - split));
    return src_load<COH & 1>(xa + c);
}

// One long row per warp (the 32 lanes load and multiply a chunk of kChunk
// entries, lane 0 adds the chunk's products in storage order while the next
// chunk's loads are in flight).  Shared by the plain and compressed kernels.
template <bool TWO, int COH = 0>
__device__ __forceinline__ void spmv_long_row_at(const SellView& A, const double* __restrict__ xa,
                                                 const double* __restrict__ xb, int32_t split, double* __restrict__ y,
                                                 double* P, int lane, int64_t r);
template <bool TWO>
__device__ __forceinline__ void spmv_long_row(const SellView& A, const double* __restrict__ xa,
                                              const double* __restrict__ xb, int32_t split, double* __restrict__ y,
                                              double* P, int lane, int w) {
    const int64_t r = int64_t(blockIdx.x) * kWarpsPerBlock + w;
    if (r >= A.nlong) return;
    spmv_long_row_at<TWO>(A, xa, xb, split, y, P, lane, r);
}
template <bool TWO, int COH>
__device__ __forceinline__ void spmv_long_row_at(const SellView& A, const double* __restrict__ xa,
                                                 const double* __restrict__ xb, int32_t split, double* __restrict__ y,
                                                 double* P, int lane, int64_t r) {
    const int64_t e0 = A.long_ptr[r], e1 = A.long_ptr[r + 1];
    double acc = 0.0;
    constexpr int per = kChunk / 32;
    double p[per];
    // chunk 0 products
    int n = int(lmin(kChunk, e1 - e0));
    {
        int32_t c[per];
        double v[per];
#pragma unroll
        for (int u = 0; u < per; ++u)
            if (u * 32 + lane < n) {
                c[u] = __ldcs(A.long_col + e0 + u * 32 + lane);
                v[u] = __ldcs(A.long_val + e0 + u * 32 + lane);
            }
#pragma unroll
        for (int u = 0; u < per; ++u)
            if (u * 32 + lane < n) {
                KR_DCHECK(c[u] < A.nsrc);
                p[u] = v[u] * gather<TWO, COH>(xa, xb, split, c[u]);
            }
    }
    for (int64_t t0 = e0; t0 < e1; t0 += kChunk) {
#pragma unroll
        for (int u = 0; u < per; ++u)
            if (u * 32 + lane < n) P[u * 32 + lane] = p[u];
        __syncwarp();
        // issue the next chunk's loads before lane 0 folds this one
        const int64_t t1 = t0 + kChunk;
        const int nn = int(lmin(kChunk, e1 - t1));
        int32_t c[per];
        double v[per];
#pragma unroll
        for (int u = 0; u < per; ++u)
            if (u * 32 + lane < nn) {
                c[u] = __ldcs(A.long_col + t1 + u * 32 + lane);
                v[u] = __ldcs(A.long_val + t1 + u * 32 + lane);
            }
        if (lane == 0) {
            int q = 0;
            for (; q + 8 <= n; q += 8) {
                double t[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) t[u] = P[q + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += t[u];
            }
            for (; q < n; ++q) acc += P[q];
        }
#pragma unroll
        for (int u = 0; u < per; ++u)
            if (u * 32 + lane < nn) {
                KR_DCHECK(c[u] < A.nsrc);
                p[u] = v[u] * gather<TWO, COH>(xa, xb, split, c[u]);
            }
        __syncwarp();
        n = nn;
    }
    KR_DCHECK(A.long_row[r] >= 0 && A.long_row[r] < A.ndst);
    if (lane == 0) y[A.long_row[r]] = acc;
}

// y[row] = sum_j val * src[col] over the row's entries in storage order;
// src = [xa (split entries) | xb] when TWO.  The first blocks fold one long
// row per warp (the 32 lanes load and multiply a chunk, lane 0 adds the
// chunk's products in order while the next chunk's loads are in flight); the
// remaining blocks run four SELL slices each, one per warp, with a two-stage
// register pipeline (loads of stage g+1 in flight while stage g gathers and
// accumulates).
// KU / MINB: entries per lane per pipeline stage and minimum resident
// blocks.  Matrices whose SELL rows hold at most one entry (U^T of Technique
// B: one entry per k position) take k_spmv_lean instead: their cost is the
// per-row load latency.
template <bool TWO, int KU, int COH = 0>
__device__ __forceinline__ void spmv_slice(const SellView& A, const double* __restrict__ xa,
                                           const double* __restrict__ xb, int32_t split, double* __restrict__ y,
                                           int64_t si, int lane);

template <bool TWO, int KU = kU, int MINB = 1>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, MINB)
    k_spmv(SellView A, const double* __restrict__ xa, const double* __restrict__ xb, int32_t split,
           double* __restrict__ y) {
    krb::pdl_entry();
    __shared__ double P[kWarpsPerBlock][kChunk];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t longBlocks = (A.nlong + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blockIdx.x < longBlocks) {
        spmv_long_row<TWO>(A, xa, xb, split, y, P[w], lane, w);
        return;
    }
    const int64_t si = (int64_t(blockIdx.x) - longBlocks) * kWarpsPerBlock + w;
    if (si >= A.nslices) return;
    spmv_slice<TWO, KU>(A, xa, xb, split, y, si, lane);
}

// Matrices whose SELL rows hold at most one entry (U^T of Technique B): no
// pipeline, one load round per lane (row metadata, the entry, the gather),
// y[row] = 0.0 + val * x[col] (0.0 for an empty row): k_spmv's sum for one
// entry, bit for bit.  Long rows as in k_spmv.  KR_LEAN_SLICES: slices per
// warp, all in flight together (config 3 U^T: 37.8 us at 1, 43.5 at 4,
// 43.9 at 8; the <1, 8> k_spmv instance it replaces: 41-43, k_spmv<false>:
// 49; profiles/r02/lean_ut_r02z.log).
#ifndef KR_LEAN_SLICES
#define KR_LEAN_SLICES 1
#endif
constexpr int kLeanSlices = KR_LEAN_SLICES;
__global__ void __launch_bounds__(32 * kWarpsPerBlock, 8)
    k_spmv_lean(SellView A, const double* __restrict__ xa, double* __restrict__ y) {
    krb::pdl_entry();
    __shared__ double P[kWarpsPerBlock][kChunk];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t longBlocks = (A.nlong + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blockIdx.x < longBlocks) {
        spmv_long_row<false>(A, xa, nullptr, 0, y, P[w], lane, w);
        return;
    }
    const int64_t si0 = ((int64_t(blockIdx.x) - longBlocks) * kWarpsPerBlock + w) * kLeanSlices;
    int32_t row[kLeanSlices], len[kLeanSlices], c[kLeanSlices];
    int64_t base[kLeanSlices];
    double v[kLeanSlices], x[kLeanSlices];
#pragma unroll
    for (int u = 0; u < kLeanSlices; ++u) {
        row[u] = -1;
        len[u] = 0;
        const int64_t si = si0 + u;
        if (si < A.nslices) {
            const int64_t sl = A.order ? int64_t(A.order[si]) : si;
            base[u] = A.slice_ptr[sl] + lane;
            len[u] = A.lane_len[sl * 32 + lane];
            row[u] = A.lane_row[sl * 32 + lane];
        }
    }
#pragma unroll
    for (int u = 0; u < kLeanSlices; ++u)
        if (len[u] > 0) {
            c[u] = __ldcs(A.col + base[u]);
            v[u] = __ldcs(A.val + base[u]);
        }
#pragma unroll
    for (int u = 0; u < kLeanSlices; ++u)
        if (len[u] > 0) {
            KR_DCHECK(len[u] == 1 && c[u] < A.nsrc);
            x[u] = gather<false>(xa, nullptr, 0, c[u]);
        }
#pragma unroll
    for (int u = 0; u < kLeanSlices; ++u) {
        KR_DCHECK(row[u] < A.ndst);
        if (row[u] >= 0) y[row[u]] = len[u] > 0 ? 0.0 + v[u] * x[u] : 0.0;
    }
}

// One SELL slice (32 rows) by one warp: each lane's row summed in storage
// order, KU entries per pipeline stage.
template <bool TWO, int KU, int COH>
__device__ __forceinline__ void spmv_slice(const SellView& A, const double* __restrict__ xa,
                                           const double* __restrict__ xb, int32_t split, double* __restrict__ y,
                                           int64_t si, int lane) {
    // widest slices first: a slice's latency grows with its width, so the
    // widest ones must not be the last dispatched (they would set the tail)
    const int64_t s = A.order ? int64_t(A.order[si]) : si;
    const int64_t sb = A.slice_ptr[s];
    const int64_t base = sb + lane;
    const int32_t len = A.lane_len[s * 32 + lane];
    const int32_t row = A.lane_row[s * 32 + lane];
    // Slice rows are contiguous (row r: 32 entries at sb + 32 r), so lane 0
    // (the slice's longest row: rows are sorted by length) keeps the next
    // pf batches of col / val streaming into L2 with one bulk prefetch per
    // array; each batch's loads then wait on L2, not on HBM.
    const int32_t pfRows = A.pf * KU;
    auto prefetch = [&](int32_t r0, int32_t n) {
        n = min(n, len - r0);
        if (n > 0) {
            prefetch_l2(A.col + sb + int64_t(r0) * 32, uint32_t(n) * 32u * 4u);
            prefetch_l2(A.val + sb + int64_t(r0) * 32, uint32_t(n) * 32u * 8u);
        }
    };
    if (lane == 0 && pfRows > 0) prefetch(KU, pfRows);
    double acc = 0.0;
    int32_t c[KU];
    double v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u)
        if (u < len) {
            c[u] = __ldcs(A.col + base + int64_t(u) * 32);
            v[u] = __ldcs(A.val + base + int64_t(u) * 32);
        }
    for (int32_t j = 0; j < len; j += KU) {
        if (lane == 0 && pfRows > 0) prefetch(j + KU + pfRows, KU);
        int32_t cn[KU];
        double vn[KU], x[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const int32_t jj = j + KU + u;
            if (jj < len) {
                cn[u] = __ldcs(A.col + base + int64_t(jj) * 32);
                vn[u] = __ldcs(A.val + base + int64_t(jj) * 32);
            }
        }
#pragma unroll
        for (int u = 0; u < KU; ++u)
            if (j + u < len) {
                KR_DCHECK(c[u] < A.nsrc);
                x[u] = gather<TWO, COH>(xa, xb, split, c[u]);
            }
#pragma unroll
        for (int u = 0; u < KU; ++u)
            if (j + u < len) acc += v[u] * x[u];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            c[u] = cn[u];
            v[u] = vn[u];
        }
    }
    KR_DCHECK(row < A.ndst);
    if (row >= 0) y[row] = acc;
}

struct SellCView {
    const uint16_t* col16;
    const uint16_t* code16;
    const int32_t* len0;
    const int32_t* base0;
    const int32_t* base1;
    const int32_t* tbase;
    const double* table;
};

// Entries [j0, j1) of one lane's row, one segment: x = src[cbase + col16],
// value = the coded table entry or val, accumulated in storage order.  KU
// entries per stage, the next stage's loads in flight during this one's
// gathers (as k_spmv).
template <int KU, bool CODED>
__device__ __forceinline__ double seg_sum(double acc, const SellView& A, const SellCView& C, int64_t base, int32_t j0,
                                          int32_t j1, const double* __restrict__ src, int32_t cbase, int32_t tb) {
    if (j0 >= j1) return acc;
    uint32_t c[KU], k[KU];
    double v[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u)
        if (j0 + u < j1) {
            const int64_t q = base + int64_t(j0 + u) * 32;
            c[u] = __ldcs(C.col16 + q);
            if (CODED) k[u] = __ldcs(C.code16 + q);
            else v[u] = __ldcs(A.val + q);
        }
    for (int32_t j = j0; j < j1; j += KU) {
        uint32_t cn[KU], kn[KU];
        double vn[KU], x[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            const int32_t jj = j + KU + u;
            if (jj < j1) {
                const int64_t q = base + int64_t(jj) * 32;
                cn[u] = __ldcs(C.col16 + q);
                if (CODED) kn[u] = __ldcs(C.code16 + q);
                else vn[u] = __ldcs(A.val + q);
            }
        }
#pragma unroll
        for (int u = 0; u < KU; ++u)
            if (j + u < j1) {
                KR_DCHECK(int64_t(cbase) + int64_t(c[u]) < A.nsrc && cbase >= 0);
                x[u] = __ldg(src + cbase + int32_t(c[u]));
                if (CODED) v[u] = __ldg(C.table + tb + int32_t(k[u]));
            }
#pragma unroll
        for (int u = 0; u < KU; ++u)
            if (j + u < j1) acc += v[u] * x[u];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
            c[u] = cn[u];
            if (CODED) k[u] = kn[u];
            else v[u] = vn[u];
        }
    }
    return acc;
}

// k_spmv over compressed slots: segment 0 (entries [0, len0), source xa)
// then segment 1 (entries [len0, len), source xb), one accumulator, so each
// row's sum is the storage-order sum of k_spmv bit for bit.  CSEG: the coded
// segment.  Long rows keep the plain CSR path.
template <bool TWO, int CSEG>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    k_spmvc(SellView A, SellCView C, const double* __restrict__ xa, const double* __restrict__ xb, int32_t split,
            double* __restrict__ y) {
    krb::pdl_entry();
    __shared__ double P[kWarpsPerBlock][kChunk];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t longBlocks = (A.nlong + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blockIdx.x < longBlocks) {
        spmv_long_row<TWO>(A, xa, xb, split, y, P[w], lane, w);
        return;
    }
    const int64_t si = (int64_t(blockIdx.x) - longBlocks) * kWarpsPerBlock + w;
    if (si >= A.nslices) return;
    const int64_t s = A.order ? int64_t(A.order[si]) : si;
    const int64_t base = A.slice_ptr[s] + lane;
    const int32_t len = A.lane_len[s * 32 + lane];
    const int32_t row = A.lane_row[s * 32 + lane];
    const int32_t len0 = TWO ? C.len0[s * 32 + lane] : len;
    const int32_t tb = C.tbase[s];
    double acc = 0.0;
    acc = seg_sum<kU, CSEG == 0>(acc, A, C, base, 0, len0, xa, C.base0[s], tb);
    if (TWO) acc = seg_sum<kU, CSEG == 1>(acc, A, C, base, len0, len, xb, C.base1[s], tb);
    KR_DCHECK(row < A.ndst && len0 <= len);
    if (row >= 0) y[row] = acc;
}

// x'[s*M2 + J] = x[J*n2 + s], tiled: a block stages the rows of 32 hands
// (32 * n2 contiguous doubles) in shared memory and writes each sequence's 32
// consecutive hands as one 256-byte segment.
__global__ void __launch_bounds__(256) k_seq_major_tile(const double* __restrict__ x, int64_t M2, int32_t n2,
                                                        double* __restrict__ xp, int64_t J0, int64_t J1) {
    krb::pdl_entry();
    extern __shared__ double tile[];
    const int64_t j0 = J0 + int64_t(blockIdx.x) * 32;
    const int cnt = int(lmin(32, J1 - j0));
    const double* src = x + j0 * n2;
    for (int q = threadIdx.x; q < cnt * n2; q += blockDim.x) tile[q] = __ldcs(src + q);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (lane >= cnt) return;
    for (int s = threadIdx.x >> 5; s < n2; s += blockDim.x >> 5) xp[int64_t(s) * M2 + j0 + lane] = tile[lane * n2 + s];
}

// x'[s*M2 + J] = x[J*n2 + s]: the sequence-major copy V^T x gathers from.
__global__ void k_seq_major(const double* __restrict__ x, int64_t M2, int32_t n2, double* __restrict__ xp,
                            int64_t q0, int64_t q1) {
    krb::pdl_entry();
    const int64_t q = q0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= q1) return;
    const int64_t J = q / n2;
    const int32_t s = int32_t(q - J * n2);
    xp[int64_t(s) * M2 + J] = x[q];
}

constexpr int kChainU = 8;  // chain elements per lane per pipeline stage

// ---- TMA bulk-copy pipeline for the chain solves -------------------------
// A chain slice is contiguous: row j (element j of its 32 chains) is 256
// bytes.  One warp per slice streams chunks of kChunkRows rows into a
// kStages-deep shared-memory ring with cp.async.bulk (TMA, completion on an
// mbarrier), so ~kStages*kChunkRows rows are in flight while each lane runs
// its chain's serial recurrence out of shared memory.
constexpr int kChunkRows = 32;  // rows per stage (8 KB)
constexpr int kStages = 8;      // 256 rows (64 KB) in flight per slice

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Chain solve over one slice per block (32 threads).  dir = +1 forward
// (engine.hpp:31-41), -1 backward (engine.hpp:44-54); same recurrences as
// the register kernels above.
// Dynamic shared memory: kStages chunks of t (and of the multipliers when
// the engine has any chain whose multipliers are not all -1: withMul).
// One chain slice by one warp: ROWS rows per chunk, a STAGES-deep ring
// (Tb / Mb: STAGES chunks each, bar: STAGES mbarriers initialised with count
// 1).  ring: the warp's running chunk count, so a warp can run several slices
// through one ring without re-initialising its barriers.
template <int DIR, int ROWS, int STAGES>
__device__ __forceinline__ void chain_tma_slice(const int64_t* __restrict__ sbase, const int32_t* __restrict__ slen,
                                                const double* __restrict__ cmul, const uint8_t* __restrict__ neg1,
                                                int withMul, double* __restrict__ z, int64_t s, int lane,
                                                double (*Tb)[ROWS * 32], double (*Mb)[ROWS * 32], uint64_t* bar,
                                                uint32_t& ring) {
    constexpr int kChunkRows = ROWS, kStages = STAGES;
    const int64_t b0 = sbase[s];
    const int32_t width = int32_t((sbase[s + 1] - b0) / 32);
    const int32_t len = slen[s * 32 + lane];
    const bool allneg = neg1[s * 32 + lane] != 0;
    const bool needMul = withMul && __any_sync(0xffffffffu, !allneg);
    const int nChunks = (width + kChunkRows - 1) / kChunkRows;
    KR_DCHECK(len >= 0 && len <= width && (sbase[s + 1] - b0) % 32 == 0);
    // chunk c covers rows [r0, r0 + n); forward chunks ascend, backward descend
    auto chunk_rows = [&](int c, int32_t& r0, int32_t& n) {
        if (DIR > 0) {
            r0 = c * kChunkRows;
            n = min(kChunkRows, width - r0);
        } else {
            const int32_t r1 = width - c * kChunkRows;
            r0 = max(0, r1 - kChunkRows);
            n = r1 - r0;
        }
    };
    auto issue = [&](int c) {
        if (lane == 0 && c < nChunks) {
            int32_t r0, n;
            chunk_rows(c, r0, n);
            const int st = (ring + uint32_t(c)) % kStages;
            const uint32_t bytes = uint32_t(n) * 32 * 8;
            KR_DCHECK(n > 0 && n <= kChunkRows && r0 >= 0 && r0 + n <= width);
            mbar_expect_tx(&bar[st], needMul ? 2 * bytes : bytes);
            bulk_g2s(Tb[st], z + b0 + int64_t(r0) * 32, bytes, &bar[st]);
            if (needMul) bulk_g2s(Mb[st], cmul + b0 + int64_t(r0) * 32, bytes, &bar[st]);
        }
    };
    for (int c = 0; c < kStages - 1; ++c) issue(c);
    double carry = needMul ? 0.0 : -0.0, mulNext = 0.0;
    for (int c = 0; c < nChunks; ++c) {
        issue(c + kStages - 1);
        const uint32_t gc = ring + uint32_t(c);
        const int st = gc % kStages;
        mbar_wait(&bar[st], (gc / kStages) & 1);
        int32_t r0, n;
        chunk_rows(c, r0, n);
        const double* T = Tb[st];
        const double* Mu = Mb[st];
        double* zc = z + b0 + lane;
        // Branch-free batches of 8: the shared-memory loads of a batch are
        // issued together; each element costs one dependent DADD (+ select).
        // Rows past n or past the lane's chain length are computed and
        // discarded (predicated store, carry kept).
        if (!needMul) {  // every multiplier is -1: z_p = t_p + z_{p-1}
            // One dependent DADD per element and nothing else on the chain:
            // the carry starts at -0.0, and t + (-0.0) == t for every t
            // (including -0.0), so a chain's first element needs no special
            // case; backward rows past the lane's chain end feed -0.0 instead
            // of t, which keeps the carry at -0.0 until the chain starts.
            // Forward rows past the chain end (and rows past the chunk, only
            // in the last chunk) compute unused values.  The next batch's
            // shared-memory loads are issued before this batch's adds.
            const int nbat = (n + 7) / 8;
            auto load = [&](int qb, double* dst) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int q = DIR > 0 ? qb * 8 + u : n - 1 - (qb * 8 + u);
                    dst[u] = T[(q >= 0 && q < n ? q : 0) * 32 + lane];
                }
            };
            double t[8], tn[8];
            load(0, t);
            if (n == kChunkRows) {
                // Full chunk: every row is inside the slice, so stores need no
                // predicate -- rows past a lane's chain end are that lane's
                // padding positions, which nothing reads (kpad >= k).
                double* zr = zc + int64_t(r0) * 32;
#pragma unroll
                for (int qb = 0; qb < kChunkRows / 8; ++qb) {
                    if (qb + 1 < kChunkRows / 8) load(qb + 1, tn);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int q = DIR > 0 ? qb * 8 + u : kChunkRows - 1 - (qb * 8 + u);
                        const double tv = (DIR > 0 || r0 + q < len) ? t[u] : -0.0;
                        const double zq = tv + carry;
                        zr[q * 32] = zq;
                        carry = zq;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) t[u] = tn[u];
                }
            } else {
                for (int qb = 0; qb < nbat; ++qb) {
                    if (qb + 1 < nbat) load(qb + 1, tn);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int q = DIR > 0 ? qb * 8 + u : n - 1 - (qb * 8 + u);
                        const int32_t j = r0 + q;
                        const bool live = j < len;
                        const double tv = (DIR > 0 || live) ? t[u] : -0.0;
                        const double zq = tv + carry;
                        if (q >= 0 && q < n && live) zc[int64_t(j) * 32] = zq;
                        carry = zq;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) t[u] = tn[u];
                }
            }
        } else if (DIR > 0) {
            for (int q = 0; q < n; ++q) {
                const int32_t j = r0 + q;
                if (j < len) {
                    const double tq = T[q * 32 + lane];
                    double zq = tq;
                    if (j != 0) {
                        if (allneg) zq = tq + carry;
                        else if (carry != 0.0) zq = tq - Mu[q * 32 + lane] * carry;
                    }
                    zc[int64_t(j) * 32] = zq;
                    carry = zq;
                }
            }
        } else {
            for (int q = n - 1; q >= 0; --q) {
                const int32_t j = r0 + q;
                if (j < len) {
                    const double tq = T[q * 32 + lane];
                    double zq;
                    if (allneg) {
                        zq = j != len - 1 ? tq + carry : tq;
                    } else {
                        double acc = 0.0;
                        if (j != len - 1) acc += mulNext * carry;
                        zq = tq - acc;
                        mulNext = Mu[q * 32 + lane];
                    }
                    zc[int64_t(j) * 32] = zq;
                    carry = zq;
                }
            }
        }
        // all lanes are done reading this stage before TMA refills it
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    ring += uint32_t(nChunks);
}

template <int DIR>
__global__ void __launch_bounds__(32)
    k_chain_tma(const int64_t* __restrict__ sbase, const int32_t* __restrict__ slen,
                const double* __restrict__ cmul, const uint8_t* __restrict__ neg1, int withMul,
                double* __restrict__ z, int64_t s0) {
    krb::pdl_entry();
    extern __shared__ __align__(128) double dsm[];
    __shared__ __align__(8) uint64_t bar[kStages];
    KR_SMEM_CHECK(0, size_t(kStages) * kChunkRows * 32 * 8 * (withMul ? 2 : 1));
    const int lane = threadIdx.x;
    if (lane == 0)
        for (int q = 0; q < kStages; ++q) mbar_init(&bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t ring = 0;
    chain_tma_slice<DIR, kChunkRows, kStages>(
        sbase, slen, cmul, neg1, withMul, z, s0 + blockIdx.x, lane,
        reinterpret_cast<double(*)[kChunkRows * 32]>(dsm),
        reinterpret_cast<double(*)[kChunkRows * 32]>(dsm + kStages * kChunkRows * 32), bar, ring);
}

// Forward solve M z = t along chains (engine.hpp:31-41 restricted to <=1
// off-diagonal per row/column).  Chain-sliced layout: a warp owns 32 chains,
// lane l walks chain l whose element j sits at base + 32 j + l, so every
// load and store is coalesced across the warp and each lane runs the exact
// serial recurrence of its chain from registers:
//   z_p = (z_{p-1} != 0) ? t_p - M(p,p-1) z_{p-1} : t_p
// (for M(p,p-1) == -1 this is bitwise t_p + z_{p-1}: one dependent add).
// The next stage's loads are issued before the current stage's adds.
__device__ __forceinline__ void chain_forward_slice(const int64_t* __restrict__ sbase, const int32_t* __restrict__ slen,
                                                    const double* __restrict__ cmul, const uint8_t* __restrict__ neg1,
                                                    int64_t s, double* __restrict__ z, int lane) {
    const int32_t len = slen[s * 32 + lane];
    const bool allneg = neg1[s * 32 + lane] != 0;
    double* zc = z + sbase[s] + lane;
    const double* mc = cmul + sbase[s] + lane;
    double prev = 0.0;
    double t[kChainU], m[kChainU];
#pragma unroll
    for (int u = 0; u < kChainU; ++u) {
        t[u] = u < len ? zc[int64_t(u) * 32] : 0.0;
        m[u] = (!allneg && u < len) ? mc[int64_t(u) * 32] : -1.0;
    }
    for (int32_t j0 = 0; j0 < len; j0 += kChainU) {
        double tn[kChainU], mn[kChainU];
#pragma unroll
        for (int u = 0; u < kChainU; ++u) {
            const int32_t j = j0 + kChainU + u;
            tn[u] = j < len ? zc[int64_t(j) * 32] : 0.0;
            mn[u] = (!allneg && j < len) ? mc[int64_t(j) * 32] : -1.0;
        }
#pragma unroll
        for (int u = 0; u < kChainU; ++u) {
            const int32_t j = j0 + u;
            if (j < len) {
                double zq = t[u];
                if (j != 0) {
                    if (allneg) zq = t[u] + prev;
                    else if (prev != 0.0) zq = t[u] - m[u] * prev;
                }
                zc[int64_t(j) * 32] = zq;
                prev = zq;
            }
        }
#pragma unroll
        for (int u = 0; u < kChainU; ++u) {
            t[u] = tn[u];
            m[u] = mn[u];
        }
    }
}

// Backward solve M^T z = s along chains (engine.hpp:44-54), same layout,
// each lane walking its chain in reverse: z_p = s_p - (0 + M(p+1,p) z_{p+1}).
__device__ __forceinline__ void chain_backward_slice(const int64_t* __restrict__ sbase, const int32_t* __restrict__ slen,
                                                     const double* __restrict__ cmul, const uint8_t* __restrict__ neg1,
                                                     int64_t s, double* __restrict__ z, int lane) {
    const int32_t len = slen[s * 32 + lane];
    const bool allneg = neg1[s * 32 + lane] != 0;
    double* zc = z + sbase[s] + lane;
    const double* mc = cmul + sbase[s] + lane;
    double next = 0.0, mulNext = 0.0;
    double t[kChainU], m[kChainU];
#pragma unroll
    for (int u = 0; u < kChainU; ++u) {
        const int32_t j = len - 1 - u;
        t[u] = j >= 0 ? zc[int64_t(j) * 32] : 0.0;
        m[u] = (!allneg && j >= 0) ? mc[int64_t(j) * 32] : -1.0;
    }
    for (int32_t j1 = len - 1; j1 >= 0; j1 -= kChainU) {
        double tn[kChainU], mn[kChainU];
#pragma unroll
        for (int u = 0; u < kChainU; ++u) {
            const int32_t j = j1 - kChainU - u;
            tn[u] = j >= 0 ? zc[int64_t(j) * 32] : 0.0;
            mn[u] = (!allneg && j >= 0) ? mc[int64_t(j) * 32] : -1.0;
        }
#pragma unroll
        for (int u = 0; u < kChainU; ++u) {
            const int32_t j = j1 - u;
            if (j >= 0) {
                double zq;
                if (allneg) {
                    zq = j != len - 1 ? t[u] + next : t[u];
                } else {
                    double acc = 0.0;
                    if (j != len - 1) acc += mulNext * next;
                    zq = t[u] - acc;
                    mulNext = m[u];
                }
                zc[int64_t(j) * 32] = zq;
                next = zq;
            }
        }
#pragma unroll
        for (int u = 0; u < kChainU; ++u) {
            t[u] = tn[u];
            m[u] = mn[u];
        }
    }
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    k_chain_forward(const int64_t* __restrict__ sbase, const int32_t* __restrict__ slen,
                    const double* __restrict__ cmul, const uint8_t* __restrict__ neg1, int64_t s0, int64_t s1,
                    double* __restrict__ z) {
    krb::pdl_entry();
    const int64_t s = s0 + int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    if (s < s1) chain_forward_slice(sbase, slen, cmul, neg1, s, z, threadIdx.x & 31);
}

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    k_chain_backward(const int64_t* __restrict__ sbase, const int32_t* __restrict__ slen,
                     const double* __restrict__ cmul, const uint8_t* __restrict__ neg1, int64_t s0, int64_t s1,
                     double* __restrict__ z) {
    krb::pdl_entry();
    const int64_t s = s0 + int64_t(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
    if (s < s1) chain_backward_slice(sbase, slen, cmul, neg1, s, z, threadIdx.x & 31);
}

// The whole product of a small engine in one launch: a
// cluster of CTAs runs the three stages the separate launches run -- the
// input-side SpMV (V^T x or U^T y) into tz, the M solve along the chains in
// place, the output-side SpMV ([U | Ahat] or [Ahat^T | V]) -- with a cluster
// barrier (release / acquire) between stages, each warp taking rows, slices
// and chain slices strided over the cluster's warps.  Every row, slice and
// chain runs the same device code as the separate kernels, so the result is
// bitwise theirs; the last stage reads tz through coherent loads (it was
// written inside this launch).  For engines whose three launches are
// latency-bound (a few us of work each), this takes two launch gaps and two
// grid drains off every product.
constexpr int kTinyWarps = 8;
struct TinyChains {
    const int64_t* sbase;
    const int32_t* slen;
    const double* cmul;
    const uint8_t* neg1;
    int64_t n;    // chain slices (0: M = I)
    int withMul;  // some chain has a multiplier other than -1
};
// chain stage: each warp streams its slices through a TMA ring of
// kTinyStages chunks of kTinyRows rows (t, and the multipliers withMul)
constexpr int kTinyRows = 16, kTinyStages = 3;
constexpr size_t kTinyRing = size_t(kTinyStages) * kTinyRows * 32;  // doubles per array per warp
template <int DIR>
__global__ void __launch_bounds__(32 * kTinyWarps, 1)
    k_tiny_product(SellView A1, SellView A2, TinyChains C, const double* __restrict__ in, double* __restrict__ tz,
                   int32_t split, double* __restrict__ out) {
    krb::pdl_entry();
    __shared__ double P[kTinyWarps][kChunk];
    __shared__ __align__(8) uint64_t bar[kTinyWarps][kTinyStages];
    extern __shared__ __align__(128) double ring[];
    cg::cluster_group cl = cg::this_cluster();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
        for (int q = 0; q < kTinyStages; ++q) mbar_init(&bar[w][q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t nw = int64_t(cl.num_blocks()) * kTinyWarps;
    const int64_t gw = int64_t(cl.block_rank()) * kTinyWarps + w;
    for (int64_t i = gw; i < A1.nlong + A1.nslices; i += nw) {
        if (i < A1.nlong) spmv_long_row_at<false>(A1, in, nullptr, 0, tz, P[w], lane, i);
        else spmv_slice<false, kU>(A1, in, nullptr, 0, tz, i - A1.nlong, lane);
    }
    cl.sync();
    if (C.n) {
        // stage 1's stores (ordered before this point by the cluster
        // barrier) before the bulk copies read them through the async proxy
        asm volatile("fence.proxy.async.global;" ::: "memory");
        KR_SMEM_CHECK(0, kTinyWarps * kTinyRing * 8 * (C.withMul ? 2 : 1));
        double* Tb = ring + size_t(w) * kTinyRing * (C.withMul ? 2 : 1);
        uint32_t used = 0;
        for (int64_t i = gw; i < C.n; i += nw)
            chain_tma_slice<DIR == 0 ? 1 : -1, kTinyRows, kTinyStages>(
                C.sbase, C.slen, C.cmul, C.neg1, C.withMul, tz, i, lane,
                reinterpret_cast<double(*)[kTinyRows * 32]>(Tb),
                reinterpret_cast<double(*)[kTinyRows * 32]>(Tb + kTinyRing), bar[w], used);
        cl.sync();
    }
    // [U | Ahat] over [tz | x]; [Ahat^T | V] over [y | tz]: tz (written
    // above) through coherent loads, the input through the read-only path
    const double* xa = DIR == 0 ? tz : in;
    const double* xb = DIR == 0 ? in : tz;
    constexpr int coh = DIR == 0 ? 1 : 2;
    for (int64_t i = gw; i < A2.nlong + A2.nslices; i += nw) {
        if (i < A2.nlong) spmv_long_row_at<true, coh>(A2, xa, xb, split, out, P[w], lane, i);
        else spmv_slice<true, kU, coh>(A2, xa, xb, split, out, i - A2.nlong, lane);
    }
}

// General unit-lower forward solve, one level: row-oriented gathers in
// ascending column order == the column-oriented order of engine.hpp:33-40.
__global__ void k_level_forward(const int32_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ ptr,
                                const int32_t* __restrict__ col, const double* __restrict__ val,
                                double* __restrict__ z) {
    krb::pdl_entry();
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t r = rows[q];
    double zr = z[r];
    for (int64_t e = ptr[r]; e < ptr[r + 1]; ++e) {
        const double zj = z[col[e]];
        if (zj != 0.0) zr -= val[e] * zj;
    }
    z[r] = zr;
}

// General backward solve, one level (engine.hpp:46-53).
__global__ void k_level_backward(const int32_t* __restrict__ cols, int64_t n, const int64_t* __restrict__ ptr,
                                 const int32_t* __restrict__ row, const double* __restrict__ val,
                                 double* __restrict__ z) {
    krb::pdl_entry();
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t j = cols[q];
    double acc = 0.0;
    for (int64_t e = ptr[j]; e < ptr[j + 1]; ++e) acc += val[e] * z[row[e]];
    z[j] -= acc;
}

// ------------------------------------------------------- host building ----

struct HostRows {  // one board's matrix in processing order, final indices
    std::vector<int64_t> ptr{0};
    std::vector<int32_t> col;
    std::vector<double> val;
    std::vector<int32_t> outRow;  // output row of each row (empty: rowBase + r)
    void push(int32_t c, double v) {
        col.push_back(c);
        val.push_back(v);
    }
    void endRow() { ptr.push_back(int64_t(col.size())); }
    int64_t rows() const { return int64_t(ptr.size()) - 1; }
};

struct HostSell {
    std::vector<int64_t> sptr;  // relative slice starts (no terminal entry)
    std::vector<int32_t> lrow, llen;
    std::vector<int32_t> col;
    std::vector<double> val;
    std::vector<int64_t> lptr{0};  // long rows (relative CSR)
    std::vector<int32_t> lgrow, lcol;
    std::vector<double> lval;
};

// Sizes of the SELL layout (short rows) and of the long-row CSR.
void sell_sizes(const std::vector<int64_t>& len, int64_t longRow, int64_t& slices, int64_t& padded, int64_t& nlong,
                int64_t& nnzLong) {
    const int64_t n = int64_t(len.size());
    slices = padded = nlong = nnzLong = 0;
    std::vector<int64_t> w;
    for (int64_t w0 = 0; w0 < n; w0 += kSigma) {
        const int64_t w1 = std::min<int64_t>(n, w0 + kSigma);
        w.clear();
        for (int64_t r = w0; r < w1; ++r) {
            if (len[size_t(r)] > longRow) {
                ++nlong;
                nnzLong += len[size_t(r)];
            } else {
                w.push_back(len[size_t(r)]);
            }
        }
        std::sort(w.begin(), w.end(), std::greater<int64_t>());
        for (size_t s0 = 0; s0 < w.size(); s0 += 32) {
            padded += 32 * w[s0];
            ++slices;
        }
    }
}

void to_sell(const HostRows& h, int64_t rowBase, int64_t longRow, HostSell& out) {
    const int64_t n = h.rows();
    out = HostSell{};
    std::vector<int64_t> idx;
    int64_t cur = 0;
    for (int64_t w0 = 0; w0 < n; w0 += kSigma) {
        const int64_t w1 = std::min<int64_t>(n, w0 + kSigma);
        idx.clear();
        for (int64_t r = w0; r < w1; ++r) {
            const int64_t len = h.ptr[r + 1] - h.ptr[r];
            if (len > longRow) {
                out.lgrow.push_back(h.outRow.empty() ? int32_t(rowBase + r) : h.outRow[size_t(r)]);
                out.lcol.insert(out.lcol.end(), h.col.begin() + h.ptr[r], h.col.begin() + h.ptr[r + 1]);
                out.lval.insert(out.lval.end(), h.val.begin() + h.ptr[r], h.val.begin() + h.ptr[r + 1]);
                out.lptr.push_back(int64_t(out.lcol.size()));
            } else {
                idx.push_back(r);
            }
        }
        std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
            return h.ptr[a + 1] - h.ptr[a] > h.ptr[b + 1] - h.ptr[b];
        });
        for (size_t s0 = 0; s0 < idx.size(); s0 += 32) {
            const int64_t width = h.ptr[idx[s0] + 1] - h.ptr[idx[s0]];
            out.sptr.push_back(cur);
            const size_t at = out.col.size();
            out.col.resize(at + size_t(32 * width), 0);
            out.val.resize(at + size_t(32 * width), 0.0);
            for (int l = 0; l < 32; ++l) {
                const size_t q = s0 + size_t(l);
                if (q < idx.size()) {
                    const int64_t r = idx[q];
                    const int64_t len = h.ptr[r + 1] - h.ptr[r];
                    out.lrow.push_back(h.outRow.empty() ? int32_t(rowBase + r) : h.outRow[size_t(r)]);
                    out.llen.push_back(int32_t(len));
                    for (int64_t j = 0; j < len; ++j) {
                        out.col[at + size_t(32 * j + l)] = h.col[size_t(h.ptr[r] + j)];
                        out.val[at + size_t(32 * j + l)] = h.val[size_t(h.ptr[r] + j)];
                    }
                } else {
                    out.lrow.push_back(-1);
                    out.llen.push_back(0);
                }
            }
            cur += 32 * width;
        }
    }
}

void alloc_sell(krb::DevSell& d, int64_t nrows, int64_t nslices, int64_t nnz, int64_t padded, int64_t nlong,
                int64_t nnzLong) {
    d.nlong = nlong;
    d.nnzLong = nnzLong;
    d.long_ptr = dev_alloc<int64_t>(nlong + 1);
    d.long_row = dev_alloc<int32_t>(std::max<int64_t>(nlong, 1));
    d.long_col = dev_alloc<int32_t>(std::max<int64_t>(nnzLong, 1));
    d.long_val = dev_alloc<double>(std::max<int64_t>(nnzLong, 1));
    KR_CK(cudaMemcpy(d.long_ptr + nlong, &nnzLong, 8, cudaMemcpyHostToDevice));
    d.nrows = nrows;
    d.nslices = nslices;
    d.nnz = nnz;
    d.padded = padded;
    d.slice_ptr = dev_alloc<int64_t>(nslices + 1);
    d.lane_row = dev_alloc<int32_t>(std::max<int64_t>(32 * nslices, 1));
    d.lane_len = dev_alloc<int32_t>(std::max<int64_t>(32 * nslices, 1));
    d.col = dev_alloc<int32_t>(std::max<int64_t>(padded, 1));
    d.val = dev_alloc<double>(std::max<int64_t>(padded, 1));
    KR_CK(cudaMemcpy(d.slice_ptr + nslices, &padded, 8, cudaMemcpyHostToDevice));
}

void upload_sell(const HostSell& h, int64_t sliceBase, int64_t entryBase, int64_t longBase, int64_t longEntryBase,
                 krb::DevSell& d, cudaStream_t s) {
    const int64_t nl = int64_t(h.lgrow.size());
    if (nl) {
        std::vector<int64_t> lp(h.lptr.begin(), h.lptr.end() - 1);
        for (auto& x : lp) x += longEntryBase;
        KR_CK(cudaMemcpyAsync(d.long_ptr + longBase, lp.data(), 8 * size_t(nl), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.long_row + longBase, h.lgrow.data(), 4 * size_t(nl), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.long_col + longEntryBase, h.lcol.data(), 4 * h.lcol.size(), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.long_val + longEntryBase, h.lval.data(), 8 * h.lval.size(), cudaMemcpyHostToDevice, s));
        KR_CK(cudaStreamSynchronize(s));
    }
    const int64_t ns = int64_t(h.sptr.size());
    if (ns == 0) return;
    std::vector<int64_t> p(h.sptr);
    for (auto& x : p) x += entryBase;
    KR_CK(cudaMemcpyAsync(d.slice_ptr + sliceBase, p.data(), 8 * size_t(ns), cudaMemcpyHostToDevice, s));
    KR_CK(cudaMemcpyAsync(d.lane_row + 32 * sliceBase, h.lrow.data(), 4 * h.lrow.size(), cudaMemcpyHostToDevice, s));
    KR_CK(cudaMemcpyAsync(d.lane_len + 32 * sliceBase, h.llen.data(), 4 * h.llen.size(), cudaMemcpyHostToDevice, s));
    if (!h.col.empty()) {
        KR_CK(cudaMemcpyAsync(d.col + entryBase, h.col.data(), 4 * h.col.size(), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.val + entryBase, h.val.data(), 8 * h.val.size(), cudaMemcpyHostToDevice, s));
    }
    KR_CK(cudaStreamSynchronize(s));
}

// SELL-C of one board's slices (DevSell::comp): per lane the number of
// segment-0 entries (two segments: columns below `split` come first in every
// merged row), per slice the lowest column of each segment, 16-bit column
// offsets, and 16-bit codes (first-seen order) for the values of segment
// `codedSeg`.  ok = false when a slice's segment spans more than 65,536
// columns or the board has more than 65,536 distinct coded values.
struct HostComp {
    std::vector<uint16_t> col16, code16;
    std::vector<int32_t> len0, base0, base1;
    std::vector<double> table;
    bool ok = true;
};

void compress_sell(const HostSell& h, bool two, int64_t split, int codedSeg, HostComp& c) {
    const size_t ns = h.sptr.size(), padded = h.col.size();
    c = HostComp{};
    c.col16.assign(padded, 0);
    c.code16.assign(padded, 0);
    c.len0.assign(32 * ns, 0);
    c.base0.assign(ns, 0);
    c.base1.assign(ns, 0);
    std::unordered_map<uint64_t, uint16_t> codes;
    for (size_t sl = 0; sl < ns && c.ok; ++sl) {
        const int64_t at = h.sptr[sl];
        int64_t lo[2] = {INT64_MAX, INT64_MAX}, hi[2] = {-1, -1};
        for (int l = 0; l < 32; ++l) {
            const int32_t len = h.llen[sl * 32 + size_t(l)];
            int32_t n0 = 0;
            for (int32_t j = 0; j < len; ++j) {
                const int64_t col = h.col[size_t(at + 32 * int64_t(j) + l)];
                const int sg = (two && col >= split) ? 1 : 0;
                if (sg == 0 && n0 != j) c.ok = false;  // segment 0 must come first
                if (sg == 0) ++n0;
                const int64_t cc = sg ? col - split : col;
                lo[sg] = std::min(lo[sg], cc);
                hi[sg] = std::max(hi[sg], cc);
            }
            c.len0[sl * 32 + size_t(l)] = n0;
        }
        for (int sg = 0; sg < 2; ++sg) {
            if (hi[sg] < 0) lo[sg] = 0;
            else if (hi[sg] - lo[sg] > 65535) c.ok = false;
        }
        c.base0[sl] = int32_t(lo[0]);
        c.base1[sl] = int32_t(lo[1]);
        for (int l = 0; l < 32 && c.ok; ++l) {
            const int32_t len = h.llen[sl * 32 + size_t(l)], n0 = c.len0[sl * 32 + size_t(l)];
            for (int32_t j = 0; j < len; ++j) {
                const size_t q = size_t(at + 32 * int64_t(j) + l);
                const int sg = j < n0 ? 0 : 1;
                const int64_t col = h.col[q];
                c.col16[q] = uint16_t(sg ? col - split - lo[1] : col - lo[0]);
                if (sg == codedSeg) {
                    uint64_t bits;
                    std::memcpy(&bits, &h.val[q], 8);
                    auto it = codes.find(bits);
                    if (it == codes.end()) {
                        if (c.table.size() >= size_t(kCodeSlab)) {
                            c.ok = false;
                            break;
                        }
                        it = codes.emplace(bits, uint16_t(c.table.size())).first;
                        c.table.push_back(h.val[q]);
                    }
                    c.code16[q] = it->second;
                }
            }
        }
    }
}

void alloc_comp(krb::DevSell& d, int nb) {
    d.col16 = dev_alloc<uint16_t>(std::max<int64_t>(d.padded, 1));
    d.code16 = dev_alloc<uint16_t>(std::max<int64_t>(d.padded, 1));
    d.lane_len0 = dev_alloc<int32_t>(std::max<int64_t>(32 * d.nslices, 1));
    d.base0 = dev_alloc<int32_t>(std::max<int64_t>(d.nslices, 1));
    d.base1 = dev_alloc<int32_t>(std::max<int64_t>(d.nslices, 1));
    d.tbase = dev_alloc<int32_t>(std::max<int64_t>(d.nslices, 1));
    d.table = dev_alloc<double>(int64_t(nb) * kCodeSlab);
}

void upload_comp(const HostComp& c, int b, int64_t sliceBase, int64_t entryBase, krb::DevSell& d, cudaStream_t s) {
    const size_t ns = c.base0.size();
    if (ns) {
        std::vector<int32_t> tb(ns, int32_t(int64_t(b) * kCodeSlab));
        KR_CK(cudaMemcpyAsync(d.col16 + entryBase, c.col16.data(), 2 * c.col16.size(), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.code16 + entryBase, c.code16.data(), 2 * c.code16.size(), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.lane_len0 + 32 * sliceBase, c.len0.data(), 4 * c.len0.size(), cudaMemcpyHostToDevice,
                              s));
        KR_CK(cudaMemcpyAsync(d.base0 + sliceBase, c.base0.data(), 4 * ns, cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.base1 + sliceBase, c.base1.data(), 4 * ns, cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.tbase + sliceBase, tb.data(), 4 * ns, cudaMemcpyHostToDevice, s));
    }
    if (!c.table.empty())
        KR_CK(cudaMemcpyAsync(d.table + int64_t(b) * kCodeSlab, c.table.data(), 8 * c.table.size(),
                              cudaMemcpyHostToDevice, s));
    KR_CK(cudaStreamSynchronize(s));
}

void free_comp(krb::DevSell& d) {
    krb::dev_free(d.col16);
    krb::dev_free(d.code16);
    krb::dev_free(d.lane_len0);
    krb::dev_free(d.base0);
    krb::dev_free(d.base1);
    krb::dev_free(d.tbase);
    krb::dev_free(d.table);
    d.col16 = d.code16 = nullptr;
    d.lane_len0 = d.base0 = d.base1 = d.tbase = nullptr;
    d.table = nullptr;
    d.comp = false;
}

void free_sell(krb::DevSell& d) {
    krb::dev_free(d.slice_ptr);
    krb::dev_free(d.lane_row);
    krb::dev_free(d.lane_len);
    krb::dev_free(d.col);
    krb::dev_free(d.val);
    krb::dev_free(d.long_ptr);
    krb::dev_free(d.long_row);
    krb::dev_free(d.long_col);
    krb::dev_free(d.long_val);
    krb::dev_free(d.order_all);
    krb::dev_free(d.order_grp);
    free_comp(d);
    d = krb::DevSell{};
}

// Stable counting-sort transpose of a compressed matrix: rows of the result
// list the original outer index in ascending order (== the reference's
// scatter order in matvecTranspose).
void transpose_into(int64_t outerN, int64_t innerN, const int64_t* outer, const int32_t* inner, const double* v,
                    std::vector<int64_t>& tptr, std::vector<int32_t>& tidx, std::vector<double>& tval) {
    const int64_t nnz = outer[outerN];
    tptr.assign(size_t(innerN) + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) tptr[size_t(inner[e]) + 1]++;
    for (int64_t i = 0; i < innerN; ++i) tptr[i + 1] += tptr[i];
    std::vector<int64_t> pos(tptr.begin(), tptr.end() - 1);
    tidx.resize(size_t(nnz));
    tval.resize(size_t(nnz));
    for (int64_t o = 0; o < outerN; ++o)
        for (int64_t e = outer[o]; e < outer[o + 1]; ++e) {
            const int64_t p = pos[inner[e]]++;
            tidx[p] = int32_t(o);
            tval[p] = v[e];
        }
}

void check_compressed(const kr_compressed& c, int64_t outerN, int64_t innerN, const char* name) {
    if (c.outer_size != outerN) throw Fail{KR_CONTRACT, std::string(name) + " dimensions do not match Ahat/M"};
    if (!c.outer) throw Fail{KR_INVALID_INPUT, std::string(name) + ": null outer array"};
    if (c.outer[0] != 0) throw Fail{KR_INVALID_INPUT, std::string(name) + ": outer[0] must be 0"};
    for (int64_t o = 0; o < outerN; ++o)
        if (c.outer[o + 1] < c.outer[o]) throw Fail{KR_INVALID_INPUT, std::string(name) + ": outer not monotone"};
    const int64_t nnz = c.outer[outerN];
    if (nnz > 0 && (!c.inner || !c.val)) throw Fail{KR_INVALID_INPUT, std::string(name) + ": null arrays"};
    for (int64_t e = 0; e < nnz; ++e)
        if (c.inner[e] < 0 || c.inner[e] >= innerN)
            throw Fail{KR_INVALID_INPUT, std::string(name) + ": index out of range"};
}

// Classify a board's M (CSC).  0 identity, 1 chains, 2 general, 3 invalid.
int classify_m(const kr_compressed& m, int64_t k, std::string& why) {
    bool identity = m.outer[k] == k;
    for (int64_t j = 0; j < k; ++j) {
        const int64_t e = m.outer[j];
        if (e == m.outer[j + 1] || m.inner[e] != j || m.val[e] != 1.0) {
            why = "M is not unit lower triangular at column " + std::to_string(j);
            return 3;
        }
        if (m.outer[j + 1] - e != 1) identity = false;
    }
    if (identity) return 0;
    std::vector<int32_t> perRow(static_cast<size_t>(k), 0);
    bool chain = true;
    for (int64_t j = 0; j < k; ++j) {
        if (m.outer[j + 1] - m.outer[j] > 2) chain = false;
        for (int64_t e = m.outer[j] + 1; e < m.outer[j + 1]; ++e)
            if (++perRow[m.inner[e]] > 1) chain = false;
    }
    return chain ? 1 : 2;
}

struct BoardPlan {
    const kr_factors* f = nullptr;
    int64_t rowOff = 0, colOff = 0, kOff = 0;
    int mkind = 0;
    std::string why;
    // chain-sliced relabelling of this board's k coordinates (local): chains
    // sorted by length are cut into slices of 32; element j of the chain in
    // lane l of slice s sits at position sbase[s] + 32 j + l.
    int64_t kpad = 0;              // positions incl. padding (>= k)
    std::vector<int32_t> pos;      // t -> position
    std::vector<int32_t> at;       // position -> t, -1 = padding
    std::vector<double> mul;       // per position: M(t, previous t in chain)
    std::vector<int64_t> sbase;    // per slice
    std::vector<int32_t> slen;     // per slice lane: chain length
    std::vector<uint8_t> sneg;     // per slice lane: all multipliers are -1
    // SELL sizes and offsets in the combined arrays
    int64_t sl[4] = {0, 0, 0, 0}, pad[4] = {0, 0, 0, 0}, slOff[4] = {0, 0, 0, 0}, padOff[4] = {0, 0, 0, 0};
    int64_t nl[4] = {0, 0, 0, 0}, nlz[4] = {0, 0, 0, 0}, nlOff[4] = {0, 0, 0, 0}, nlzOff[4] = {0, 0, 0, 0};
    int32_t maxLen[4] = {0, 0, 0, 0};  // longest slice row per matrix
};

void build_chain_order(BoardPlan& p, bool chainMode) {
    const kr_factors& f = *p.f;
    const int64_t k = f.k;
    p.pos.assign(static_cast<size_t>(k), 0);
    p.at.clear();
    p.mul.clear();
    p.sbase.clear();
    p.slen.clear();
    p.sneg.clear();
    if (!chainMode) {
        for (int64_t t = 0; t < k; ++t) {
            p.pos[t] = int32_t(t);
            p.at.push_back(int32_t(t));
        }
        p.kpad = k;
        return;
    }
    std::vector<int64_t> nxt(static_cast<size_t>(k), -1);
    std::vector<double> mulOf(static_cast<size_t>(k), 0.0);
    std::vector<char> hasPrev(static_cast<size_t>(k), 0);
    for (int64_t j = 0; j < k; ++j)
        for (int64_t q = f.m.outer[j] + 1; q < f.m.outer[j + 1]; ++q) {
            nxt[j] = f.m.inner[q];
            mulOf[size_t(f.m.inner[q])] = f.m.val[q];
            hasPrev[size_t(f.m.inner[q])] = 1;
        }
    std::vector<std::vector<int32_t>> chains;
    for (int64_t j = 0; j < k; ++j) {
        if (hasPrev[j]) continue;
        chains.emplace_back();
        for (int64_t r = j; r >= 0; r = nxt[r]) chains.back().push_back(int32_t(r));
    }
    std::stable_sort(chains.begin(), chains.end(),
                     [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) { return a.size() > b.size(); });
    int64_t cur = 0;
    for (size_t s0 = 0; s0 < chains.size(); s0 += 32) {
        const int64_t width = int64_t(chains[s0].size());
        p.sbase.push_back(cur);
        p.at.resize(size_t(cur + 32 * width), -1);
        p.mul.resize(size_t(cur + 32 * width), 0.0);
        for (int l = 0; l < 32; ++l) {
            const size_t c = s0 + size_t(l);
            if (c >= chains.size()) {
                p.slen.push_back(0);
                p.sneg.push_back(1);
                continue;
            }
            bool neg = true;
            for (size_t j = 0; j < chains[c].size(); ++j) {
                const int32_t t = chains[c][j];
                const int64_t q = cur + 32 * int64_t(j) + l;
                p.pos[size_t(t)] = int32_t(q);
                p.at[size_t(q)] = t;
                p.mul[size_t(q)] = mulOf[size_t(t)];
                if (j > 0 && mulOf[size_t(t)] != -1.0) neg = false;
            }
            p.slen.push_back(int32_t(chains[c].size()));
            p.sneg.push_back(neg ? 1 : 0);
        }
        cur += 32 * width;
    }
    p.kpad = cur;
}

// Real k positions of a board in chain-major order (chain by chain, element
// by element): the order V^T and U^T rows are processed in, which keeps the
// rows of one window on one showdown sequence (one stripe of x') while the
// results land at their chain-sliced positions.
std::vector<int64_t> k_order(const BoardPlan& p) {
    std::vector<int64_t> out;
    out.reserve(size_t(p.f->k));
    if (p.sbase.empty()) {
        for (int64_t q = 0; q < p.kpad; ++q)
            if (p.at[size_t(q)] >= 0) out.push_back(q);
        return out;
    }
    for (size_t s = 0; s < p.sbase.size(); ++s)
        for (int l = 0; l < 32; ++l)
            for (int32_t j = 0; j < p.slen[s * 32 + size_t(l)]; ++j) out.push_back(p.sbase[s] + 32 * int64_t(j) + l);
    return out;
}

// The four matrices of one board in processing order with final indices.
//  which 0: VT (rows = k positions), 1: UA (rows = Ahat rows), 2: UT (rows =
//  k positions), 3: AV (rows = Ahat cols).
void board_rows(const BoardPlan& p, int which, int64_t R, int64_t K, bool xseq, int64_t M2, int32_t n2,
                HostRows& h) {
    const kr_factors& f = *p.f;
    h = HostRows{};
    auto xcol = [&](int64_t c) -> int32_t {  // global x index -> gather index
        const int64_t g = p.colOff + c;
        return xseq ? int32_t((g % n2) * M2 + g / n2) : int32_t(g);
    };
    auto kcol = [&](int64_t t) -> int32_t { return int32_t(p.kOff + p.pos[size_t(t)]); };
    if (which == 0) {
        for (int64_t q : k_order(p)) {
            const int64_t t = p.at[size_t(q)];
            for (int64_t e = f.v.outer[t]; e < f.v.outer[t + 1]; ++e) h.push(xcol(f.v.inner[e]), f.v.val[e]);
            h.endRow();
            h.outRow.push_back(int32_t(p.kOff + q));
        }
    } else if (which == 1) {
        for (int64_t i = 0; i < f.rows; ++i) {
            for (int64_t e = f.u.outer[i]; e < f.u.outer[i + 1]; ++e) h.push(kcol(f.u.inner[e]), f.u.val[e]);
            for (int64_t e = f.ahat.outer[i]; e < f.ahat.outer[i + 1]; ++e)
                h.push(int32_t(K + p.colOff + f.ahat.inner[e]), f.ahat.val[e]);
            h.endRow();
        }
    } else if (which == 2) {
        std::vector<int64_t> tp;
        std::vector<int32_t> ti;
        std::vector<double> tv;
        transpose_into(f.rows, f.k, f.u.outer, f.u.inner, f.u.val, tp, ti, tv);
        for (int64_t q : k_order(p)) {
            const int64_t t = p.at[size_t(q)];
            for (int64_t e = tp[t]; e < tp[t + 1]; ++e) h.push(int32_t(p.rowOff + ti[e]), tv[e]);
            h.endRow();
            h.outRow.push_back(int32_t(p.kOff + q));
        }
    } else {
        std::vector<int64_t> ap, vp;
        std::vector<int32_t> ai, vi;
        std::vector<double> av, vv;
        transpose_into(f.rows, f.cols, f.ahat.outer, f.ahat.inner, f.ahat.val, ap, ai, av);
        transpose_into(f.k, f.cols, f.v.outer, f.v.inner, f.v.val, vp, vi, vv);
        h.col.reserve(ai.size() + vi.size());
        h.val.reserve(ai.size() + vi.size());
        for (int64_t c = 0; c < f.cols; ++c) {
            for (int64_t e = ap[c]; e < ap[c + 1]; ++e) h.push(int32_t(p.rowOff + ai[e]), av[e]);
            for (int64_t e = vp[c]; e < vp[c + 1]; ++e) h.push(int32_t(R + kcol(vi[e])), vv[e]);
            h.endRow();
        }
    }
}

// Row lengths of the four matrices (for the sizing pass).
std::vector<int64_t> board_lengths(const BoardPlan& p, int which) {
    const kr_factors& f = *p.f;
    std::vector<int64_t> L;
    if (which == 0) {
        for (int64_t q : k_order(p)) {
            const int64_t t = p.at[size_t(q)];
            L.push_back(f.v.outer[t + 1] - f.v.outer[t]);
        }
    } else if (which == 1) {
        for (int64_t i = 0; i < f.rows; ++i)
            L.push_back(f.u.outer[i + 1] - f.u.outer[i] + f.ahat.outer[i + 1] - f.ahat.outer[i]);
    } else if (which == 2) {
        std::vector<int64_t> cnt(static_cast<size_t>(f.k), 0);
        for (int64_t e = 0; e < f.u.outer[f.rows]; ++e) cnt[size_t(f.u.inner[e])]++;
        for (int64_t q : k_order(p)) L.push_back(cnt[size_t(p.at[size_t(q)])]);
    } else {
        L.assign(static_cast<size_t>(f.cols), 0);
        for (int64_t e = 0; e < f.ahat.outer[f.rows]; ++e) L[size_t(f.ahat.inner[e])]++;
        for (int64_t e = 0; e < f.v.outer[f.k]; ++e) L[size_t(f.v.inner[e])]++;
    }
    return L;
}

void destroy_engine(kr_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    for (int q = 0; q < 2; ++q) {
        krb::HostPipe& P = e->pipe[q];
        for (auto* v : {&P.evIn, &P.evOut, &P.evMid, &P.evSolve})
            for (cudaEvent_t ev : *v) cudaEventDestroy(ev);
        for (cudaStream_t st : {P.copyIn, P.copyOut, P.stage2, P.stage3})
            if (st) cudaStreamDestroy(st);
        if (P.evStart) cudaEventDestroy(P.evStart);
        if (P.evEnd) cudaEventDestroy(P.evEnd);
        if (q == 1) {
            if (P.main) cudaStreamDestroy(P.main);
            krb::dev_free(P.d_in);
            krb::dev_free(P.d_out);
        }
    }
    {
        krb::QueuePipe& Q = e->queue;
        for (cudaStream_t st : {Q.cin, Q.cout, Q.comp[0], Q.comp[1]})
            if (st) cudaStreamDestroy(st);
        for (int d = 0; d < 2; ++d)
            for (int k = 0; k < 2; ++k) {
                for (cudaEvent_t ev : {Q.evIn[d][k], Q.evDone[d][k], Q.evOut[d][k]})
                    if (ev) cudaEventDestroy(ev);
                krb::dev_free(Q.in[d][k]);
                krb::dev_free(Q.out[d][k]);
            }
        for (cudaEvent_t ev : Q.evEnd)
            if (ev) cudaEventDestroy(ev);
        if (Q.evStart) cudaEventDestroy(Q.evStart);
    }
    for (auto& pg : e->pipeGraphs) cudaGraphExecDestroy(pg.exec);
    if (e->side) cudaStreamDestroy(e->side);
    if (e->evFork) cudaEventDestroy(e->evFork);
    if (e->evJoin) cudaEventDestroy(e->evJoin);
    kron_destroy(e->kron);
    kf_destroy(e->kf);
    free_sell(e->VT);
    free_sell(e->UA);
    free_sell(e->UT);
    free_sell(e->AV);
    krb::dev_free(e->chain_ptr);
    krb::dev_free(e->chain_len);
    krb::dev_free(e->chain_mul);
    krb::dev_free(e->chain_neg1);
    krb::dev_free(e->lvl_fwd_rows);
    krb::dev_free(e->lvl_bwd_cols);
    krb::dev_free(e->mr_ptr);
    krb::dev_free(e->mr_col);
    krb::dev_free(e->mr_val);
    krb::dev_free(e->mc_ptr);
    krb::dev_free(e->mc_row);
    krb::dev_free(e->mc_val);
    krb::dev_free(e->d_tz);
    krb::dev_free(e->d_tz2);
    krb::dev_free(e->d_xp);
    krb::dev_free(e->d_in);
    krb::dev_free(e->d_out);
    krb::dev_free(e->scBuf[0]);
    krb::dev_free(e->scBuf[1]);
    krb::dev_free(e->scStat);
    for (auto& p : e->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto ev : e->eventPool) cudaEventDestroy(ev);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

template <class F>
void parallel_boards(int nb, F&& body) {
    std::atomic<int> next{0};
    std::mutex mu;
    Fail firstFail{KR_OK, ""};
    auto worker = [&] {
        try {
            for (int b; (b = next.fetch_add(1)) < nb;) body(b);
        } catch (const Fail& f) {
            std::lock_guard<std::mutex> g(mu);
            if (firstFail.code == KR_OK) firstFail = f;
        } catch (const std::exception& x) {
            std::lock_guard<std::mutex> g(mu);
            if (firstFail.code == KR_OK) firstFail = Fail{KR_CUDA, x.what()};
        }
    };
    int nth = int(std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 16u));
    nth = std::min(nth, nb);
    std::vector<std::thread> pool;
    for (int t = 1; t < nth; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (firstFail.code != KR_OK) throw firstFail;
}

int group_count(int nb, uint32_t flags);
void make_pipeline(kr_engine* e);
}  // namespace
void set_carveout();
namespace {

kr_engine* create_engine(const kr_factors* boards, int nb, int device, uint32_t flags) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Fail{KR_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    }
    if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
    if (!boards || nb < 1) throw Fail{KR_INVALID_INPUT, "at least one factor set is required"};
    KR_CK(cudaSetDevice(device));

    std::vector<BoardPlan> plan(static_cast<size_t>(nb));
    int64_t R = 0, Cc = 0, K = 0, nA = 0, nU = 0, nV = 0, nM = 0;
    int32_t n1 = boards[0].n1, n2 = boards[0].n2;
    for (int b = 0; b < nb; ++b) {
        const kr_factors& f = boards[b];
        if (f.rows < 0 || f.cols < 0 || f.k < 0) throw Fail{KR_INVALID_INPUT, "negative dimension"};
        check_compressed(f.ahat, f.rows, f.cols, "Ahat");
        check_compressed(f.u, f.rows, f.k, "U");
        check_compressed(f.m, f.k, f.k, "M");
        check_compressed(f.v, f.k, f.cols, "V");
        if (f.n1 != n1 || f.n2 != n2) n1 = n2 = 0;
        BoardPlan& p = plan[size_t(b)];
        p.f = &f;
        p.rowOff = R;
        p.colOff = Cc;
        p.kOff = K;
        nA += f.ahat.outer[f.rows];
        nU += f.u.outer[f.rows];
        nV += f.v.outer[f.k];
        nM += f.m.outer[f.k];
        R += f.rows;
        Cc += f.cols;
        K += f.k;
        p.mkind = classify_m(f.m, f.k, p.why);
    }
    if (R + K > INT32_MAX || Cc + K > INT32_MAX) throw Fail{KR_INVALID_INPUT, "dimensions exceed 32-bit indices"};
    bool xseq = n2 > 0;
    for (auto& p : plan)
        if (xseq && (p.f->cols % n2 != 0)) xseq = false;
    // The sequence-major copy of x (x', k_seq_major_tile before V^T): about
    // 1% faster sustained at config 3 (2.2M columns), 2-5% slower on small
    // engines (one more launch per product than its locality saves).  On
    // from 1M columns of x; KR_XSEQ=0/1 overrides.
    {
        int64_t cols = 0;
        for (int b = 0; b < nb; ++b) cols += boards[b].cols;
        const char* env = std::getenv("KR_XSEQ");
        xseq = xseq && (env ? std::atoi(env) != 0 : cols >= 1000000);
    }

    kr_engine* e = new kr_engine();
    try {
        e->device = device;
        KR_CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->rows = R;
        e->cols = Cc;
        e->k = K;
        e->nnzA = nA;
        e->nnzU = nU;
        e->nnzV = nV;
        e->nnzM = nM;
        e->n1 = n1;
        e->n2 = n2;
        e->xseq = xseq;
        e->M2 = xseq ? Cc / n2 : 0;
        bool invalid = false, anyGeneral = false, allIdentity = true;
        for (auto& p : plan) {
            if (p.mkind == 3 && !invalid) {
                invalid = true;
                e->mfail = p.why;
            }
            if (p.mkind == 2) anyGeneral = true;
            if (p.mkind != 0) allIdentity = false;
        }
        e->mkind = invalid ? 3 : allIdentity ? 0 : anyGeneral ? 2 : 1;
        // flop rule (engine.hpp:72,77,90-91): the combined M is the identity
        // iff every board's is.
        e->flops_per_product = nV + nU + nA + (e->mkind == 0 ? 0 : nM - K);
        // Identity boards inside a chain engine are sets of singleton chains.
        const bool chainMode = e->mkind == 1;
        // Rows longer than longRow[w] take the warp-per-row path: a SELL
        // lane's row is a chain of dependent gather batches, a long row's
        // entries are gathered by 32 lanes at once and summed by one.  Per
        // matrix, the smallest threshold in {16, 32, ..., kLongRow} whose long
        // rows (over all boards) fit one resident round of warps
        // (kLongRowBudget); more long rows than that queue behind each other's
        // serial sums (config 2 at 128: 8,960 / 21,591 long V^T / AV rows,
        // 2.4x slower).  Measured (profiles/r02/long_rows_r02z.log): config-1
        // CFR+ 15,100 -> 17,900 it/s, config-4 DCFR 15,360 -> 16,950; configs
        // 2 and 3 keep 256.  KR_LONG_ROW=n: one fixed threshold.
        int64_t longRow[4] = {kLongRow, kLongRow, kLongRow, kLongRow};
        const int kThr = 5;
        const int64_t thr[5] = {16, 32, 64, 128, kLongRow};
        std::vector<int64_t> over(size_t(nb) * 4 * kThr, 0);  // [board][matrix][threshold]
        // pass 1: relabelling, long-row counts per threshold
        parallel_boards(nb, [&](int b) {
            BoardPlan& p = plan[size_t(b)];
            build_chain_order(p, chainMode);
            int64_t* o = over.data() + size_t(b) * 4 * kThr;
            for (int w = 0; w < 4; ++w)
                for (int64_t l : board_lengths(p, w))
                    for (int t = 0; t < kThr; ++t) o[w * kThr + t] += l > thr[t];
        });
        if (const char* env = std::getenv("KR_LONG_ROW")) {
            for (auto& l : longRow) l = std::max<int64_t>(8, std::atoll(env));
        } else {
            for (int w = 0; w < 4; ++w)
                for (int t = 0; t < kThr; ++t) {
                    int64_t n = 0;
                    for (int b = 0; b < nb; ++b) n += over[size_t(b) * 4 * kThr + size_t(w * kThr + t)];
                    if (n <= kLongRowBudget) {
                        longRow[w] = thr[t];
                        break;
                    }
                }
        }
        // SELL sizes
        parallel_boards(nb, [&](int b) {
            BoardPlan& p = plan[size_t(b)];
            for (int w = 0; w < 4; ++w)
                sell_sizes(board_lengths(p, w), longRow[w], p.sl[w], p.pad[w], p.nl[w], p.nlz[w]);
        });
        // internal k space: each board's chain-sliced positions, in board order
        int64_t Kp = 0;
        for (auto& p : plan) {
            p.kOff = Kp;
            Kp += p.kpad;
        }
        if (R + Kp > INT32_MAX || Cc + Kp > INT32_MAX)
            throw Fail{KR_INVALID_INPUT, "dimensions exceed 32-bit indices"};
        e->kpad = Kp;
        int64_t tsl[4] = {0, 0, 0, 0}, tpad[4] = {0, 0, 0, 0}, tnl[4] = {0, 0, 0, 0}, tnlz[4] = {0, 0, 0, 0};
        for (auto& p : plan)
            for (int w = 0; w < 4; ++w) {
                p.slOff[w] = tsl[w];
                p.padOff[w] = tpad[w];
                p.nlOff[w] = tnl[w];
                p.nlzOff[w] = tnlz[w];
                tsl[w] += p.sl[w];
                tpad[w] += p.pad[w];
                tnl[w] += p.nl[w];
                tnlz[w] += p.nlz[w];
            }
        krb::DevSell* mats[4] = {&e->VT, &e->UA, &e->UT, &e->AV};
        const int64_t nrowsOf[4] = {Kp, R, Kp, Cc};
        const int64_t nnzOf[4] = {nV, nU + nA, nU, nA + nV};
        for (int w = 0; w < 4; ++w) alloc_sell(*mats[w], nrowsOf[w], tsl[w], nnzOf[w], tpad[w], tnl[w], tnlz[w]);
        // SELL-C (opt-in, KR_SELL_COMP=1) for VT (all V,
        // coded), UA ([U coded | Ahat]) and AV ([Ahat^T | V coded]); U^T stays
        // plain.  Measured: half the bytes, no faster (the SpMVs are bound by
        // entries in flight and x gathers, not by DRAM bytes).
        const bool compOn = std::getenv("KR_SELL_COMP") != nullptr;
        // KR_SELL_CODES=0: 16-bit columns only, every value stays fp64 (codedSeg 2)
        const char* codesEnv = std::getenv("KR_SELL_CODES");
        const bool codesOn = !(codesEnv && std::atoi(codesEnv) == 0);
        const int codedSegOf[4] = {codesOn ? 0 : 2, codesOn ? 0 : 2, -1, codesOn ? 1 : 2};
        const int64_t splitOf[4] = {0, Kp, 0, R};
        std::atomic<bool> compFail[4] = {false, false, false, false};
        for (int w = 0; w < 4; ++w)
            if (compOn && codedSegOf[w] >= 0) {
                alloc_comp(*mats[w], nb);
                mats[w]->codedSeg = codedSegOf[w];
            }
        e->d_tz = dev_alloc<double>(std::max<int64_t>(Kp, 1));
        e->d_tz2 = dev_alloc<double>(std::max<int64_t>(Kp, 1));
        e->d_xp = dev_alloc<double>(std::max<int64_t>(Cc, 1));
        e->d_in = dev_alloc<double>(std::max<int64_t>(std::max(R, Cc), 1));
        e->d_out = dev_alloc<double>(std::max<int64_t>(std::max(R, Cc), 1));

        // pass 2: build and upload each board's slices
        parallel_boards(nb, [&](int b) {
            KR_CK(cudaSetDevice(device));
            cudaStream_t s;
            KR_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            const BoardPlan& p = plan[size_t(b)];
            const int64_t rowBase[4] = {p.kOff, p.rowOff, p.kOff, p.colOff};
            HostRows h;
            HostSell hs;
            for (int w = 0; w < 4; ++w) {
                board_rows(p, w, R, Kp, xseq, e->M2, n2, h);
                to_sell(h, rowBase[w], longRow[w], hs);
                if (int64_t(hs.sptr.size()) != p.sl[w] || int64_t(hs.col.size()) != p.pad[w] ||
                    int64_t(hs.lgrow.size()) != p.nl[w] || int64_t(hs.lcol.size()) != p.nlz[w])
                    throw Fail{KR_CUDA, "internal: SELL sizing mismatch"};
                upload_sell(hs, p.slOff[w], p.padOff[w], p.nlOff[w], p.nlzOff[w], *mats[w], s);
                if (mats[w]->col16 && !compFail[w].load()) {
                    HostComp hc;
                    compress_sell(hs, w == 1 || w == 3, splitOf[w], codedSegOf[w], hc);
                    if (hc.ok) upload_comp(hc, b, p.slOff[w], p.padOff[w], *mats[w], s);
                    else compFail[w] = true;
                }
                int32_t ml = 0;
                for (int32_t l : hs.llen) ml = std::max(ml, l);
                plan[size_t(b)].maxLen[w] = ml;
            }
            cudaStreamDestroy(s);
        });

        // M solve structures (global, relabelled indices).
        if (chainMode) {
            std::vector<int64_t> sbase;
            std::vector<int32_t> slen;
            std::vector<uint8_t> sneg;
            std::vector<double> cmul(static_cast<size_t>(Kp), 0.0);
            e->bCh.assign(1, 0);
            for (auto& p : plan) {
                for (int64_t b0 : p.sbase) sbase.push_back(p.kOff + b0);
                e->bCh.push_back(int64_t(sbase.size()));
                slen.insert(slen.end(), p.slen.begin(), p.slen.end());
                sneg.insert(sneg.end(), p.sneg.begin(), p.sneg.end());
                std::copy(p.mul.begin(), p.mul.end(), cmul.begin() + p.kOff);
            }
            e->nchains = int64_t(sbase.size());  // chain slices (32 chains each)
            sbase.push_back(Kp);                 // terminal: slice s spans [sbase[s], sbase[s+1])
            for (uint8_t v : sneg) e->chain_withmul |= v == 0;
            if (const char* env = std::getenv("KR_CHAIN")) e->chain_tma = std::string(env) != "reg";
            e->chain_ptr = dev_alloc<int64_t>(e->nchains + 1);
            e->chain_len = dev_alloc<int32_t>(std::max<int64_t>(32 * e->nchains, 1));
            e->chain_neg1 = dev_alloc<uint8_t>(std::max<int64_t>(32 * e->nchains, 1));
            e->chain_mul = dev_alloc<double>(std::max<int64_t>(Kp, 1));
            const int smem = int(size_t(kStages) * kChunkRows * 32 * sizeof(double) * 2);
            raise_smem_limit(k_chain_tma<1>, size_t(smem));
            raise_smem_limit(k_chain_tma<-1>, size_t(smem));
            if (e->nchains) {
                KR_CK(cudaMemcpy(e->chain_ptr, sbase.data(), 8 * sbase.size(), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(e->chain_len, slen.data(), 4 * slen.size(), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(e->chain_neg1, sneg.data(), sneg.size(), cudaMemcpyHostToDevice));
            }
            if (Kp) KR_CK(cudaMemcpy(e->chain_mul, cmul.data(), 8 * size_t(Kp), cudaMemcpyHostToDevice));
        } else if (e->mkind == 2) {
            std::vector<int64_t> cp{0};
            std::vector<int32_t> crow;
            std::vector<double> cval;
            for (auto& p : plan) {
                const kr_factors& f = *p.f;
                for (int64_t j = 0; j < f.k; ++j) {
                    for (int64_t q = f.m.outer[j] + 1; q < f.m.outer[j + 1]; ++q) {
                        crow.push_back(int32_t(p.kOff + f.m.inner[q]));
                        cval.push_back(f.m.val[q]);
                    }
                    cp.push_back(int64_t(crow.size()));
                }
            }
            std::vector<int64_t> rp;
            std::vector<int32_t> rcol;
            std::vector<double> rval;
            transpose_into(K, K, cp.data(), crow.data(), cval.data(), rp, rcol, rval);
            std::vector<int32_t> lf(static_cast<size_t>(K), 0), lb(static_cast<size_t>(K), 0);
            int32_t maxf = 0, maxb = 0;
            for (int64_t r = 0; r < K; ++r) {
                for (int64_t q = rp[r]; q < rp[r + 1]; ++q) lf[r] = std::max(lf[r], lf[rcol[q]] + 1);
                maxf = std::max(maxf, lf[r]);
            }
            for (int64_t j = K - 1; j >= 0; --j) {
                for (int64_t q = cp[j]; q < cp[j + 1]; ++q) lb[j] = std::max(lb[j], lb[crow[q]] + 1);
                maxb = std::max(maxb, lb[j]);
            }
            auto bucket = [&](const std::vector<int32_t>& lv, int32_t maxl, std::vector<int64_t>& lptr) {
                lptr.assign(size_t(maxl) + 2, 0);
                for (int64_t r = 0; r < K; ++r) lptr[size_t(lv[r]) + 1]++;
                for (int32_t l = 0; l <= maxl; ++l) lptr[l + 1] += lptr[l];
                std::vector<int64_t> pos(lptr.begin(), lptr.end() - 1);
                std::vector<int32_t> out(static_cast<size_t>(K));
                for (int64_t r = 0; r < K; ++r) out[pos[lv[r]]++] = int32_t(r);
                return out;
            };
            std::vector<int32_t> fr = bucket(lf, maxf, e->lvl_fwd_ptr);
            std::vector<int32_t> bc = bucket(lb, maxb, e->lvl_bwd_ptr);
            e->lvl_fwd_rows = dev_alloc<int32_t>(K);
            e->lvl_bwd_cols = dev_alloc<int32_t>(K);
            KR_CK(cudaMemcpy(e->lvl_fwd_rows, fr.data(), 4 * size_t(K), cudaMemcpyHostToDevice));
            KR_CK(cudaMemcpy(e->lvl_bwd_cols, bc.data(), 4 * size_t(K), cudaMemcpyHostToDevice));
            const int64_t no = int64_t(crow.size());
            e->mr_ptr = dev_alloc<int64_t>(K + 1);
            e->mc_ptr = dev_alloc<int64_t>(K + 1);
            e->mr_col = dev_alloc<int32_t>(std::max<int64_t>(no, 1));
            e->mc_row = dev_alloc<int32_t>(std::max<int64_t>(no, 1));
            e->mr_val = dev_alloc<double>(std::max<int64_t>(no, 1));
            e->mc_val = dev_alloc<double>(std::max<int64_t>(no, 1));
            KR_CK(cudaMemcpy(e->mr_ptr, rp.data(), 8 * size_t(K + 1), cudaMemcpyHostToDevice));
            KR_CK(cudaMemcpy(e->mc_ptr, cp.data(), 8 * size_t(K + 1), cudaMemcpyHostToDevice));
            if (no) {
                KR_CK(cudaMemcpy(e->mr_col, rcol.data(), 4 * size_t(no), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(e->mc_row, crow.data(), 4 * size_t(no), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(e->mr_val, rval.data(), 8 * size_t(no), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(e->mc_val, cval.data(), 8 * size_t(no), cudaMemcpyHostToDevice));
            }
        }
        for (int w = 0; w < 4; ++w)
            for (auto& p : plan) mats[w]->maxLen = std::max(mats[w]->maxLen, p.maxLen[w]);
        for (int w = 0; w < 4; ++w) {
            if (!mats[w]->col16) continue;
            if (compFail[w].load()) free_comp(*mats[w]);  // plain slots for this matrix
            else mats[w]->comp = true;
        }
        for (int w = 0; w < 4; ++w) {
            e->bSl[w].clear();
            e->bNl[w].clear();
            for (auto& p : plan) {
                e->bSl[w].push_back(p.slOff[w]);
                e->bNl[w].push_back(p.nlOff[w]);
            }
            e->bSl[w].push_back(tsl[w]);
            e->bNl[w].push_back(tnl[w]);
        }
        e->lean = std::getenv("KR_NO_LEAN") == nullptr;
        if (const char* env = std::getenv("KR_PF")) e->pf = std::max(0, std::atoi(env));
        for (int g1 : group_ends(nb, flags)) {
            e->grpBoard.push_back(g1);
            e->grpRow.push_back(g1 < nb ? plan[size_t(g1)].rowOff : R);
            e->grpCol.push_back(g1 < nb ? plan[size_t(g1)].colOff : Cc);
        }
        make_pipeline(e);
        KR_CK(cudaDeviceSynchronize());
    } catch (...) {
        destroy_engine(e);
        throw;
    }
    return e;
}

// Host-call pipeline resources: two copy streams and one event pair per group.
// Slice dispatch orders (DevSell::order_all / order_grp): a stable sort by
// width, widest first, within each board group (and over all slices with
// KR_LPT_ALL).  A group's launch lasts only ~50 us, so a wide slice (~30 us of
// dependent loads) dispatched late would set its length.  The whole-range
// launches keep storage order: there the tail is amortised and the sorted
// order measured 1-2% slower.  The sums are untouched (each row is still one
// lane's sequential sum).  KR_LPT=0 keeps storage order everywhere.
void build_orders(kr_engine* e) {
    if (const char* env = std::getenv("KR_LPT"))
        if (std::atoi(env) == 0) return;
    krb::DevSell* mats[4] = {&e->VT, &e->UA, &e->UT, &e->AV};
    const int G = e->ngroups();
    for (int w = 0; w < 4; ++w) {
        krb::DevSell& A = *mats[w];
        if (A.nslices < 2) continue;
        std::vector<int64_t> sp(size_t(A.nslices) + 1);
        KR_CK(cudaMemcpy(sp.data(), A.slice_ptr, 8 * sp.size(), cudaMemcpyDeviceToHost));
        auto sorted = [&](int64_t a, int64_t b) {  // slices [a, b), relative to a
            std::vector<int32_t> o(size_t(b - a));
            std::iota(o.begin(), o.end(), 0);
            std::stable_sort(o.begin(), o.end(), [&](int32_t i, int32_t j) {
                return sp[size_t(a + i) + 1] - sp[size_t(a + i)] > sp[size_t(a + j) + 1] - sp[size_t(a + j)];
            });
            return o;
        };
        if (std::getenv("KR_LPT_ALL")) {  // whole-range launches too (measured: -1-2%, off)
            std::vector<int32_t> all = sorted(0, A.nslices);
            A.order_all = dev_alloc<int32_t>(A.nslices);
            KR_CK(cudaMemcpy(A.order_all, all.data(), 4 * all.size(), cudaMemcpyHostToDevice));
        } else if (const char* ord = std::getenv("KR_ORDER"); ord && std::string(ord) == "sm") {
            // SM-affine: blocks are dealt to SMs round-robin, so launch block
            // r * nsm + q (likely on SM q) takes block r of SM q's contiguous
            // region of slices; an SM then works inside one or two boards' x.
            int nsm = 148;
            KR_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, e->device));
            const int64_t full = A.nslices / kWarpsPerBlock;  // whole blocks (a partial one stays last)
            std::vector<int32_t> all(size_t(A.nslices));
            std::iota(all.begin(), all.end(), 0);
            int64_t i = 0, maxReg = (full + nsm - 1) / nsm;
            for (int64_t r = 0; r < maxReg; ++r)
                for (int q = 0; q < nsm; ++q) {
                    const int64_t a = full * q / nsm, b = full * (q + 1) / nsm;
                    if (a + r >= b) continue;
                    for (int w = 0; w < kWarpsPerBlock; ++w)
                        all[size_t(i * kWarpsPerBlock + w)] = int32_t((a + r) * kWarpsPerBlock + w);
                    ++i;
                }
            A.order_all = dev_alloc<int32_t>(A.nslices);
            KR_CK(cudaMemcpy(A.order_all, all.data(), 4 * all.size(), cudaMemcpyHostToDevice));
        }
        if (G >= 2 && int64_t(e->bSl[w].size()) > int64_t(e->grpBoard.back())) {
            std::vector<int32_t> grp(size_t(A.nslices));
            for (int g = 0; g < G; ++g) {
                const int64_t a = e->bSl[w][size_t(e->grpBoard[size_t(g)])];
                const int64_t b = e->bSl[w][size_t(e->grpBoard[size_t(g) + 1])];
                std::vector<int32_t> o = sorted(a, b);
                std::copy(o.begin(), o.end(), grp.begin() + a);
            }
            A.order_grp = dev_alloc<int32_t>(A.nslices);
            KR_CK(cudaMemcpy(A.order_grp, grp.data(), 4 * grp.size(), cudaMemcpyHostToDevice));
        }
    }
}

// Streams and events of one host pipe (>= 2 board groups).
void make_host_pipe(kr_engine* e, krb::HostPipe& P) {
    const int G = e->ngroups();
    KR_CK(cudaStreamCreateWithFlags(&P.copyIn, cudaStreamNonBlocking));
    KR_CK(cudaStreamCreateWithFlags(&P.copyOut, cudaStreamNonBlocking));
    KR_CK(cudaStreamCreateWithFlags(&P.stage2, cudaStreamNonBlocking));
    KR_CK(cudaEventCreateWithFlags(&P.evStart, cudaEventDisableTiming));
    KR_CK(cudaEventCreateWithFlags(&P.evEnd, cudaEventDisableTiming));
    const char* ps = std::getenv("KR_PIPE_STREAMS");
    if (!(ps && std::atoi(ps) == 2)) KR_CK(cudaStreamCreateWithFlags(&P.stage3, cudaStreamNonBlocking));
    for (auto* v : {&P.evIn, &P.evOut, &P.evMid, &P.evSolve}) {
        v->resize(size_t(G));
        for (auto& ev : *v) KR_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    P.made = true;
}

void make_pipeline(kr_engine* e) {
    set_carveout();
    build_orders(e);
    e->pipe[0].main = e->stream;
    e->pipe[0].d_in = e->d_in;
    e->pipe[0].d_out = e->d_out;
    if (e->ngroups() < 2) return;
    make_host_pipe(e, e->pipe[0]);
}

// Board groups of the pipelined host-buffer calls: up to eight contiguous
// board ranges (KR_FLAG_SINGLE_PART: one; KR_GROUPS overrides the count).
// Measured at config 3 (profiles/r01l_e2e_pipeline.md): with the pipeline
// replayed as a graph, 8 groups 586 pairs/s, 6 580, 12 568, 16 519.
int group_count(int nb, uint32_t flags) {
    if (flags & KR_FLAG_SINGLE_PART) return 1;
    int G = 8;
    if (const char* env = std::getenv("KR_GROUPS")) G = std::atoi(env);
    return std::max(1, std::min(G, nb));
}

cudaEvent_t pool_event(kr_engine* e) {
    if (!e->eventPool.empty()) {
        cudaEvent_t ev = e->eventPool.back();
        e->eventPool.pop_back();
        return ev;
    }
    cudaEvent_t ev;
    KR_CK(cudaEventCreate(&ev));
    return ev;
}

// Boards [b0, b1) only when b1 >= 0 (a board's slices and long rows are
// contiguous: SELL windows never straddle boards); untimed.
// Deep batches (2 kU entries per lane per pipeline stage) for a launch of
// `blocks` CTAs over rows of up to maxLen entries.  In a small grid every
// SELL lane's row is a chain of dependent gather batches (each waits on L2),
// so fewer, wider batches shorten it; large grids are bandwidth-bound and keep
// kU (the registers buy residency).  Measured (profiles/r02/deep_batches_r02z.log):
// config-1 CFR+ 13,984 -> 15,100 it/s, config-2 factored DCFR 7,171 -> 7,712,
// config-4 DCFR 14,037 -> 15,357; 12 or 24 entries measured no better, 32
// spills.  KR_DEEP_KU=0: off; KR_DEEP_BLOCKS: the largest grid (default 8
// CTAs per SM).  Read per launch, so a process can switch.
bool deep_batches(int64_t blocks, int32_t maxLen) {
    const char* env = std::getenv("KR_DEEP_KU");
    if (env && std::atoi(env) == 0) return false;
    if (maxLen <= kU) return false;
    env = std::getenv("KR_DEEP_BLOCKS");
    return blocks <= (env ? std::atoll(env) : int64_t(1184));
}

void launch_sell(kr_engine* e, int which, const krb::DevSell& A, const double* xa, const double* xb, int64_t split,
                 double* y, cudaStream_t s, int b0 = 0, int b1 = -1) {
    int64_t s0 = 0, s1 = A.nslices, l0 = 0, l1 = A.nlong;
    if (b1 >= 0) {
        s0 = e->bSl[which][size_t(b0)];
        s1 = e->bSl[which][size_t(b1)];
        l0 = e->bNl[which][size_t(b0)];
        l1 = e->bNl[which][size_t(b1)];
    }
    const int64_t blocks = (l1 - l0 + kWarpsPerBlock - 1) / kWarpsPerBlock +
                           (s1 - s0 + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (blocks == 0) return;
    const int32_t* order = b1 < 0 ? A.order_all : A.order_grp ? A.order_grp + s0 : nullptr;
    // gather sources and outputs: V^T x (x or x': cols -> k), [U | Ahat] ([tz | x] -> rows),
    // U^T y (y: rows -> k), [Ahat^T | V] ([y | tz2] -> cols)
    const int64_t nsrc = which == 0 ? e->cols : which == 1 ? e->kpad + e->cols : which == 2 ? e->rows
                                                                                               : e->rows + e->kpad;
    const int64_t ndst = which == 0 || which == 2 ? e->kpad : which == 1 ? e->rows : e->cols;
    SellView v{A.slice_ptr + s0, A.lane_row + 32 * s0, A.lane_len + 32 * s0, A.col, A.val, s1 - s0,
               A.long_ptr + l0, A.long_row + l0, A.long_col, A.long_val, l1 - l0, order, e->pf, nsrc, ndst};
    const bool timed = e->timing && ((e->timingMask >> which) & 1) && b1 < 0;
    kr_engine::Pending pend{which, nullptr, nullptr};
    if (timed) {
        pend.a = pool_event(e);
        pend.b = pool_event(e);
        KR_CK(cudaEventRecord(pend.a, s));
    }
    if (A.comp) {
        const SellCView c{A.col16, A.code16, A.lane_len0 + 32 * s0, A.base0 + s0, A.base1 + s0, A.tbase + s0, A.table};
        if (!xb && A.codedSeg == 2)
            krb::launch(k_spmvc<false, 2>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, c, xa, nullptr, 0, y);
        else if (!xb) krb::launch(k_spmvc<false, 0>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, c, xa, nullptr, 0, y);
        else if (A.codedSeg == 2)
            krb::launch(k_spmvc<true, 2>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, c, xa, xb, int32_t(split), y);
        else if (A.codedSeg == 0)
            krb::launch(k_spmvc<true, 0>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, c, xa, xb, int32_t(split), y);
        else krb::launch(k_spmvc<true, 1>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, c, xa, xb, int32_t(split), y);
    } else if (A.maxLen <= 1 && e->lean && !xb) {
        const int64_t lb = (l1 - l0 + kWarpsPerBlock - 1) / kWarpsPerBlock +
                           (s1 - s0 + kWarpsPerBlock * kLeanSlices - 1) / (kWarpsPerBlock * kLeanSlices);
        krb::launch(k_spmv_lean, unsigned(lb), 32 * kWarpsPerBlock, 0, s, v, xa, y);
    }
    else if (deep_batches(blocks, A.maxLen)) {
        // small grids: each lane's row is a chain of dependent gather
        // batches, so twice the entries per batch halves it (same order)
        if (xb) krb::launch(k_spmv<true, 2 * kU>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, xa, xb, int32_t(split), y);
        else krb::launch(k_spmv<false, 2 * kU>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, xa, nullptr, 0, y);
    } else if (xb) krb::launch(k_spmv<true>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, xa, xb, int32_t(split), y);
    else krb::launch(k_spmv<false>, unsigned(blocks), 32 * kWarpsPerBlock, 0, s, v, xa, nullptr, 0, y);
    KR_CK_LAUNCH();
    if (timed) {
        KR_CK(cudaEventRecord(pend.b, s));
        e->pending.push_back(pend);
    }
    e->launches++;
}

// Algorithmic bytes of one launch of matrix `which`: fp64
// values + int32 indices of the factor entries it streams, int32 outer
// pointers of each merged factor, the input vector(s) read once and the
// output written once; the intermediates t / z are excluded, as in the
// per-matvec formula of BASELINE.md §2.
double launch_bytes(const kr_engine* e, int which) {
    const double R = double(e->rows), Cc = double(e->cols), K = double(e->k);
    switch (which) {
        case 0: return 12.0 * double(e->nnzV) + 4.0 * (K + 1) + 8.0 * Cc;
        case 1: return 12.0 * double(e->nnzU + e->nnzA) + 8.0 * (R + 1) + 8.0 * Cc + 8.0 * R;
        case 2: return 12.0 * double(e->nnzU) + 4.0 * (K + 1) + 8.0 * R;
        default: return 12.0 * double(e->nnzA + e->nnzV) + 8.0 * (Cc + 1) + 8.0 * R + 8.0 * Cc;
    }
}

size_t chain_smem(const kr_engine* e) {
    return size_t(kStages) * kChunkRows * 32 * sizeof(double) * (e->chain_withmul ? 2 : 1);
}

// Chain slices [c0, c1) (a board group's: slices are per board, in board
// order, bCh), or all of them (c1 < 0).
void solve_forward(kr_engine* e, cudaStream_t s, int64_t c0 = 0, int64_t c1 = -1) {
    if (c1 < 0) c1 = e->nchains;
    if (e->mkind == 1 && c1 > c0) {
        if (e->chain_tma) {
            krb::launch(k_chain_tma<1>, unsigned(c1 - c0), 32, chain_smem(e), s, e->chain_ptr, e->chain_len, e->chain_mul,
                                                                      e->chain_neg1, e->chain_withmul, e->d_tz, c0);
        } else {
            const int wpb = kWarpsPerBlock;
            krb::launch(k_chain_forward, unsigned((c1 - c0 + wpb - 1) / wpb), 32 * wpb, 0, s, e->chain_ptr, e->chain_len, e->chain_mul, e->chain_neg1, c0, c1, e->d_tz);
        }
        KR_CK_LAUNCH();
        e->launches++;
    } else if (e->mkind == 2) {
        for (size_t l = 0; l + 1 < e->lvl_fwd_ptr.size(); ++l) {
            const int64_t a = e->lvl_fwd_ptr[l], n = e->lvl_fwd_ptr[l + 1] - a;
            if (n == 0) continue;
            krb::launch(k_level_forward, unsigned((n + 127) / 128), 128, 0, s, e->lvl_fwd_rows + a, n, e->mr_ptr, e->mr_col,
                                                                      e->mr_val, e->d_tz);
            KR_CK_LAUNCH();
            e->launches++;
        }
    }
}

void solve_backward(kr_engine* e, cudaStream_t s, int64_t c0 = 0, int64_t c1 = -1) {
    if (c1 < 0) c1 = e->nchains;
    if (e->mkind == 1 && c1 > c0) {
        if (e->chain_tma) {
            krb::launch(k_chain_tma<-1>, unsigned(c1 - c0), 32, chain_smem(e), s, e->chain_ptr, e->chain_len, e->chain_mul,
                                                                       e->chain_neg1, e->chain_withmul, e->d_tz2, c0);
        } else {
            const int wpb = kWarpsPerBlock;
            krb::launch(k_chain_backward, unsigned((c1 - c0 + wpb - 1) / wpb), 32 * wpb, 0, s, e->chain_ptr, e->chain_len, e->chain_mul, e->chain_neg1, c0, c1, e->d_tz2);
        }
        KR_CK_LAUNCH();
        e->launches++;
    } else if (e->mkind == 2) {
        for (size_t l = 0; l + 1 < e->lvl_bwd_ptr.size(); ++l) {
            const int64_t a = e->lvl_bwd_ptr[l], n = e->lvl_bwd_ptr[l + 1] - a;
            if (n == 0) continue;
            krb::launch(k_level_backward, unsigned((n + 127) / 128), 128, 0, s, e->lvl_bwd_cols + a, n, e->mc_ptr,
                                                                       e->mc_row, e->mc_val, e->d_tz2);
            KR_CK_LAUNCH();
            e->launches++;
        }
    }
}

}  // namespace

// One board group's product (monolithic engine: the only group), no flop
// accounting.  Pointers address the whole vectors.
void engine_make_pipeline(kr_engine* e) { make_pipeline(e); }

// End board of each board group: G equal groups (group_count), or groups
// weighted by KR_GROUP_SIZES ("2,4,8,...": relative sizes, scaled to nb).
std::vector<int> group_ends(int nb, uint32_t flags) {
    std::vector<int> ends;
    const char* env = std::getenv("KR_GROUP_SIZES");
    if (env && !(flags & KR_FLAG_SINGLE_PART)) {
        std::vector<double> w;
        for (const char* p = env; *p;) {
            char* q = nullptr;
            const double v = std::strtod(p, &q);
            if (q == p) break;
            if (v > 0) w.push_back(v);
            p = *q == ',' ? q + 1 : q;
        }
        double tot = 0, cum = 0;
        for (double v : w) tot += v;
        for (double v : w) {
            cum += v;
            const int g1 = std::min(nb, int(std::lround(nb * cum / tot)));
            if (g1 > (ends.empty() ? 0 : ends.back())) ends.push_back(g1);
        }
        if (!ends.empty() && ends.back() != nb) ends.back() = nb;
        if (!ends.empty()) return ends;
    }
    const int G = group_count(nb, flags);
    for (int g = 0; g < G; ++g) ends.push_back(int(int64_t(nb) * (g + 1) / G));
    return ends;
}

void engine_chain_setup(kr_engine*) {
    const size_t smem = size_t(kStages) * kChunkRows * 32 * sizeof(double) * 2;
    raise_smem_limit(k_chain_tma<1>, smem);
    raise_smem_limit(k_chain_tma<-1>, smem);
}

// One preferred L1 / shared-memory split for every engine kernel (percent of
// the maximum shared memory), so kernels of different stages resident on an
// SM together never force it to drain and reconfigure (KR_CARVEOUT).
void set_carveout() {
    static const int pct = [] {
        const char* env = std::getenv("KR_CARVEOUT");
        return env ? std::atoi(env) : -1;
    }();
    static bool done = false;
    if (done || pct < 0) return;
    done = true;
    auto set = [](const void* f) { KR_CK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct)); };
    set(reinterpret_cast<const void*>(k_spmv<true>));
    set(reinterpret_cast<const void*>(k_spmv<false>));
    set(reinterpret_cast<const void*>(k_spmv_lean));
    set(reinterpret_cast<const void*>(k_seq_major_tile));
    set(reinterpret_cast<const void*>(k_seq_major));
    set(reinterpret_cast<const void*>(k_chain_tma<1>));
    set(reinterpret_cast<const void*>(k_chain_tma<-1>));
}

namespace {

// The product as first stage (per board group: the input-side kernels),
// middle (the M solve, all groups) and last stage (per group: the kernel
// writing the output).  Pointers address the whole vectors.
void seq_major(kr_engine* e, const double* x, int64_t c0, int64_t c1, cudaStream_t s) {
    if (c1 <= c0) return;
    const size_t smem = size_t(32) * size_t(e->n2) * sizeof(double);
    if (smem <= 48 * 1024 && c0 % e->n2 == 0 && c1 % e->n2 == 0) {
        const int64_t J0 = c0 / e->n2, J1 = c1 / e->n2;
        krb::launch(k_seq_major_tile, unsigned((J1 - J0 + 31) / 32), 256, smem, s, x, e->M2, e->n2, e->d_xp, J0, J1);
        KR_CK_LAUNCH();
        e->launches++;
        return;
    }
    krb::launch(k_seq_major, unsigned((c1 - c0 + 255) / 256), 256, 0, s, x, e->M2, e->n2, e->d_xp, c0, c1);
    KR_CK_LAUNCH();
    e->launches++;
}

void first_stage(kr_engine* e, int dir, const double* in, cudaStream_t s, int g = -1) {
    if (e->kron || e->kf) return;
    const int b0 = g < 0 ? 0 : e->grpBoard[size_t(g)], b1 = g < 0 ? -1 : e->grpBoard[size_t(g) + 1];
    if (dir == 0) {
        const double* xg = in;
        if (e->xseq && e->cols > 0) {
            seq_major(e, in, g < 0 ? 0 : e->grpCol[size_t(g)], g < 0 ? e->cols : e->grpCol[size_t(g) + 1], s);
            xg = e->d_xp;
        }
        launch_sell(e, 0, e->VT, xg, nullptr, 0, e->d_tz, s, b0, b1);      // t = V^T x    engine.hpp:65-72
    } else {
        launch_sell(e, 2, e->UT, in, nullptr, 0, e->d_tz2, s, b0, b1);     // s = U^T y    engine.hpp:103-110
    }
}

void middle(kr_engine* e, int dir, cudaStream_t s, int g = -1) {
    if (e->kron || e->kf) return;
    const int64_t c0 = g < 0 ? 0 : e->bCh[size_t(e->grpBoard[size_t(g)])];
    const int64_t c1 = g < 0 ? -1 : e->bCh[size_t(e->grpBoard[size_t(g) + 1])];
    if (dir == 0) solve_forward(e, s, c0, c1);   // z = M^-1 t    engine.hpp:74-78
    else solve_backward(e, s, c0, c1);           // z = M^-T s    engine.hpp:112-115
}

void last_stage(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int g = -1) {
    const int b0 = g < 0 ? 0 : e->grpBoard[size_t(g)], b1 = g < 0 ? -1 : e->grpBoard[size_t(g) + 1];
    if (e->kron) return kron_product(e, dir, in, out, s, b0, b1);
    if (e->kf) return kf_product(e, dir, in, out, s, b0, b1);
    if (dir == 0) launch_sell(e, 1, e->UA, e->d_tz, in, e->kpad, out, s, b0, b1);   // y = U z + Ahat x
    else launch_sell(e, 3, e->AV, in, e->d_tz2, e->rows, out, s, b0, b1);          // x = Ahat^T y + V z
}

// Cluster size of the fused small-engine product (k_tiny_product), 0 = the
// three launches.  Measured (profiles/r02/tiny_product_r02z.log): a product
// launched on a stream runs ~1.5-2x faster fused on the smallest engines (its
// three launches are each a launch latency), but inside a CUDA graph the
// three kernel nodes with programmatic dependent launch cost the same or less
// (twenty_card: 14.0 us three nodes, 16.5 us fused), so captured products --
// the solver's iterations, the host API's replayed graphs -- keep the three
// launches.  KR_TINY: the largest product (stored entries of the two SpMV
// stages + the chain positions) launched fused, everywhere including
// captures (0 = never; default 16384, outside captures only);
// KR_TINY_CLUSTER: CTAs per cluster (1 to 16, default 8).  Engines with
// per-stage timing, a sequence-major x, compressed slots or level-scheduled
// M keep the separate launches.
int tiny_cluster(const kr_engine* e, int dir, cudaStream_t s) {
    if (e->kron || e->kf || e->xseq || e->mkind > 1 || e->timing) return 0;
    const krb::DevSell& A1 = dir == 0 ? e->VT : e->UT;
    const krb::DevSell& A2 = dir == 0 ? e->UA : e->AV;
    if (A1.comp || A2.comp) return 0;
    // read per product (tens of ns against a launch), so a process can switch
    const char* env = std::getenv("KR_TINY");
    const int64_t lim = env ? std::atoll(env) : int64_t(16384);
    const int64_t nnz = e->nnzA + e->nnzU + e->nnzV + (e->mkind == 1 ? e->kpad : 0);
    if (nnz > lim) return 0;
    if (!env) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        KR_CK(cudaStreamIsCapturing(s, &cs));
        if (cs != cudaStreamCaptureStatusNone) return 0;
    }
    env = std::getenv("KR_TINY_CLUSTER");
    return env ? std::max(1, std::min(16, std::atoi(env))) : 8;
}

// false when the device cannot co-schedule a cluster of that shape (a
// partitioned GPU, too few SMs per GPC): the caller keeps the three launches.
template <int DIR>
bool launch_tiny(kr_engine* e, int cl, const double* in, double* out, cudaStream_t s) {
    const krb::DevSell& A1 = DIR == 0 ? e->VT : e->UT;
    const krb::DevSell& A2 = DIR == 0 ? e->UA : e->AV;
    const int64_t n1 = DIR == 0 ? e->cols : e->rows, n2 = DIR == 0 ? e->rows : e->cols;
    const int64_t src2 = DIR == 0 ? e->kpad + e->cols : e->rows + e->kpad;
    SellView v1{A1.slice_ptr, A1.lane_row, A1.lane_len, A1.col, A1.val, A1.nslices, A1.long_ptr, A1.long_row,
                A1.long_col, A1.long_val, A1.nlong, A1.order_all, e->pf, n1, e->kpad};
    SellView v2{A2.slice_ptr, A2.lane_row, A2.lane_len, A2.col, A2.val, A2.nslices, A2.long_ptr, A2.long_row,
                A2.long_col, A2.long_val, A2.nlong, A2.order_all, e->pf, src2, n2};
    const TinyChains C{e->chain_ptr, e->chain_len, e->chain_mul, e->chain_neg1, e->mkind == 1 ? e->nchains : 0,
                       e->chain_withmul};
    const size_t smem = C.n ? size_t(kTinyWarps) * kTinyRing * 8 * (C.withMul ? 2 : 1) : 0;
    double* tz = DIR == 0 ? e->d_tz : e->d_tz2;
    const int32_t split = int32_t(DIR == 0 ? e->kpad : e->rows);
    static bool attr = [] {
        KR_CK(cudaFuncSetAttribute(k_tiny_product<DIR>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        krb::raise_smem_limit(k_tiny_product<DIR>, size_t(kTinyWarps) * kTinyRing * 8 * 2);
        return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(cl));
    cfg.blockDim = dim3(32 * kTinyWarps);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(cl);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    {
        static std::mutex mu;
        static std::unordered_map<int64_t, bool> fits;  // (device, cluster, smem) -> schedulable
        const int64_t key = (int64_t(e->device) << 40) | (int64_t(cl) << 32) | int64_t(smem);
        std::lock_guard<std::mutex> lk(mu);
        auto it = fits.find(key);
        if (it == fits.end()) {
            cfg.numAttrs = 1;
            int n = 0;
            const bool ok = cudaOccupancyMaxActiveClusters(&n, k_tiny_product<DIR>, &cfg) == cudaSuccess && n > 0;
            (void)cudaGetLastError();
            it = fits.emplace(key, ok).first;
        }
        if (!it->second) return false;
    }
    unsigned& prev = krb::last_grid(s);
    cfg.numAttrs = krb::pdl_enabled(unsigned(cl), prev, false) ? 2 : 1;
    prev = unsigned(cl);
    KR_CK(cudaLaunchKernelEx(&cfg, k_tiny_product<DIR>, v1, v2, C, in, tz, split, out));
    KR_CK_LAUNCH();
    e->launches++;
    return true;
}

// The whole product, fused when the engine is small (tiny_cluster), else the
// three stages.
void product_stages(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s) {
    if (const int cl = tiny_cluster(e, dir, s))
        if (dir == 0 ? launch_tiny<0>(e, cl, in, out, s) : launch_tiny<1>(e, cl, in, out, s)) return;
    first_stage(e, dir, in, s);
    middle(e, dir, s);
    last_stage(e, dir, in, out, s);
}

void account(kr_engine* e, int dir) {
    e->flops_last = e->kron ? kron_flops(e, dir) : e->flops_per_product;
    e->flops_total += e->flops_last;
}

}  // namespace

void engine_product(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s) {
    if (e->mkind == 3) throw Fail{KR_CONTRACT, e->mfail};
    product_stages(e, dir, in, out, s);
    account(e, dir);
}

// SelfCheck reduction: max |got - exp| and max |exp| as the bit patterns of
// non-negative doubles (unsigned order == numeric order), then one verdict
// thread: err > tol (1 + max|exp|) sets the sticky flag (solver.hpp:84-91).
__global__ void k_sc_reduce(const double* __restrict__ got, const double* __restrict__ exp, int64_t n,
                            unsigned long long* __restrict__ stat) {
    krb::pdl_entry();
    double e = 0.0, m = 0.0;
    for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n; q += int64_t(gridDim.x) * blockDim.x) {
        const double x = exp[q];
        e = fmax(e, fabs(got[q] - x));
        m = fmax(m, fabs(x));
        if (got[q] != got[q] || x != x) e = __longlong_as_double(0x7ff0000000000000LL);  // NaN fails the check
    }
    for (int o = 16; o > 0; o >>= 1) {
        e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(stat, (unsigned long long)__double_as_longlong(e));
        atomicMax(stat + 1, (unsigned long long)__double_as_longlong(m));
    }
}
__global__ void k_sc_verdict(const unsigned long long* __restrict__ stat, double tol, double* __restrict__ flags) {
    krb::pdl_entry();
    const double err = __longlong_as_double((long long)stat[0]), scale = 1.0 + __longlong_as_double((long long)stat[1]);
    const double ratio = err / (tol * scale);
    if (!(err <= tol * scale)) flags[0] = 1.0;
    flags[1] = fmax(flags[1], ratio);
}

void engine_selfcheck(kr_engine* e, int dir, const double* in, const double* out, cudaStream_t s) {
    if (!e->scRef || e->scEvery < 1) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    KR_CK(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return;
    if (e->scCalls++ % e->scEvery != 0) return;  // SelfCheckEngine: calls_++ % every_ == 0
    const int64_t n = dir == 0 ? e->rows : e->cols;
    engine_product(e->scRef, dir, in, e->scBuf[dir], s);
    unsigned long long* st = reinterpret_cast<unsigned long long*>(e->scStat) + 2 * dir;
    KR_CK(cudaMemsetAsync(st, 0, 16, s));
    const unsigned grid = unsigned(std::min<int64_t>((n + 255) / 256, 4 * 148));
    krb::launch(k_sc_reduce, std::max(grid, 1u), 256, 0, s, out, e->scBuf[dir], n, st);
    KR_CK_LAUNCH();
    krb::launch(k_sc_verdict, 1, 1, 0, s, st, e->scTol, e->scStat + 4);
    KR_CK_LAUNCH();
    e->scChecks++;
}

void engine_selfcheck_raise(kr_engine* e) {
    if (!e->scRef) return;
    double f[2] = {0, 0};
    KR_CK(cudaMemcpy(f, e->scStat + 4, 16, cudaMemcpyDeviceToHost));
    if (f[0] != 0.0)
        throw Fail{KR_CONTRACT, "self-check: the gradient deviates from the reference engine by " +
                                    std::to_string(f[1]) + " x tol (1 + max|expect|) (solver.hpp:84-91)"};
}

bool engine_product_boards(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0, int b1) {
    if (e->kron) kron_product(e, dir, in, out, s, b0, b1);
    else if (e->kf) kf_product(e, dir, in, out, s, b0, b1);
    else return false;
    return true;
}
void engine_account(kr_engine* e, int dir) { account(e, dir); }
int engine_boards(const kr_engine* e) { return e->grpBoard.empty() ? 1 : e->grpBoard.back(); }

void engine_ax(kr_engine* e, const double* x, double* y, cudaStream_t s) { engine_product(e, 0, x, y, s); }
void engine_atx(kr_engine* e, const double* y, double* x, cudaStream_t s) { engine_product(e, 1, y, x, s); }

// Host-buffer product (the reference's synchronous Ax / ATx).  With several
// board groups the input copy of group g overlaps the first-stage kernels of
// the groups already copied, and the output copy of group g overlaps the
// last-stage kernels of the groups after it (copyIn / stream / copyOut).
void enqueue_pipeline(kr_engine* e, int dir, const double* hin, double* hout, const HostPipe& P);

bool pinned_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void check_sizes(const kr_engine* e, int dir, int64_t nin, int64_t nout) {
    const int64_t wantIn = dir == 0 ? e->cols : e->rows, wantOut = dir == 0 ? e->rows : e->cols;
    if (nin != wantIn)
        throw Fail{KR_INVALID_INPUT,
                   "matvec input has size " + std::to_string(nin) + ", expected " + std::to_string(wantIn)};
    if (nout != wantOut) throw Fail{KR_INVALID_INPUT, "matvec output has the wrong size"};
    if (e->mkind == 3) throw Fail{KR_CONTRACT, e->mfail};
}

// Replay the captured graph of this key, or capture it on the second call
// with the same pinned buffers (later calls replay it with one launch: the
// ~60 launches, copies and event edges per direction are no longer enqueued
// by the host one by one).  Returns true when the work has been launched.
// KR_NO_PIPE_GRAPH: always enqueue.
template <class Enqueue>
bool graph_call(kr_engine* e, int key, const double* in, double* out, const double* in2, double* out2,
                Enqueue&& enqueue) {
    if (std::getenv("KR_NO_PIPE_GRAPH")) return false;
    if (!pinned_host(in) || !pinned_host(out) || (in2 && (!pinned_host(in2) || !pinned_host(out2)))) return false;
    auto same = [&](const kr_engine::PipeGraph& pg) {
        return pg.dir == key && pg.in == in && pg.out == out && pg.in2 == in2 && pg.out2 == out2;
    };
    for (auto& pg : e->pipeGraphs)
        if (same(pg)) {
            KR_CK(cudaGraphLaunch(pg.exec, e->stream));
            e->launches += pg.launches;
            return true;
        }
    bool seen = false;
    for (auto& pg : e->pipeSeen) seen = seen || same(pg);
    if (seen && e->pipeGraphs.size() < 8) {
        const int64_t l0 = e->launches;
        cudaGraph_t gr;
        KR_CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            cudaStreamEndCapture(e->stream, &gr);
            cudaGetLastError();
            throw;
        }
        KR_CK(cudaStreamEndCapture(e->stream, &gr));
        cudaGraphExec_t exec;
        const cudaError_t ie = cudaGraphInstantiate(&exec, gr, 0);
        cudaGraphDestroy(gr);
        KR_CK(ie);
        const int64_t dl = e->launches - l0;
        e->launches = l0;
        e->pipeGraphs.push_back({key, in, out, exec, dl, in2, out2});
        KR_CK(cudaGraphLaunch(exec, e->stream));
        e->launches += dl;
        return true;
    }
    if (!seen && e->pipeSeen.size() < 16) e->pipeSeen.push_back({key, in, out, nullptr, 0, in2, out2});
    return false;
}

// One direction's copies and product on pipe P (P.main forked from and
// joined into e->stream by the caller when P.main != e->stream).
void enqueue_direction(kr_engine* e, int dir, const double* hin, double* hout, const HostPipe& P) {
    const int64_t nin = dir == 0 ? e->cols : e->rows, nout = dir == 0 ? e->rows : e->cols;
    if (e->ngroups() < 2) {
        KR_CK(cudaMemcpyAsync(P.d_in, hin, 8 * size_t(nin), cudaMemcpyHostToDevice, P.main));
        product_stages(e, dir, P.d_in, P.d_out, P.main);   // engine_product's; the caller accounts
        KR_CK(cudaMemcpyAsync(hout, P.d_out, 8 * size_t(nout), cudaMemcpyDeviceToHost, P.main));
        return;
    }
    enqueue_pipeline(e, dir, hin, hout, P);
}

void host_product(kr_engine* e, int dir, const double* hin, int64_t nin, double* hout, int64_t nout) {
    check_sizes(e, dir, nin, nout);
    KR_CK(cudaSetDevice(e->device));
    if (!graph_call(e, dir, hin, hout, nullptr, nullptr, [&] { enqueue_direction(e, dir, hin, hout, e->pipe[0]); }))
        enqueue_direction(e, dir, hin, hout, e->pipe[0]);
    engine_selfcheck(e, dir, e->pipe[0].d_in, e->pipe[0].d_out, e->stream);
    KR_CK(cudaStreamSynchronize(e->stream));
    account(e, dir);
    engine_selfcheck_raise(e);
}

// The second direction's pipe of kr_engine_pair (own streams, events and
// staging buffers, so the two directions' copies and kernels overlap).
void ensure_pair_pipe(kr_engine* e) {
    HostPipe& P = e->pipe[1];
    if (P.main) return;
    KR_CK(cudaStreamCreateWithFlags(&P.main, cudaStreamNonBlocking));
    const int64_t n = std::max<int64_t>(std::max(e->rows, e->cols), 1);
    P.d_in = dev_alloc<double>(n);
    P.d_out = dev_alloc<double>(n);
    if (e->ngroups() >= 2) make_host_pipe(e, P);
    if (!e->evFork) {
        KR_CK(cudaEventCreateWithFlags(&e->evFork, cudaEventDisableTiming));
        KR_CK(cudaEventCreateWithFlags(&e->evJoin, cudaEventDisableTiming));
    }
}

// kr_engine_pair: A x on pipe 0 (from e->stream) and A^T y on pipe 1, both
// directions' copies on the bus at once and their kernels side by side; one
// synchronisation at the end.  Each direction has its own scratch (d_tz /
// d_tz2, and the implicit engines' per-direction buffers), so the results are
// the bits of kr_engine_ax then kr_engine_atx.
void host_pair(kr_engine* e, const double* x, int64_t nx, double* ax, int64_t nax, const double* y, int64_t ny,
               double* atx, int64_t natx) {
    check_sizes(e, 0, nx, nax);
    check_sizes(e, 1, ny, natx);
    KR_CK(cudaSetDevice(e->device));
    ensure_pair_pipe(e);
    auto enqueue = [&] {
        KR_CK(cudaEventRecord(e->evFork, e->stream));
        KR_CK(cudaStreamWaitEvent(e->pipe[1].main, e->evFork, 0));
        enqueue_direction(e, 1, y, atx, e->pipe[1]);
        enqueue_direction(e, 0, x, ax, e->pipe[0]);
        KR_CK(cudaEventRecord(e->evJoin, e->pipe[1].main));
        KR_CK(cudaStreamWaitEvent(e->stream, e->evJoin, 0));
    };
    if (!graph_call(e, 2, x, ax, y, atx, enqueue)) enqueue();
    engine_selfcheck(e, 0, e->pipe[0].d_in, e->pipe[0].d_out, e->stream);
    engine_selfcheck(e, 1, e->pipe[1].d_in, e->pipe[1].d_out, e->stream);
    KR_CK(cudaStreamSynchronize(e->stream));
    account(e, 0);
    account(e, 1);
    engine_selfcheck_raise(e);
}

void ensure_queue(kr_engine* e) {
    QueuePipe& Q = e->queue;
    if (Q.made) return;
    for (cudaStream_t* st : {&Q.cin, &Q.cout, &Q.comp[0], &Q.comp[1]})
        KR_CK(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    for (int d = 0; d < 2; ++d)
        for (int k = 0; k < 2; ++k) {
            for (cudaEvent_t* ev : {&Q.evIn[d][k], &Q.evDone[d][k], &Q.evOut[d][k]})
                KR_CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
            Q.in[d][k] = dev_alloc<double>(std::max<int64_t>(d == 0 ? e->cols : e->rows, 1));
            Q.out[d][k] = dev_alloc<double>(std::max<int64_t>(d == 0 ? e->rows : e->cols, 1));
        }
    for (cudaEvent_t& ev : Q.evEnd) KR_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    KR_CK(cudaEventCreateWithFlags(&Q.evStart, cudaEventDisableTiming));
    Q.made = true;
}

// kr_engine_pair_queue: `count` independent pairs (x_i, y_i) -> (A x_i,
// A^T y_i), each result the bits of kr_engine_pair on that pair.  Pair i's
// products run whole (no board groups) on the direction's compute stream from
// slot i % 2; the copy of pair i + 1's inputs waits only for pair i - 1's
// products to have consumed that slot, the products of pair i only for pair
// i - 2's output copy to have drained theirs.  In steady state the bus carries
// inputs and outputs at once, back to back, and the kernels hide under them.
void host_pair_queue(kr_engine* e, int64_t count, const double* const* xs, int64_t nx, double* const* axs,
                     int64_t nax, const double* const* ys, int64_t ny, double* const* atxs, int64_t natx) {
    check_sizes(e, 0, nx, nax);
    check_sizes(e, 1, ny, natx);
    if (count <= 0) return;
    for (int64_t i = 0; i < count; ++i)
        if (!xs[i] || !axs[i] || !ys[i] || !atxs[i]) throw Fail{KR_INVALID_INPUT, "null buffer in the pair queue"};
    KR_CK(cudaSetDevice(e->device));
    if (e->scRef) {  // SelfCheck compares every N-th product: pair by pair
        for (int64_t i = 0; i < count; ++i) host_pair(e, xs[i], nx, axs[i], nax, ys[i], ny, atxs[i], natx);
        return;
    }
    ensure_queue(e);
    QueuePipe& Q = e->queue;
    KR_CK(cudaEventRecord(Q.evStart, e->stream));
    for (cudaStream_t st : {Q.cin, Q.cout, Q.comp[0], Q.comp[1]}) KR_CK(cudaStreamWaitEvent(st, Q.evStart, 0));
    for (int64_t i = 0; i < count; ++i) {
        const int k = int(i & 1);
        for (int d : {1, 0}) {  // A^T y first, as kr_engine_pair
            const double* hin = d == 0 ? xs[i] : ys[i];
            double* hout = d == 0 ? axs[i] : atxs[i];
            const int64_t nin = d == 0 ? nx : ny, nout = d == 0 ? nax : natx;
            if (i >= 2) KR_CK(cudaStreamWaitEvent(Q.cin, Q.evDone[d][k], 0));
            KR_CK(cudaMemcpyAsync(Q.in[d][k], hin, 8 * size_t(nin), cudaMemcpyHostToDevice, Q.cin));
            KR_CK(cudaEventRecord(Q.evIn[d][k], Q.cin));
            KR_CK(cudaStreamWaitEvent(Q.comp[d], Q.evIn[d][k], 0));
            if (i >= 2) KR_CK(cudaStreamWaitEvent(Q.comp[d], Q.evOut[d][k], 0));
            first_stage(e, d, Q.in[d][k], Q.comp[d]);
            middle(e, d, Q.comp[d]);
            last_stage(e, d, Q.in[d][k], Q.out[d][k], Q.comp[d]);
            KR_CK(cudaEventRecord(Q.evDone[d][k], Q.comp[d]));
            KR_CK(cudaStreamWaitEvent(Q.cout, Q.evDone[d][k], 0));
            KR_CK(cudaMemcpyAsync(hout, Q.out[d][k], 8 * size_t(nout), cudaMemcpyDeviceToHost, Q.cout));
            KR_CK(cudaEventRecord(Q.evOut[d][k], Q.cout));
        }
    }
    int j = 0;
    for (cudaStream_t st : {Q.cin, Q.cout, Q.comp[0], Q.comp[1]}) {
        KR_CK(cudaEventRecord(Q.evEnd[j], st));
        KR_CK(cudaStreamWaitEvent(e->stream, Q.evEnd[j++], 0));
    }
    KR_CK(cudaStreamSynchronize(e->stream));
    for (int64_t i = 0; i < count; ++i) {
        account(e, 0);
        account(e, 1);
    }
}

// The pipelined host-buffer product (board groups), enqueued from and
// joined back into P.main: every stream it uses waits for the work already
// queued on P.main, and P.main waits for all of it.
void enqueue_pipeline(kr_engine* e, int dir, const double* hin, double* hout, const HostPipe& P) {
    const int G = e->ngroups();
    const std::vector<int64_t>& io = dir == 0 ? e->grpCol : e->grpRow;
    const std::vector<int64_t>& oo = dir == 0 ? e->grpRow : e->grpCol;
    KR_CK(cudaEventRecord(P.evStart, P.main));
    for (cudaStream_t q : {P.copyIn, P.copyOut, P.stage2, P.stage3})
        if (q) KR_CK(cudaStreamWaitEvent(q, P.evStart, 0));
    auto copy_out = [&](int g, cudaStream_t from) {
        KR_CK(cudaEventRecord(P.evOut[size_t(g)], from));
        KR_CK(cudaStreamWaitEvent(P.copyOut, P.evOut[size_t(g)], 0));
        const size_t a = size_t(oo[size_t(g)]), n = size_t(oo[size_t(g) + 1]) - a;
        KR_CK(cudaMemcpyAsync(hout + a, P.d_out + a, 8 * n, cudaMemcpyDeviceToHost, P.copyOut));
    };
    // Input copies run two groups ahead of the kernel enqueue: group g's
    // kernels are queued before its input lands (enqueueing every copy first
    // delayed the first kernels by ~30 us of host time), and copy g+2 is
    // enqueued while copy g+1 (~60 us on the bus) is still running, since a
    // group's kernels take the host ~40-90 us to enqueue.
    int nextIn = 0;
    auto copy_in = [&](int upto) {
        for (; nextIn < std::min(upto + 1, G); ++nextIn) {
            const int g = nextIn;
            const size_t a = size_t(io[size_t(g)]), n = size_t(io[size_t(g) + 1]) - a;
            KR_CK(cudaMemcpyAsync(P.d_in + a, hin + a, 8 * n, cudaMemcpyHostToDevice, P.copyIn));
            KR_CK(cudaEventRecord(P.evIn[size_t(g)], P.copyIn));
        }
    };
    // Every factor is block diagonal over boards, and so is M's chain solve
    // (chain slices per board, bCh): with chains (or none) a group's whole
    // product runs as soon as its input has arrived: its first SpMV on the
    // main stream, its M solve on stage3 (latency-bound: it hides under the
    // SpMVs of the groups around it), its last SpMV on stage2 while the next
    // group's first SpMV streams on the main stream (each kernel's tail under
    // the other's), its output copy on copyOut.  The level solve (mkind 2)
    // spans boards, so there it waits for every group's first stage.
    if (e->kron || e->kf) {
        for (int g = 0; g < G; ++g) {
            copy_in(g + 1);
            KR_CK(cudaStreamWaitEvent(P.main, P.evIn[size_t(g)], 0));
            last_stage(e, dir, P.d_in, P.d_out, P.main, g);
            copy_out(g, P.main);
        }
    } else if (e->mkind == 0 ||
               (e->mkind == 1 && int64_t(e->bCh.size()) == int64_t(e->grpBoard.back()) + 1)) {
        // KR_PIPE_STREAMS=2: the M solve on stage2 ahead of the last SpMV
        const bool three = P.stage3 != nullptr;
        for (int g = 0; g < G; ++g) {
            copy_in(g + 1);
            KR_CK(cudaStreamWaitEvent(P.main, P.evIn[size_t(g)], 0));
            first_stage(e, dir, P.d_in, P.main, g);
            KR_CK(cudaEventRecord(P.evMid[size_t(g)], P.main));
            if (three) {  // the latency-bound solve on its own stream
                KR_CK(cudaStreamWaitEvent(P.stage3, P.evMid[size_t(g)], 0));
                middle(e, dir, P.stage3, g);
                KR_CK(cudaEventRecord(P.evSolve[size_t(g)], P.stage3));
                KR_CK(cudaStreamWaitEvent(P.stage2, P.evSolve[size_t(g)], 0));
            } else {
                KR_CK(cudaStreamWaitEvent(P.stage2, P.evMid[size_t(g)], 0));
                middle(e, dir, P.stage2, g);
            }
            last_stage(e, dir, P.d_in, P.d_out, P.stage2, g);
            copy_out(g, P.stage2);
        }
    } else {
        copy_in(G - 1);
        for (int g = 0; g < G; ++g) {
            KR_CK(cudaStreamWaitEvent(P.main, P.evIn[size_t(g)], 0));
            first_stage(e, dir, P.d_in, P.main, g);
        }
        middle(e, dir, P.main);
        for (int g = 0; g < G; ++g) {
            last_stage(e, dir, P.d_in, P.d_out, P.main, g);
            copy_out(g, P.main);
        }
    }
    KR_CK(cudaEventRecord(P.evEnd, P.copyOut));
    KR_CK(cudaStreamWaitEvent(P.main, P.evEnd, 0));
}

}  // namespace krb

using krb::Fail;
using krb::guarded;

extern "C" {

const char* kr_last_error(int* code) {
    if (code) *code = krb::g_code;
    return krb::g_msg.c_str();
}

int64_t kr_checked_verify(void) {
#ifdef KR_CHECKED
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> g(krb::g_checked_mu);
    int64_t bad = krb::g_checked_bad;
    for (auto& [p, a] : krb::checked_allocs()) bad += krb::guards_intact(p, a) ? 0 : 1;
    return bad;
#else
    return -1;
#endif
}

#ifdef KR_CHECKED
namespace {
__global__ void k_checked_poke(double* p, int64_t i, int checkIndex, int64_t n) {
    if (checkIndex) KR_DCHECK(i < n);
    p[i] = 1.0;
}
}  // namespace
#endif

int64_t kr_checked_selftest(int mode) {
#ifdef KR_CHECKED
    // mode 0: write one element past a 100-double allocation and report how
    // many corrupted guard zones kr_checked_verify finds (1), leaving the
    // global count as it was; mode 1: the same write behind a failing
    // KR_DCHECK (traps: the context is lost, run it in a child process)
    double* p = krb::dev_alloc<double>(100);
    k_checked_poke<<<1, 1>>>(p, 100, mode == 1, 100);
    const cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) return -int64_t(err);
    int64_t found = 0;
    {
        std::lock_guard<std::mutex> g(krb::g_checked_mu);
        auto it = krb::checked_allocs().find(p);
        found = krb::guards_intact(p, it->second) ? 0 : 1;
        cudaFree(it->second.base);
        krb::checked_allocs().erase(it);
    }
    return found;
#else
    (void)mode;
    return -1;
#endif
}

int kr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int kr_engine_create(const kr_factors* f, int device, uint32_t flags, kr_engine** out) {
    return guarded([&] {
        if (!out) throw Fail{KR_INVALID_INPUT, "null output handle"};
        *out = krb::create_engine(f, 1, device, flags);
    });
}

int kr_engine_create_boards(const kr_factors* boards, int nboards, int device, uint32_t flags, kr_engine** out) {
    return guarded([&] {
        if (!out) throw Fail{KR_INVALID_INPUT, "null output handle"};
        *out = krb::create_engine(boards, nboards, device, flags);
    });
}

int kr_engine_destroy(kr_engine* e) {
    return guarded([&] { krb::destroy_engine(e); });
}

int kr_engine_dims(const kr_engine* e, int64_t out[8]) {
    return guarded([&] {
        if (!e || !out) throw Fail{KR_INVALID_INPUT, "null argument"};
        const int64_t v[8] = {e->rows, e->cols, e->k, e->nnzA, e->nnzU, e->nnzM, e->nnzV, e->mkind == 0 ? 1 : 0};
        std::memcpy(out, v, sizeof(v));
    });
}

int kr_engine_ax(kr_engine* e, const double* x, int64_t nx, double* y, int64_t ny) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        krb::host_product(e, 0, x, nx, y, ny);
    });
}

int kr_engine_atx(kr_engine* e, const double* y, int64_t ny, double* x, int64_t nx) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        krb::host_product(e, 1, y, ny, x, nx);
    });
}

int kr_engine_pair(kr_engine* e, const double* x, int64_t nx, double* ax, int64_t nax, const double* y, int64_t ny,
                   double* atx, int64_t natx) {
    return guarded([&] {
        if (!e || !x || !ax || !y || !atx) throw Fail{KR_INVALID_INPUT, "null argument"};
        if (x == atx || y == ax) throw Fail{KR_INVALID_INPUT, "pair outputs must not alias the other direction's input"};
        krb::host_pair(e, x, nx, ax, nax, y, ny, atx, natx);
    });
}

int kr_engine_pair_queue(kr_engine* e, int64_t count, const double* const* xs, int64_t nx, double* const* axs,
                         int64_t nax, const double* const* ys, int64_t ny, double* const* atxs, int64_t natx) {
    return guarded([&] {
        if (!e || (count > 0 && (!xs || !axs || !ys || !atxs))) throw Fail{KR_INVALID_INPUT, "null argument"};
        if (count < 0) throw Fail{KR_INVALID_INPUT, "negative pair count"};
        for (int64_t i = 0; i < count; ++i)
            if (xs[i] == atxs[i] || ys[i] == axs[i])
                throw Fail{KR_INVALID_INPUT, "pair outputs must not alias the other direction's input"};
        krb::host_pair_queue(e, count, xs, nx, axs, nax, ys, ny, atxs, natx);
    });
}

int kr_engine_ax_device(kr_engine* e, const double* x, double* y, void* stream) {
    return guarded([&] {
        if (!e || !x || !y) throw Fail{KR_INVALID_INPUT, "null argument"};
        KR_CK(cudaSetDevice(e->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->stream;
        krb::engine_ax(e, x, y, s);
        krb::engine_selfcheck(e, 0, x, y, s);
    });
}

int kr_engine_atx_device(kr_engine* e, const double* y, double* x, void* stream) {
    return guarded([&] {
        if (!e || !x || !y) throw Fail{KR_INVALID_INPUT, "null argument"};
        KR_CK(cudaSetDevice(e->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->stream;
        krb::engine_atx(e, y, x, s);
        krb::engine_selfcheck(e, 1, y, x, s);
    });
}

int kr_engine_pair_device(kr_engine* e, const double* x, double* ax, const double* y, double* atx, void* stream) {
    return guarded([&] {
        if (!e || !x || !ax || !y || !atx) throw Fail{KR_INVALID_INPUT, "null argument"};
        KR_CK(cudaSetDevice(e->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->stream;
        // Above ~8 GB of factor traffic per pair (KR_PAIR_SERIAL_GB) both
        // directions are bandwidth-bound on their own and running them
        // together measured 3-6% slower (profiles/r01p_sweep.md): one after
        // the other there.
        const char* sgb = std::getenv("KR_PAIR_SERIAL_GB");
        const double serialGB = sgb ? std::atof(sgb) : 8.0;
        const double pairGB = (e->kron || e->kf) ? 0.0 : 12e-9 * 2.0 * double(e->nnzA + e->nnzU + e->nnzV);
        if (pairGB > serialGB) {
            krb::engine_ax(e, x, ax, s);
            krb::engine_selfcheck(e, 0, x, ax, s);
            krb::engine_atx(e, y, atx, s);
            krb::engine_selfcheck(e, 1, y, atx, s);
            return;
        }
        if (!e->side) {
            // KR_PAIR_PRIORITY (measurement knob): the side stream's priority
            const char* pr = std::getenv("KR_PAIR_PRIORITY");
            KR_CK(cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking, pr ? std::atoi(pr) : 0));
            KR_CK(cudaEventCreateWithFlags(&e->evFork, cudaEventDisableTiming));
            KR_CK(cudaEventCreateWithFlags(&e->evJoin, cudaEventDisableTiming));
        }
        // A^T y on the side stream, A x on s; s then waits for both
        KR_CK(cudaEventRecord(e->evFork, s));
        KR_CK(cudaStreamWaitEvent(e->side, e->evFork, 0));
        krb::engine_atx(e, y, atx, e->side);
        krb::engine_selfcheck(e, 1, y, atx, e->side);
        krb::engine_ax(e, x, ax, s);
        krb::engine_selfcheck(e, 0, x, ax, s);
        KR_CK(cudaEventRecord(e->evJoin, e->side));
        KR_CK(cudaStreamWaitEvent(s, e->evJoin, 0));
    });
}

int kr_engine_set_selfcheck(kr_engine* e, kr_engine* reference, int every, double tol) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        KR_CK(cudaSetDevice(e->device));
        if (!reference) {
            e->scRef = nullptr;
            return;
        }
        if (reference == e) throw Fail{KR_INVALID_INPUT, "an engine cannot check itself"};
        if (reference->device != e->device) throw Fail{KR_INVALID_INPUT, "reference engine on another device"};
        if (reference->rows != e->rows || reference->cols != e->cols)
            throw Fail{KR_INVALID_INPUT, "reference engine has other dimensions"};
        if (every < 1 || !(tol > 0)) throw Fail{KR_INVALID_INPUT, "self-check period and tolerance must be positive"};
        for (int d = 0; d < 2; ++d)
            if (!e->scBuf[d]) e->scBuf[d] = krb::dev_alloc<double>(std::max<int64_t>(d == 0 ? e->rows : e->cols, 1));
        if (!e->scStat) e->scStat = krb::dev_alloc<double>(6);
        KR_CK(cudaMemset(e->scStat, 0, 6 * sizeof(double)));
        e->scRef = reference;
        e->scEvery = every;
        e->scTol = tol;
        e->scCalls = e->scChecks = 0;
    });
}

int kr_engine_selfcheck_status(kr_engine* e, int64_t* checks, double* worst) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        KR_CK(cudaSetDevice(e->device));
        KR_CK(cudaStreamSynchronize(e->stream));
        double f[2] = {0, 0};
        if (e->scStat) KR_CK(cudaMemcpy(f, e->scStat + 4, 16, cudaMemcpyDeviceToHost));
        if (checks) *checks = e->scChecks;
        if (worst) *worst = f[1];
        krb::engine_selfcheck_raise(e);
    });
}

int kr_engine_set_timing_mask(kr_engine* e, int mask) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        e->timingMask = mask & 0xF;
    });
}

int kr_engine_set_timing(kr_engine* e, int enabled) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        e->timing = enabled != 0;
    });
}

int kr_engine_kernel_times(kr_engine* e, int64_t launches[4], double ms[4], double bytes[4]) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        KR_CK(cudaSetDevice(e->device));
        for (auto& p : e->pending) {
            KR_CK(cudaEventSynchronize(p.b));
            float t = 0;
            KR_CK(cudaEventElapsedTime(&t, p.a, p.b));
            e->tLaunches[p.which]++;
            e->tMs[p.which] += double(t);
            e->eventPool.push_back(p.a);
            e->eventPool.push_back(p.b);
        }
        e->pending.clear();
        for (int w = 0; w < 4; ++w) {
            if (launches) launches[w] = e->tLaunches[w];
            if (ms) ms[w] = e->tMs[w];
            if (bytes) bytes[w] = krb::launch_bytes(e, w);
            e->tLaunches[w] = 0;
            e->tMs[w] = 0;
        }
    });
}

int64_t kr_engine_flops(const kr_engine* e) { return e ? e->flops_total : 0; }
int64_t kr_engine_last_flops(const kr_engine* e) { return e ? e->flops_last : 0; }
void* kr_engine_stream(const kr_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }
int kr_engine_device(const kr_engine* e) { return e ? e->device : -1; }
int64_t kr_engine_launches(const kr_engine* e) { return e ? e->launches : 0; }

void* kr_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, size_t(bytes)) != cudaSuccess) {
        cudaGetLastError();
        krb::set_error(KR_CUDA, "cudaMallocHost failed");
        return nullptr;
    }
    return p;
}

void kr_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
