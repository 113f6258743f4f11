// kr_devengine.cu — the factored engine built entirely on the device from the
// boards' KronPayoff pieces: Technique B with
// postprocessing (sparsify.hpp:246-406) generated row by row straight into
// the engine's own layout (chain-sliced k positions, SELL-32 windows, long
// rows), with no factor arrays and no layout work on the host.
//
// Only each output row's entry ORDER is fixed (the reference's storage order,
// engine.hpp:67-70, 82-88, 104-108, 118-129); the layout is free.  Each of the
// engine's four matrices has a device row enumerator emitting its entries in
// that order, with every value computed by the host builder's expressions
// (kr_factors_dev.cu, techniqueBPost), so products equal the host-built
// engine's bit for bit (tests/test_gpu_factors_device.py).
//   VT row k (i,d)  j asc, S row d asc: (lambda2_j * Y_ij) * S_db  at x' index
//                   (rows chain-major, written to their relabelled positions)
//   VT row f(d)     j asc, F row d asc:  lambda2_j * F_db
//   UA row (i,a)    [last kept column of chain a] [f(a)]: lambda1_i; then the
//                   blocked j asc, F row a asc: (-lambda1_i * lambda2_j) * F_ab
//   UT row k        the U rows (i', d) whose last kept column is k, i' asc
//   AV row (j,b)    blocked i asc, F column b asc: (-lambda1_i * lambda2_j) * F_ab;
//                   then k asc: V entries (j,b | k)
// k relabelling: the S chains (one per sequence d with a showdown, nAlive
// long, multipliers -1) are packed 32 per slice (element r of chain c at
// base + 32 r + c % 32), the F columns are singletons after them.
// Windows of 1024 rows are sorted by length in shared memory (bitonic), cut
// into slices of 32; rows longer than kLongRow go to the long-row CSR.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <numeric>
#include <string>
#include <vector>

#include "kr_common.cuh"

namespace krb {
namespace {

constexpr int kWin = 1024;

struct BoardDev {
    int m1, m2, n1, n2;
    int64_t rowOff, colOff, hand2Off, kOff;  // global y row / x col / player-2 hand / k position offsets
    int64_t rowsTotal, kpadTotal, M2;        // merged-index splits and x' stride
    const uint32_t *key1, *key2;
    const uint8_t *c1, *c2;
    const double *l1, *l2;
    const int64_t* fptr;  const int32_t* fcol;  const double* fval;   // F CSR
    const int64_t* fcptr; const int32_t* fcrow; const double* fcval;  // F CSC
    const int64_t* sptr;  const int32_t* scol;  const double* sval;   // S CSR
    const int64_t* scptr; const int32_t* scrow; const double* scval;  // S CSC
    const int32_t *blk2ptr, *blk2;  // per player-1 hand: blocked player-2 hands, asc
    const int32_t *blk1ptr, *blk1;  // per player-2 hand: blocked player-1 hands, asc
    const int32_t *aliveRows, *aliveRank, *prevAlive;
    const int32_t *sRank, *dOfS;   // d -> chain index (-1), chain -> d
    const int32_t *fcolOf, *dOfF;  // d -> local k of its F column (-1), F column -> d
    int nAlive, nS, nF;
    int64_t KS, SB, kpadLocal;     // S columns, S-slice positions, local positions
};

__device__ __forceinline__ bool compat(const BoardDev& B, int i, int j) {
    const int a0 = B.c1[2 * i], a1 = B.c1[2 * i + 1], b0 = B.c2[2 * j], b1 = B.c2[2 * j + 1];
    return a0 != b0 && a0 != b1 && a1 != b0 && a1 != b1;
}
__device__ __forceinline__ int wsign(const BoardDev& B, int i, int j) {
    if (!compat(B, i, j)) return 0;
    const uint32_t a = B.key1[i], b = B.key2[j];
    return a > b ? 1 : (a < b ? -1 : 0);
}
__device__ __forceinline__ int ydiff(const BoardDev& B, int i, int j) {
    return i == 0 ? wsign(B, 0, j) : wsign(B, i, j) - wsign(B, i - 1, j);
}
// local k -> local position (chain-sliced)
__device__ __forceinline__ int64_t kpos(const BoardDev& B, int64_t k) {
    if (k < B.KS) {
        const int64_t r = k / B.nS, c = k - r * B.nS;
        return (c / 32) * 32 * int64_t(B.nAlive) + 32 * r + (c % 32);
    }
    return B.SB + (k - B.KS);
}
// local position -> local k, or -1 for padding
__device__ __forceinline__ int64_t posk(const BoardDev& B, int64_t p) {
    if (p < B.SB) {
        const int64_t per = 32 * int64_t(B.nAlive);
        const int64_t s = p / per, rem = p - s * per, r = rem / 32, c = s * 32 + (rem % 32);
        return c < B.nS ? r * B.nS + c : -1;
    }
    const int64_t f = p - B.SB;
    return f < B.nF ? B.KS + f : -1;
}

// ---- row enumerators: emit(col, val) in storage order; return output row --
// V^T rows run chain-major (chain c, then its hands r): consecutive rows share
// the x' stripes of one sequence (as the host layout's outRow order does)
__device__ __forceinline__ int64_t vt_k(const BoardDev& B, int64_t rho) {
    if (rho < B.KS) {
        const int64_t c = rho / B.nAlive, r = rho - c * B.nAlive;
        return r * B.nS + c;
    }
    return rho;
}

template <class Emit>
__device__ void rows_vt(const BoardDev& B, int64_t rho, Emit& emit) {
    const int64_t k = vt_k(B, rho);
    if (k < B.KS) {
        const int r = int(k / B.nS), d = B.dOfS[k - int64_t(r) * B.nS];
        const int i = B.aliveRows[r];
        for (int j = 0; j < B.m2; ++j) {
            const double scale = B.l2[j] * double(ydiff(B, i, j));
            if (scale == 0.0) continue;
            for (int64_t e = B.sptr[d]; e < B.sptr[d + 1]; ++e) {
                const double v = scale * B.sval[e];
                if (v != 0.0) emit(int64_t(B.scol[e]) * B.M2 + B.hand2Off + j, v);
            }
        }
    } else {
        const int d = B.dOfF[k - B.KS];
        for (int j = 0; j < B.m2; ++j) {
            const double scale = B.l2[j];
            if (scale == 0.0) continue;
            for (int64_t e = B.fptr[d]; e < B.fptr[d + 1]; ++e) {
                const double v = scale * B.fval[e];
                if (v != 0.0) emit(int64_t(B.fcol[e]) * B.M2 + B.hand2Off + j, v);
            }
        }
    }
}

template <class Emit>
__device__ void rows_ua(const BoardDev& B, int64_t r, Emit& emit) {
    const int i = int(r / B.n1), a = int(r - int64_t(i) * B.n1);
    const double v = B.l1[i];
    if (v != 0.0) {
        if (B.sRank[a] >= 0 && B.prevAlive[i] >= 0)
            emit(B.kOff + kpos(B, int64_t(B.aliveRank[B.prevAlive[i]]) * B.nS + B.sRank[a]), v);
        if (B.fcolOf[a] >= 0) emit(B.kOff + kpos(B, B.fcolOf[a]), v);
    }
    for (int t = B.blk2ptr[i]; t < B.blk2ptr[i + 1]; ++t) {
        const int j = B.blk2[t];
        const double scale = -v * B.l2[j];
        for (int64_t e = B.fptr[a]; e < B.fptr[a + 1]; ++e) {
            const double w = scale * B.fval[e];
            if (w != 0.0) emit(B.kpadTotal + B.colOff + int64_t(j) * B.n2 + B.fcol[e], w);
        }
    }
}

template <class Emit>
__device__ void rows_ut(const BoardDev& B, int64_t p, Emit& emit) {
    const int64_t k = posk(B, p);
    if (k < 0) return;
    if (k < B.KS) {
        const int r = int(k / B.nS), d = B.dOfS[k - int64_t(r) * B.nS];
        const int i0 = B.aliveRows[r], i1 = r + 1 < B.nAlive ? B.aliveRows[r + 1] : B.m1;
        for (int i = i0; i < i1; ++i) {
            const double v = B.l1[i];
            if (v != 0.0) emit(B.rowOff + int64_t(i) * B.n1 + d, v);
        }
    } else {
        const int d = B.dOfF[k - B.KS];
        for (int i = 0; i < B.m1; ++i) {
            const double v = B.l1[i];
            if (v != 0.0) emit(B.rowOff + int64_t(i) * B.n1 + d, v);
        }
    }
}

template <class Emit>
__device__ void rows_av(const BoardDev& B, int64_t c, Emit& emit) {
    const int j = int(c / B.n2), b = int(c - int64_t(j) * B.n2);
    const double l2 = B.l2[j];
    for (int t = B.blk1ptr[j]; t < B.blk1ptr[j + 1]; ++t) {  // Ahat^T
        const int i = B.blk1[t];
        const double scale = -B.l1[i] * l2;
        for (int64_t e = B.fcptr[b]; e < B.fcptr[b + 1]; ++e) {
            const double w = scale * B.fcval[e];
            if (w != 0.0) emit(B.rowOff + int64_t(i) * B.n1 + B.fcrow[e], w);
        }
    }
    for (int r = 0; r < B.nAlive; ++r) {  // V, S columns: k = r nS + sRank(d) ascending
        const double scale = l2 * double(ydiff(B, B.aliveRows[r], j));
        if (scale == 0.0) continue;
        for (int64_t e = B.scptr[b]; e < B.scptr[b + 1]; ++e) {
            const int d = B.scrow[e];
            const double w = scale * B.scval[e];
            if (w != 0.0) emit(B.rowsTotal + B.kOff + kpos(B, int64_t(r) * B.nS + B.sRank[d]), w);
        }
    }
    if (l2 != 0.0)  // V, F columns
        for (int64_t e = B.fcptr[b]; e < B.fcptr[b + 1]; ++e) {
            const int d = B.fcrow[e];
            if (B.fcolOf[d] < 0) continue;
            const double w = l2 * B.fcval[e];
            if (w != 0.0) emit(B.rowsTotal + B.kOff + kpos(B, B.fcolOf[d]), w);
        }
}

struct Counter {
    int32_t n = 0;
    __device__ void operator()(int64_t, double) { ++n; }
};
struct Writer {
    int32_t* col;
    double* val;
    int64_t at, stride;
    __device__ void operator()(int64_t c, double v) {
        col[at] = int32_t(c);
        val[at] = v;
        at += stride;
    }
};

template <int W>
__device__ void rows_any(const BoardDev& B, int64_t r, Counter& e) {
    if (W == 0) rows_vt(B, r, e);
    else if (W == 1) rows_ua(B, r, e);
    else if (W == 2) rows_ut(B, r, e);
    else rows_av(B, r, e);
}
template <int W>
__device__ void rows_any(const BoardDev& B, int64_t r, Writer& e) {
    if (W == 0) rows_vt(B, r, e);
    else if (W == 1) rows_ua(B, r, e);
    else if (W == 2) rows_ut(B, r, e);
    else rows_av(B, r, e);
}

template <int W>
__global__ void k_len(BoardDev B, int64_t R, int32_t* len) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= R) return;
    Counter c;
    rows_any<W>(B, r, c);
    len[r] = c.n;
}

// Per window of kWin rows: the non-long rows sorted by (length desc, row asc)
// (std::stable_sort by length, as to_sell), their count, and the long rows in
// row order.  One block of kWin / 2 threads, bitonic sort in shared memory.
__global__ void __launch_bounds__(kWin / 2) k_window_sort(const int32_t* len, int64_t R, int longRow, int32_t* perm,
                                                          int32_t* wcount, int32_t* lcount) {
    __shared__ int64_t key[kWin];
    const int w = blockIdx.x;
    const int64_t r0 = int64_t(w) * kWin;
    const int n = int(lmin(kWin, R - r0));
    __shared__ int nl, nlong;
    if (threadIdx.x == 0) nl = nlong = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < kWin; q += blockDim.x) {
        int64_t k = INT64_MAX;  // empty / long rows sort last
        if (q < n) {
            const int L = len[r0 + q];
            if (L <= longRow) {
                k = (int64_t(longRow + 1 - L) << 20) | q;  // length desc, then row asc
                atomicAdd(&nl, 1);
            } else {
                atomicAdd(&nlong, 1);
            }
        }
        key[q] = k;
    }
    __syncthreads();
    for (int size = 2; size <= kWin; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < kWin / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const int64_t a = key[lo], b = key[hi];
                if ((a > b) == up) {
                    key[lo] = b;
                    key[hi] = a;
                }
            }
            __syncthreads();
        }
    for (int q = threadIdx.x; q < nl; q += blockDim.x) perm[r0 + q] = int32_t(key[q] & 0xFFFFF);
    if (threadIdx.x == 0) {
        wcount[w] = nl;
        lcount[w] = nlong;
    }
}

// Slot of each row: slice * 32 + lane for the sliced rows, -(long index + 1)
// for the long ones; lane_row / lane_len / slice widths alongside.
__global__ void k_slots(const int32_t* len, const int32_t* perm, const int32_t* wcount, const int64_t* wslice,
                        const int64_t* wlong, int64_t R, int longRow, int64_t rowBase, int64_t sliceBase,
                        int64_t longBase, int64_t* slot, int32_t* laneRow, int32_t* laneLen, int32_t* width,
                        int32_t* longRowOut, int32_t* longLen, const BoardDev* vtB) {
    // output row of local row r (V^T: its relabelled position)
    auto outRow = [&](int64_t r) { return int32_t(vtB ? vtB->kOff + kpos(*vtB, vt_k(*vtB, r)) : rowBase + r); };
    const int w = blockIdx.x;
    const int64_t r0 = int64_t(w) * kWin;
    const int n = int(lmin(kWin, R - r0));
    const int nl = wcount[w];
    for (int q = threadIdx.x; q < nl; q += blockDim.x) {
        const int64_t r = r0 + perm[r0 + q];
        const int64_t s = wslice[w] + q / 32;
        slot[r] = (sliceBase + s) * 32 + (q % 32);
        laneRow[(sliceBase + s) * 32 + (q % 32)] = outRow(r);
        laneLen[(sliceBase + s) * 32 + (q % 32)] = len[r];
        if (q % 32 == 0) width[s] = len[r];
    }
    if (threadIdx.x == 0) {  // long rows in row order
        int64_t li = wlong[w];
        for (int q = 0; q < n; ++q)
            if (len[r0 + q] > longRow) {
                slot[r0 + q] = -(longBase + li + 1);
                longRowOut[longBase + li] = outRow(r0 + q);
                longLen[li] = len[r0 + q];
                ++li;
            }
    }
}

template <int W>
__global__ void k_fill(BoardDev B, int64_t R, const int64_t* slot, const int64_t* slicePtr, const int64_t* longPtr,
                       int32_t* col, double* val, int32_t* lcol, double* lval) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const int64_t sl = slot[r];
    Writer wr;
    if (sl >= 0) {
        wr = Writer{col, val, slicePtr[sl / 32] + (sl % 32), 32};
    } else {
        wr = Writer{lcol, lval, longPtr[-sl - 1], 1};
    }
    rows_any<W>(B, r, wr);
}

template <class T>
T* upv(std::vector<void*>& keep, const std::vector<T>& v) {
    T* p = dev_alloc<T>(std::max<int64_t>(int64_t(v.size()), 1));
    keep.push_back(p);
    if (!v.empty()) KR_CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return p;
}
template <class T>
std::vector<T> down(const T* d, int64_t n) {
    std::vector<T> h(static_cast<size_t>(std::max<int64_t>(n, 0)));
    if (n > 0) KR_CK(cudaMemcpy(h.data(), d, sizeof(T) * size_t(n), cudaMemcpyDeviceToHost));
    return h;
}

__global__ void k_row_alive_dev(BoardDev B, uint8_t* alive) {
    const int i = blockIdx.x;
    int any = 0;
    for (int j = threadIdx.x; j < B.m2; j += blockDim.x)
        if (B.l2[j] * double(ydiff(B, i, j)) != 0.0) any = 1;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) alive[i] = uint8_t(any);
}

void csc_of(const kr_compressed& A, int rows, int cols, std::vector<int64_t>& ptr, std::vector<int32_t>& idx,
            std::vector<double>& val) {
    ptr.assign(size_t(cols) + 1, 0);
    for (int64_t e = 0; e < A.outer[rows]; ++e) ptr[size_t(A.inner[e]) + 1]++;
    for (int c = 0; c < cols; ++c) ptr[size_t(c) + 1] += ptr[size_t(c)];
    idx.resize(size_t(ptr.back()));
    val.resize(size_t(ptr.back()));
    std::vector<int64_t> pos(ptr.begin(), ptr.end() - 1);
    for (int r = 0; r < rows; ++r)
        for (int64_t e = A.outer[r]; e < A.outer[r + 1]; ++e) {
            const int64_t q = pos[size_t(A.inner[e])]++;
            idx[size_t(q)] = r;
            val[size_t(q)] = A.val[e];
        }
}

// blocked lists: for each hand of `a`, the hands of `b` sharing a card, asc
void blocked_lists(const uint8_t* ca, int ma, const uint8_t* cb, int mb, std::vector<int32_t>& ptr,
                   std::vector<int32_t>& out) {
    std::vector<std::vector<int32_t>> byCard(52);
    for (int j = 0; j < mb; ++j) {
        byCard[cb[2 * j]].push_back(j);
        byCard[cb[2 * j + 1]].push_back(j);
    }
    ptr.assign(1, 0);
    out.clear();
    std::vector<int32_t> tmp;
    for (int i = 0; i < ma; ++i) {
        const auto& x = byCard[ca[2 * i]];
        const auto& y = byCard[ca[2 * i + 1]];
        tmp.clear();
        std::set_union(x.begin(), x.end(), y.begin(), y.end(), std::back_inserter(tmp));
        out.insert(out.end(), tmp.begin(), tmp.end());
        ptr.push_back(int32_t(out.size()));
    }
}

struct BoardHost {
    BoardDev dev{};
    int64_t R[4] = {0, 0, 0, 0};
    int32_t* len[4] = {nullptr, nullptr, nullptr, nullptr};
    int32_t* perm[4] = {nullptr, nullptr, nullptr, nullptr};
    int32_t* wcount[4] = {nullptr, nullptr, nullptr, nullptr};
    int32_t* lcount[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<int64_t> wslice[4], wlong[4];
    std::vector<int32_t> hlen[4];  // row lengths (host copy)
    int64_t slices[4] = {0, 0, 0, 0}, nlong[4] = {0, 0, 0, 0};
    int64_t slOff[4] = {0, 0, 0, 0}, nlOff[4] = {0, 0, 0, 0};
    int64_t nnz[4] = {0, 0, 0, 0};
    int32_t maxLen[4] = {0, 0, 0, 0};
    int64_t K = 0, nnzM = 0;
    int nAlive = 0, nS = 0, nF = 0;
};

}  // namespace

kr_engine* create_engine_device_b(const kr_kron_board* boards, int nb, int device, uint32_t flags) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Fail{KR_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    }
    if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
    if (!boards || nb < 1) throw Fail{KR_INVALID_INPUT, "at least one board is required"};
    KR_CK(cudaSetDevice(device));
    const int n1 = boards[0].n1, n2 = boards[0].n2;
    int longRow = kLongRow;
    if (const char* env = std::getenv("KR_LONG_ROW")) longRow = std::max(8, std::atoi(env));
    std::vector<void*> keep;  // per-board device tables, freed at the end
    std::vector<BoardHost> bh(static_cast<size_t>(nb));
    int64_t rowsTotal = 0, colsTotal = 0, hands2 = 0, kpadTotal = 0, kTotal = 0;
    // pass 0: per-board tables, alive rows, chain bookkeeping
    for (int b = 0; b < nb; ++b) {
        const kr_kron_board& K = boards[b];
        if (K.n1 != n1 || K.n2 != n2) throw Fail{KR_INVALID_INPUT, "boards must share one betting tree"};
        if (K.m1 < 1 || K.m2 < 1 || K.F.outer_size != n1 || K.S.outer_size != n1)
            throw Fail{KR_INVALID_INPUT, "bad board"};
        BoardDev& B = bh[size_t(b)].dev;
        B.m1 = K.m1;
        B.m2 = K.m2;
        B.n1 = n1;
        B.n2 = n2;
        B.key1 = upv(keep, std::vector<uint32_t>(K.key1, K.key1 + K.m1));
        B.key2 = upv(keep, std::vector<uint32_t>(K.key2, K.key2 + K.m2));
        B.c1 = upv(keep, std::vector<uint8_t>(K.cards1, K.cards1 + 2 * K.m1));
        B.c2 = upv(keep, std::vector<uint8_t>(K.cards2, K.cards2 + 2 * K.m2));
        B.l1 = upv(keep, std::vector<double>(K.lambda1, K.lambda1 + K.m1));
        B.l2 = upv(keep, std::vector<double>(K.lambda2, K.lambda2 + K.m2));
        const int64_t nF = K.F.outer[n1], nSn = K.S.outer[n1];
        B.fptr = upv(keep, std::vector<int64_t>(K.F.outer, K.F.outer + n1 + 1));
        B.fcol = upv(keep, std::vector<int32_t>(K.F.inner, K.F.inner + nF));
        B.fval = upv(keep, std::vector<double>(K.F.val, K.F.val + nF));
        B.sptr = upv(keep, std::vector<int64_t>(K.S.outer, K.S.outer + n1 + 1));
        B.scol = upv(keep, std::vector<int32_t>(K.S.inner, K.S.inner + nSn));
        B.sval = upv(keep, std::vector<double>(K.S.val, K.S.val + nSn));
        std::vector<int64_t> cp;
        std::vector<int32_t> ci;
        std::vector<double> cv;
        csc_of(K.F, n1, n2, cp, ci, cv);
        B.fcptr = upv(keep, cp);
        B.fcrow = upv(keep, ci);
        B.fcval = upv(keep, cv);
        csc_of(K.S, n1, n2, cp, ci, cv);
        B.scptr = upv(keep, cp);
        B.scrow = upv(keep, ci);
        B.scval = upv(keep, cv);
        std::vector<int32_t> bp, bl;
        blocked_lists(K.cards1, K.m1, K.cards2, K.m2, bp, bl);
        B.blk2ptr = upv(keep, bp);
        B.blk2 = upv(keep, bl);
        blocked_lists(K.cards2, K.m2, K.cards1, K.m1, bp, bl);
        B.blk1ptr = upv(keep, bp);
        B.blk1 = upv(keep, bl);
        uint8_t* dAlive = dev_alloc<uint8_t>(K.m1);
        keep.push_back(dAlive);
        k_row_alive_dev<<<unsigned(K.m1), 256>>>(B, dAlive);
        KR_CK_LAUNCH();
        const auto alive = down(dAlive, K.m1);
        std::vector<int32_t> aliveRows, aliveRank(size_t(K.m1), -1), prevAlive(size_t(K.m1), -1);
        for (int i = 0; i < K.m1; ++i) {
            if (alive[size_t(i)]) {
                aliveRank[size_t(i)] = int32_t(aliveRows.size());
                aliveRows.push_back(i);
            }
            prevAlive[size_t(i)] = alive[size_t(i)] ? i : (i ? prevAlive[size_t(i) - 1] : -1);
        }
        std::vector<int32_t> sRank(size_t(n1), -1), dOfS, fcolOf(size_t(n1), -1), dOfF;
        for (int d = 0; d < n1; ++d)
            if (K.S.outer[d + 1] > K.S.outer[d]) {
                sRank[size_t(d)] = int32_t(dOfS.size());
                dOfS.push_back(d);
            }
        bool anyL2 = false;
        for (int j = 0; j < K.m2; ++j) anyL2 |= K.lambda2[j] != 0.0;
        B.nAlive = int(aliveRows.size());
        B.nS = int(dOfS.size());
        B.KS = int64_t(B.nAlive) * B.nS;
        for (int d = 0; d < n1; ++d)
            if (K.F.outer[d + 1] > K.F.outer[d] && anyL2) {
                fcolOf[size_t(d)] = int32_t(B.KS + int64_t(dOfF.size()));
                dOfF.push_back(d);
            }
        B.nF = int(dOfF.size());
        B.SB = int64_t((B.nS + 31) / 32) * 32 * B.nAlive;
        B.kpadLocal = B.SB + int64_t((B.nF + 31) / 32) * 32;
        B.aliveRows = upv(keep, aliveRows);
        B.aliveRank = upv(keep, aliveRank);
        B.prevAlive = upv(keep, prevAlive);
        B.sRank = upv(keep, sRank);
        B.dOfS = upv(keep, dOfS);
        B.fcolOf = upv(keep, fcolOf);
        B.dOfF = upv(keep, dOfF);
        B.rowOff = rowsTotal;
        B.colOff = colsTotal;
        B.hand2Off = hands2;
        B.kOff = kpadTotal;
        rowsTotal += int64_t(K.m1) * n1;
        colsTotal += int64_t(K.m2) * n2;
        hands2 += K.m2;
        kpadTotal += B.kpadLocal;
        BoardHost& H = bh[size_t(b)];
        H.K = B.KS + B.nF;
        H.nnzM = H.K + (B.nAlive > 0 ? int64_t(B.nAlive - 1) * B.nS : 0);
        H.nAlive = B.nAlive;
        H.nS = B.nS;
        H.nF = B.nF;
        kTotal += H.K;
    }
    if (rowsTotal + kpadTotal > INT32_MAX || colsTotal + kpadTotal > INT32_MAX)
        throw Fail{KR_INVALID_INPUT, "dimensions exceed 32-bit indices"};
    for (auto& H : bh) {
        H.dev.rowsTotal = rowsTotal;
        H.dev.kpadTotal = kpadTotal;
        H.dev.M2 = hands2;
    }
    kr_engine* e = new kr_engine();
    try {
        e->device = device;
        KR_CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->rows = rowsTotal;
        e->cols = colsTotal;
        e->k = kTotal;
        e->n1 = n1;
        e->n2 = n2;
        e->xseq = true;
        e->M2 = hands2;
        e->mkind = 1;
        e->kpad = kpadTotal;
        // pass 1: lengths, window sorts, sizes
        DevSell* mats[4] = {&e->VT, &e->UA, &e->UT, &e->AV};
        int64_t tsl[4] = {0, 0, 0, 0}, tnl[4] = {0, 0, 0, 0}, tnnz[4] = {0, 0, 0, 0};
        for (int b = 0; b < nb; ++b) {
            BoardHost& H = bh[size_t(b)];
            const BoardDev& B = H.dev;
            const int64_t Rs[4] = {B.KS + B.nF, int64_t(B.m1) * n1, B.kpadLocal, int64_t(B.m2) * n2};
            for (int w = 0; w < 4; ++w) {
                const int64_t R = Rs[w];
                H.R[w] = R;
                H.len[w] = dev_alloc<int32_t>(std::max<int64_t>(R, 1));
                H.perm[w] = dev_alloc<int32_t>(std::max<int64_t>(R, 1));
                keep.push_back(H.len[w]);
                keep.push_back(H.perm[w]);
                const int64_t nw = (R + kWin - 1) / kWin;
                H.wcount[w] = dev_alloc<int32_t>(std::max<int64_t>(nw, 1));
                H.lcount[w] = dev_alloc<int32_t>(std::max<int64_t>(nw, 1));
                keep.push_back(H.wcount[w]);
                keep.push_back(H.lcount[w]);
                if (R == 0) continue;
                const unsigned g = unsigned((R + 127) / 128);
                if (w == 0) k_len<0><<<g, 128>>>(B, R, H.len[w]);
                else if (w == 1) k_len<1><<<g, 128>>>(B, R, H.len[w]);
                else if (w == 2) k_len<2><<<g, 128>>>(B, R, H.len[w]);
                else k_len<3><<<g, 128>>>(B, R, H.len[w]);
                KR_CK_LAUNCH();
                H.hlen[w] = down(H.len[w], R);
            }
        }
        // the long-row threshold per matrix, as the host-built engine picks it
        // (kr_engine.cu): the smallest of 16 .. kLongRow whose long rows over
        // all boards number at most kLongRowBudget (KR_LONG_ROW: fixed)
        int longRowW[4] = {longRow, longRow, longRow, longRow};
        if (!std::getenv("KR_LONG_ROW")) {
            const int thr[5] = {16, 32, 64, 128, kLongRow};
            for (int w = 0; w < 4; ++w)
                for (int t : thr) {
                    int64_t n = 0;
                    for (int b = 0; b < nb; ++b)
                        for (int32_t v : bh[size_t(b)].hlen[w]) n += v > t;
                    if (n <= kLongRowBudget) {
                        longRowW[w] = t;
                        break;
                    }
                }
        }
        for (int b = 0; b < nb; ++b) {
            BoardHost& H = bh[size_t(b)];
            for (int w = 0; w < 4; ++w) {
                const int64_t R = H.R[w];
                const int longRow = longRowW[w];
                const int64_t nw = (R + kWin - 1) / kWin;
                if (R == 0) continue;
                k_window_sort<<<unsigned(nw), kWin / 2>>>(H.len[w], R, longRow, H.perm[w], H.wcount[w], H.lcount[w]);
                KR_CK_LAUNCH();
                const auto wc = down(H.wcount[w], nw), lc = down(H.lcount[w], nw);
                H.wslice[w].assign(size_t(nw) + 1, 0);
                H.wlong[w].assign(size_t(nw) + 1, 0);
                for (int64_t q = 0; q < nw; ++q) {
                    H.wslice[w][size_t(q) + 1] = H.wslice[w][size_t(q)] + (wc[size_t(q)] + 31) / 32;
                    H.wlong[w][size_t(q) + 1] = H.wlong[w][size_t(q)] + lc[size_t(q)];
                }
                H.slices[w] = H.wslice[w].back();
                H.nlong[w] = H.wlong[w].back();
                for (int32_t v : H.hlen[w]) {
                    H.nnz[w] += v;
                    if (v <= longRow) H.maxLen[w] = std::max(H.maxLen[w], v);
                }
                std::vector<int32_t>().swap(H.hlen[w]);
            }
            for (int w = 0; w < 4; ++w) {
                H.slOff[w] = tsl[w];
                H.nlOff[w] = tnl[w];
                tsl[w] += H.slices[w];
                tnl[w] += H.nlong[w];
                tnnz[w] += H.nnz[w];
            }
        }
        // pass 2: slots, slice widths -> pointers, allocation, fill
        std::vector<int64_t> padded(4, 0);
        std::vector<std::vector<int64_t>> slicePtrH(4), longPtrH(4);
        std::vector<int64_t*> dSlot(size_t(nb) * 4, nullptr);
        for (int w = 0; w < 4; ++w) {
            DevSell& S = *mats[w];
            S.nrows = w == 0 || w == 2 ? kpadTotal : (w == 1 ? rowsTotal : colsTotal);
            S.nslices = tsl[w];
            S.nlong = tnl[w];
            S.lane_row = dev_alloc<int32_t>(std::max<int64_t>(32 * tsl[w], 1));
            S.lane_len = dev_alloc<int32_t>(std::max<int64_t>(32 * tsl[w], 1));
            KR_CK(cudaMemset(S.lane_row, 0xFF, 4 * size_t(std::max<int64_t>(32 * tsl[w], 1))));
            KR_CK(cudaMemset(S.lane_len, 0, 4 * size_t(std::max<int64_t>(32 * tsl[w], 1))));
            S.long_row = dev_alloc<int32_t>(std::max<int64_t>(tnl[w], 1));
            std::vector<int32_t> widths;
            std::vector<int32_t> llens;
            for (int b = 0; b < nb; ++b) {
                BoardHost& H = bh[size_t(b)];
                const int64_t R = H.R[w];
                int64_t* slot = dev_alloc<int64_t>(std::max<int64_t>(R, 1));
                dSlot[size_t(b) * 4 + w] = slot;
                keep.push_back(slot);
                int32_t* wd = dev_alloc<int32_t>(std::max<int64_t>(H.slices[w], 1));
                int32_t* ll = dev_alloc<int32_t>(std::max<int64_t>(H.nlong[w], 1));
                keep.push_back(wd);
                keep.push_back(ll);
                if (R) {
                    const int64_t nw = (R + kWin - 1) / kWin;
                    int64_t* dws = upv(keep, H.wslice[w]);
                    int64_t* dwl = upv(keep, H.wlong[w]);
                    BoardDev* vtB = nullptr;
                    if (w == 0) {
                        vtB = dev_alloc<BoardDev>(1);
                        keep.push_back(vtB);
                        KR_CK(cudaMemcpy(vtB, &H.dev, sizeof(BoardDev), cudaMemcpyHostToDevice));
                    }
                    k_slots<<<unsigned(nw), 256>>>(H.len[w], H.perm[w], H.wcount[w], dws, dwl, R, longRowW[w],
                                                  w == 1 ? H.dev.rowOff : (w == 3 ? H.dev.colOff : H.dev.kOff),
                                                  H.slOff[w], H.nlOff[w], slot, S.lane_row, S.lane_len, wd,
                                                  S.long_row, ll, vtB);
                    KR_CK_LAUNCH();
                }
                const auto wv = down(wd, H.slices[w]);
                widths.insert(widths.end(), wv.begin(), wv.end());
                const auto lv = down(ll, H.nlong[w]);
                llens.insert(llens.end(), lv.begin(), lv.end());
            }
            auto& sp = slicePtrH[w];
            sp.assign(1, 0);
            for (int32_t x : widths) sp.push_back(sp.back() + 32 * int64_t(x));
            padded[size_t(w)] = sp.back();
            auto& lp = longPtrH[w];
            lp.assign(1, 0);
            for (int32_t x : llens) lp.push_back(lp.back() + x);
            S.padded = sp.back();
            S.nnz = tnnz[w];
            S.nnzLong = lp.back();
            S.slice_ptr = dev_alloc<int64_t>(int64_t(sp.size()));
            KR_CK(cudaMemcpy(S.slice_ptr, sp.data(), 8 * sp.size(), cudaMemcpyHostToDevice));
            S.long_ptr = dev_alloc<int64_t>(int64_t(lp.size()));
            KR_CK(cudaMemcpy(S.long_ptr, lp.data(), 8 * lp.size(), cudaMemcpyHostToDevice));
            S.col = dev_alloc<int32_t>(std::max<int64_t>(S.padded, 1));
            S.val = dev_alloc<double>(std::max<int64_t>(S.padded, 1));
            KR_CK(cudaMemset(S.col, 0, 4 * size_t(std::max<int64_t>(S.padded, 1))));
            KR_CK(cudaMemset(S.val, 0, 8 * size_t(std::max<int64_t>(S.padded, 1))));
            S.long_col = dev_alloc<int32_t>(std::max<int64_t>(S.nnzLong, 1));
            S.long_val = dev_alloc<double>(std::max<int64_t>(S.nnzLong, 1));
            for (int b = 0; b < nb; ++b) {
                BoardHost& H = bh[size_t(b)];
                const int64_t R = H.R[w];
                if (!R) continue;
                const unsigned g = unsigned((R + 127) / 128);
                int64_t* slot = dSlot[size_t(b) * 4 + w];
                if (w == 0) k_fill<0><<<g, 128>>>(H.dev, R, slot, S.slice_ptr, S.long_ptr, S.col, S.val, S.long_col, S.long_val);
                else if (w == 1) k_fill<1><<<g, 128>>>(H.dev, R, slot, S.slice_ptr, S.long_ptr, S.col, S.val, S.long_col, S.long_val);
                else if (w == 2) k_fill<2><<<g, 128>>>(H.dev, R, slot, S.slice_ptr, S.long_ptr, S.col, S.val, S.long_col, S.long_val);
                else k_fill<3><<<g, 128>>>(H.dev, R, slot, S.slice_ptr, S.long_ptr, S.col, S.val, S.long_col, S.long_val);
                KR_CK_LAUNCH();
            }
            for (auto& H : bh) S.maxLen = std::max(S.maxLen, H.maxLen[w]);
            for (int b = 0; b < nb; ++b) {
                e->bSl[w].push_back(bh[size_t(b)].slOff[w]);
                e->bNl[w].push_back(bh[size_t(b)].nlOff[w]);
            }
            e->bSl[w].push_back(tsl[w]);
            e->bNl[w].push_back(tnl[w]);
        }
        // factor nnz (the reference's flop rule): U, Ahat, V from the rows, M from the chains
        {
            int64_t nU = 0, nM = 0;
            for (auto& H : bh) nM += H.nnzM;
            nU = tnnz[2];                       // U^T rows hold every U entry
            const int64_t nV = tnnz[0];         // V^T rows hold every V entry
            const int64_t nA = tnnz[1] - nU;    // UA = U + Ahat
            e->nnzA = nA;
            e->nnzU = nU;
            e->nnzV = nV;
            e->nnzM = nM;
            e->flops_per_product = nV + nU + nA + (nM - kTotal);
        }
        // chains: S slices (32 chains, nAlive long), then F singletons
        {
            std::vector<int64_t> sbase;
            std::vector<int32_t> slen;
            e->bCh.assign(1, 0);
            for (auto& H : bh) {
                const BoardDev& B = H.dev;
                for (int s = 0; s < (B.nS + 31) / 32; ++s) {
                    sbase.push_back(B.kOff + int64_t(s) * 32 * B.nAlive);
                    for (int l = 0; l < 32; ++l) slen.push_back(s * 32 + l < B.nS ? B.nAlive : 0);
                }
                for (int s = 0; s < (B.nF + 31) / 32; ++s) {
                    sbase.push_back(B.kOff + B.SB + int64_t(s) * 32);
                    for (int l = 0; l < 32; ++l) slen.push_back(s * 32 + l < B.nF ? 1 : 0);
                }
                e->bCh.push_back(int64_t(sbase.size()));
            }
            e->nchains = int64_t(sbase.size());
            sbase.push_back(kpadTotal);
            e->chain_withmul = 0;
            if (const char* env = std::getenv("KR_CHAIN")) e->chain_tma = std::string(env) != "reg";
            e->chain_ptr = dev_alloc<int64_t>(int64_t(sbase.size()));
            KR_CK(cudaMemcpy(e->chain_ptr, sbase.data(), 8 * sbase.size(), cudaMemcpyHostToDevice));
            e->chain_len = dev_alloc<int32_t>(std::max<int64_t>(int64_t(slen.size()), 1));
            if (!slen.empty()) KR_CK(cudaMemcpy(e->chain_len, slen.data(), 4 * slen.size(), cudaMemcpyHostToDevice));
            const std::vector<uint8_t> neg(slen.size(), 1);
            e->chain_neg1 = dev_alloc<uint8_t>(std::max<int64_t>(int64_t(neg.size()), 1));
            if (!neg.empty()) KR_CK(cudaMemcpy(e->chain_neg1, neg.data(), neg.size(), cudaMemcpyHostToDevice));
            e->chain_mul = dev_alloc<double>(std::max<int64_t>(kpadTotal, 1));
            KR_CK(cudaMemset(e->chain_mul, 0, 8 * size_t(std::max<int64_t>(kpadTotal, 1))));
            engine_chain_setup(e);
        }
        e->d_tz = dev_alloc<double>(std::max<int64_t>(kpadTotal, 1));
        KR_CK(cudaMemset(e->d_tz, 0, 8 * size_t(std::max<int64_t>(kpadTotal, 1))));
        e->d_tz2 = dev_alloc<double>(std::max<int64_t>(kpadTotal, 1));
        KR_CK(cudaMemset(e->d_tz2, 0, 8 * size_t(std::max<int64_t>(kpadTotal, 1))));
        e->d_xp = dev_alloc<double>(std::max<int64_t>(colsTotal, 1));
        e->d_in = dev_alloc<double>(std::max<int64_t>(std::max(rowsTotal, colsTotal), 1));
        e->d_out = dev_alloc<double>(std::max<int64_t>(std::max(rowsTotal, colsTotal), 1));
        e->lean = std::getenv("KR_NO_LEAN") == nullptr;
        // board groups for the host-buffer pipeline
        for (int g1 : group_ends(nb, flags)) {
            e->grpBoard.push_back(g1);
            e->grpRow.push_back(g1 < nb ? bh[size_t(g1)].dev.rowOff : rowsTotal);
            e->grpCol.push_back(g1 < nb ? bh[size_t(g1)].dev.colOff : colsTotal);
        }
        if (const char* env = std::getenv("KR_PF")) e->pf = std::max(0, std::atoi(env));
        engine_make_pipeline(e);
        KR_CK(cudaDeviceSynchronize());
    } catch (...) {
        for (void* p : keep) krb::dev_free(p);
        kr_engine_destroy(e);
        throw;
    }
    for (void* p : keep) krb::dev_free(p);
    return e;
}

}  // namespace krb

extern "C" int kr_engine_create_device_b(const kr_kron_board* boards, int nboards, int device, uint32_t flags,
                                         kr_engine** out) {
    return krb::guarded([&] {
        if (!out) throw krb::Fail{KR_INVALID_INPUT, "null output handle"};
        *out = krb::create_engine_device_b(boards, nboards, device, flags);
    });
}
