// kr_factors_dev.cu — Technique B with postprocessing built on the device
// (SURVEY.md §8(f) row 3): the factors of sparsify.hpp:246-406 for one board,
// from the KronPayoff pieces (strength keys, hand cards, lambda, F, S), in the
// reference's storage order and bit-exact against the host builder
// (techniqueBPost in csrc/host/kr_host.cpp, itself bit-exact against
// postprocess(techniqueB(...)) of the oracle).
//
// Every entry of every factor is a closed-form product:
//   Ahat (i,a | j,b)  = (-lambda1_i * lambda2_j) * F_ab        j blocked by i
//   U    (i,d | c)    = lambda1_i                              c = last kept column of chain d
//   M                 = unit diagonal, -1 to the next kept column of a chain
//   V    (j,b | (i,d))= (lambda2_j * Y_ij) * S_db,  Y_ij = W_ij - W_{i-1,j}
//   V    (j,b | f(d)) = lambda2_j * F_db
// and it exists iff its value is nonzero (the host ColBuilder, like makeSparse,
// prunes exact zeros, linalg.hpp:18-25).  So each matrix is built in two
// passes — count the nonzero values per row / column, prefix-sum, fill —
// with the value recomputed identically in both.  The prefix sums and the
// per-hand chain bookkeeping (a few thousand integers) run on the host.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>
#include <vector>

#include "kr_common.cuh"

// Host copies in pinned memory (fast downloads), ahat / u / m / v.
template <class T>
struct Pinned {
    T* p = nullptr;
    int64_t n = 0;
    Pinned() = default;
    Pinned(const Pinned&) = delete;
    Pinned& operator=(const Pinned&) = delete;
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
    void alloc(int64_t count) {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = count;
        if (cudaMallocHost(&p, sizeof(T) * size_t(std::max<int64_t>(count, 1))) != cudaSuccess) {
            cudaGetLastError();
            throw krb::Fail{KR_CUDA, "cudaMallocHost failed"};
        }
    }
    T* data() const { return p; }
};

struct kr_devfactors {
    int64_t rows = 0, cols = 0, k = 0;
    int32_t n1 = 0, n2 = 0;
    Pinned<int64_t> outer[4];
    Pinned<int32_t> inner[4];
    Pinned<double> val[4];
    double seconds = 0;
};

namespace krb {
namespace {

struct Pieces {
    int m1, m2, n1, n2;
    const uint32_t* key1;
    const uint32_t* key2;
    const uint8_t* c1;
    const uint8_t* c2;
    const double* l1;
    const double* l2;
    const int64_t* fptr;  // F CSR (n1 x n2)
    const int32_t* fcol;
    const double* fval;
    const int64_t* sptr;  // S CSR
    const int32_t* scol;
    const double* sval;
};

__device__ __forceinline__ bool compat(const Pieces& P, int i, int j) {
    const int a0 = P.c1[2 * i], a1 = P.c1[2 * i + 1], b0 = P.c2[2 * j], b1 = P.c2[2 * j + 1];
    return a0 != b0 && a0 != b1 && a1 != b0 && a1 != b1;
}

// gamma(h1_i, h2_j) for compatible pairs, 0 otherwise (kron.hpp:152-157)
__device__ __forceinline__ int wsign(const Pieces& P, int i, int j) {
    if (!compat(P, i, j)) return 0;
    const uint32_t a = P.key1[i], b = P.key2[j];
    return a > b ? 1 : (a < b ? -1 : 0);
}

// Y_ij = W_ij - W_{i-1,j} (sparsify.hpp:251-254)
__device__ __forceinline__ int ydiff(const Pieces& P, int i, int j) {
    return i == 0 ? wsign(P, 0, j) : wsign(P, i, j) - wsign(P, i - 1, j);
}

// Block-wide ordered list of the j in [0, m2) with pred(j), into smem list;
// returns the count.  256 threads.
template <class Pred>
__device__ int block_list(int m2, Pred pred, int* list, int* warpCnt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int total = 0;
    for (int j0 = 0; j0 < m2; j0 += blockDim.x) {
        const int j = j0 + int(threadIdx.x);
        const bool f = j < m2 && pred(j);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) warpCnt[warp] = __popc(bal);
        __syncthreads();
        int before = total;
        for (int w = 0; w < warp; ++w) before += warpCnt[w];
        if (f) list[before + __popc(bal & ((1u << lane) - 1))] = j;
        int add = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) add += warpCnt[w];
        __syncthreads();
        total += add;
    }
    return total;
}

// rowAlive[i]: some j with lambda2_j * Y_ij != 0 (techniqueBPost).
__global__ void k_row_alive(Pieces P, uint8_t* alive) {
    const int i = blockIdx.x;
    int any = 0;
    for (int j = threadIdx.x; j < P.m2; j += blockDim.x)
        if (P.l2[j] * double(ydiff(P, i, j)) != 0.0) any = 1;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) alive[i] = uint8_t(any);
}

// Ahat rows (i, a): blocked j ascending, F row a's entries ascending.
// count: cnt[i*n1 + a]; fill: writes at ptr[i*n1 + a].
template <bool FILL>
__global__ void k_ahat(Pieces P, int64_t* cnt, const int64_t* ptr, int32_t* inner, double* val) {
    extern __shared__ int list[];
    __shared__ int warpCnt[8];
    const int i = blockIdx.x;
    const int nb = block_list(P.m2, [&](int j) { return !compat(P, i, j); }, list, warpCnt);
    const double li = P.l1[i];
    for (int a = threadIdx.x; a < P.n1; a += blockDim.x) {
        int64_t q = FILL ? ptr[int64_t(i) * P.n1 + a] : 0;
        int64_t c = 0;
        for (int t = 0; t < nb; ++t) {
            const int j = list[t];
            const double scale = -li * P.l2[j];
            for (int64_t e = P.fptr[a]; e < P.fptr[a + 1]; ++e) {
                const double v = scale * P.fval[e];
                if (v != 0.0) {
                    if (FILL) {
                        inner[q] = int32_t(int64_t(j) * P.n2 + P.fcol[e]);
                        val[q] = v;
                        ++q;
                    } else {
                        ++c;
                    }
                }
            }
        }
        if (!FILL) cnt[int64_t(i) * P.n1 + a] = c;
    }
}

// V's S-part columns (i, d) for an alive i: J_i = {j : lambda2_j * Y_ij != 0}
// ascending, S row d's entries ascending.  Column index col(i, d) given.
template <bool FILL>
__global__ void k_vs(Pieces P, const int32_t* aliveRows, const int32_t* sRank, int nS, int64_t* cnt,
                     const int64_t* ptr, int32_t* inner, double* val) {
    extern __shared__ int list[];
    __shared__ int warpCnt[8];
    const int r = blockIdx.x;          // alive rank
    const int i = aliveRows[r];
    const int nj = block_list(P.m2, [&](int j) { return P.l2[j] * double(ydiff(P, i, j)) != 0.0; }, list, warpCnt);
    for (int d = threadIdx.x; d < P.n1; d += blockDim.x) {
        if (sRank[d] < 0) continue;
        const int64_t col = int64_t(r) * nS + sRank[d];
        int64_t q = FILL ? ptr[col] : 0;
        int64_t c = 0;
        for (int t = 0; t < nj; ++t) {
            const int j = list[t];
            const double scale = P.l2[j] * double(ydiff(P, i, j));
            for (int64_t e = P.sptr[d]; e < P.sptr[d + 1]; ++e) {
                const double v = scale * P.sval[e];
                if (v != 0.0) {
                    if (FILL) {
                        inner[q] = int32_t(int64_t(j) * P.n2 + P.scol[e]);
                        val[q] = v;
                        ++q;
                    } else {
                        ++c;
                    }
                }
            }
        }
        if (!FILL) cnt[col] = c;
    }
}

// V's F-part column f(d): j with lambda2_j != 0 ascending, F row d ascending.
template <bool FILL>
__global__ void k_vf(Pieces P, const int32_t* fCols /* d of each F column */, int64_t colBase, int64_t* cnt,
                     const int64_t* ptr, int32_t* inner, double* val) {
    const int f = blockIdx.x;
    const int d = fCols[f];
    const int64_t col = colBase + f;
    if (threadIdx.x != 0) return;
    int64_t q = FILL ? ptr[col] : 0;
    int64_t c = 0;
    for (int j = 0; j < P.m2; ++j) {
        const double scale = P.l2[j];
        if (scale == 0.0) continue;
        for (int64_t e = P.fptr[d]; e < P.fptr[d + 1]; ++e) {
            const double v = scale * P.fval[e];
            if (v != 0.0) {
                if (FILL) {
                    inner[q] = int32_t(int64_t(j) * P.n2 + P.fcol[e]);
                    val[q] = v;
                    ++q;
                } else {
                    ++c;
                }
            }
        }
    }
    if (!FILL) cnt[col] = c;
}

// U rows (i, d): [last kept column of chain d at or above i] [f(d)], value lambda1_i.
template <bool FILL>
__global__ void k_u(int m1, int n1, const double* l1, const int32_t* lastKept /* m1*n1 */,
                    const int32_t* fcolOf /* n1 */, int64_t* cnt, const int64_t* ptr, int32_t* inner, double* val) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= int64_t(m1) * n1) return;
    const int i = int(r / n1), d = int(r - int64_t(i) * n1);
    const double v = l1[i];
    int64_t q = FILL ? ptr[r] : 0;
    int c = 0;
    if (v != 0.0) {
        if (lastKept[r] >= 0) {
            if (FILL) {
                inner[q] = lastKept[r];
                val[q] = v;
                ++q;
            }
            ++c;
        }
        if (fcolOf[d] >= 0) {
            if (FILL) {
                inner[q] = fcolOf[d];
                val[q] = v;
                ++q;
            }
            ++c;
        }
    }
    if (!FILL) cnt[r] = c;
}

template <class T>
std::vector<T> download(const T* d, int64_t n) {
    std::vector<T> h(static_cast<size_t>(n));
    if (n) KR_CK(cudaMemcpy(h.data(), d, sizeof(T) * size_t(n), cudaMemcpyDeviceToHost));
    return h;
}

template <class T>
T* upload_vec(const std::vector<T>& v) {
    T* p = dev_alloc<T>(int64_t(v.size()));
    if (!v.empty()) KR_CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return p;
}

void fetch(kr_devfactors* out, int w, const std::vector<int64_t>& ptr, const int32_t* in, const double* va) {
    const int64_t n = ptr.back();
    out->outer[w].alloc(int64_t(ptr.size()));
    std::memcpy(out->outer[w].p, ptr.data(), 8 * ptr.size());
    out->inner[w].alloc(n);
    out->val[w].alloc(n);
    if (n) {
        KR_CK(cudaMemcpyAsync(out->inner[w].p, in, 4 * size_t(n), cudaMemcpyDeviceToHost));
        KR_CK(cudaMemcpyAsync(out->val[w].p, va, 8 * size_t(n), cudaMemcpyDeviceToHost));
        KR_CK(cudaDeviceSynchronize());
    }
}

std::vector<int64_t> exclusive(const std::vector<int64_t>& c) {
    std::vector<int64_t> p(c.size() + 1, 0);
    for (size_t q = 0; q < c.size(); ++q) p[q + 1] = p[q] + c[q];
    return p;
}

struct DevBuf {
    std::vector<void*> ptrs;
    template <class T>
    T* alloc(int64_t n) {
        T* p = dev_alloc<T>(std::max<int64_t>(n, 1));
        ptrs.push_back(p);
        return p;
    }
    template <class T>
    T* up(const std::vector<T>& v) {
        T* p = upload_vec(v);
        ptrs.push_back(p);
        return p;
    }
    ~DevBuf() {
        for (void* p : ptrs) krb::dev_free(p);
    }
};

kr_devfactors* build(const kr_kron_board& B, int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Fail{KR_NO_DEVICE, "no CUDA device available (no CPU fallback)"};
    }
    if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
    if (B.m1 < 1 || B.m2 < 1 || B.n1 < 1 || B.n2 < 1) throw Fail{KR_INVALID_INPUT, "empty board"};
    if (B.F.outer_size != B.n1 || B.S.outer_size != B.n1) throw Fail{KR_INVALID_INPUT, "F / S must be n1 x n2 CSR"};
    KR_CK(cudaSetDevice(device));
    cudaEvent_t e0, e1;
    KR_CK(cudaEventCreate(&e0));
    KR_CK(cudaEventCreate(&e1));
    KR_CK(cudaEventRecord(e0));
    const int m1 = B.m1, m2 = B.m2, n1 = B.n1, n2 = B.n2;
    DevBuf D;
    const int64_t nF = B.F.outer[n1], nSn = B.S.outer[n1];
    Pieces P{m1, m2, n1, n2,
             D.up(std::vector<uint32_t>(B.key1, B.key1 + m1)), D.up(std::vector<uint32_t>(B.key2, B.key2 + m2)),
             D.up(std::vector<uint8_t>(B.cards1, B.cards1 + 2 * m1)),
             D.up(std::vector<uint8_t>(B.cards2, B.cards2 + 2 * m2)),
             D.up(std::vector<double>(B.lambda1, B.lambda1 + m1)), D.up(std::vector<double>(B.lambda2, B.lambda2 + m2)),
             D.up(std::vector<int64_t>(B.F.outer, B.F.outer + n1 + 1)),
             D.up(std::vector<int32_t>(B.F.inner, B.F.inner + nF)), D.up(std::vector<double>(B.F.val, B.F.val + nF)),
             D.up(std::vector<int64_t>(B.S.outer, B.S.outer + n1 + 1)),
             D.up(std::vector<int32_t>(B.S.inner, B.S.inner + nSn)),
             D.up(std::vector<double>(B.S.val, B.S.val + nSn))};
    // sequence facts and chain bookkeeping (host, O(m1 + n1))
    std::vector<int32_t> sRank(static_cast<size_t>(n1), -1), fRankD;
    int nS = 0;
    for (int d = 0; d < n1; ++d)
        if (B.S.outer[d + 1] > B.S.outer[d]) sRank[size_t(d)] = nS++;
    bool anyL2 = false;
    for (int j = 0; j < m2; ++j) anyL2 |= B.lambda2[j] != 0.0;
    uint8_t* dAlive = D.alloc<uint8_t>(m1);
    k_row_alive<<<unsigned(m1), 256>>>(P, dAlive);
    KR_CK_LAUNCH();
    const std::vector<uint8_t> alive = download(dAlive, m1);
    std::vector<int32_t> aliveRows, aliveRank(static_cast<size_t>(m1), -1), prevAlive(static_cast<size_t>(m1), -1);
    for (int i = 0; i < m1; ++i) {
        if (alive[size_t(i)]) {
            aliveRank[size_t(i)] = int32_t(aliveRows.size());
            aliveRows.push_back(i);
        }
        prevAlive[size_t(i)] = alive[size_t(i)] ? i : (i ? prevAlive[size_t(i) - 1] : -1);
    }
    const int64_t KS = int64_t(aliveRows.size()) * nS;
    std::vector<int32_t> fcolOf(static_cast<size_t>(n1), -1);
    int64_t k = KS;
    for (int d = 0; d < n1; ++d)
        if (B.F.outer[d + 1] > B.F.outer[d] && anyL2) {
            fcolOf[size_t(d)] = int32_t(k++);
            fRankD.push_back(d);
        }
    std::vector<int32_t> lastKept(static_cast<size_t>(m1) * n1, -1);
    for (int i = 0; i < m1; ++i)
        for (int d = 0; d < n1; ++d)
            if (sRank[size_t(d)] >= 0 && prevAlive[size_t(i)] >= 0)
                lastKept[size_t(i) * n1 + d] = int32_t(int64_t(aliveRank[size_t(prevAlive[size_t(i)])]) * nS + sRank[size_t(d)]);
    auto* out = new kr_devfactors();
    try {
        out->rows = int64_t(m1) * n1;
        out->cols = int64_t(m2) * n2;
        out->k = k;
        out->n1 = n1;
        out->n2 = n2;
        const int64_t R = out->rows;
        // --- Ahat (CSR rows x cols) ---
        {
            int64_t* cnt = D.alloc<int64_t>(R);
            const size_t sm = sizeof(int) * size_t(m2);
            k_ahat<false><<<unsigned(m1), 256, sm>>>(P, cnt, nullptr, nullptr, nullptr);
            KR_CK_LAUNCH();
            const auto ptr = exclusive(download(cnt, R));
            int64_t* dptr = D.up(ptr);
            int32_t* in = D.alloc<int32_t>(ptr.back());
            double* va = D.alloc<double>(ptr.back());
            k_ahat<true><<<unsigned(m1), 256, sm>>>(P, nullptr, dptr, in, va);
            KR_CK_LAUNCH();
            fetch(out, 0, ptr, in, va);
        }
        // --- U (CSR rows x k) ---
        {
            int32_t* dLast = D.up(lastKept);
            int32_t* dF = D.up(fcolOf);
            int64_t* cnt = D.alloc<int64_t>(R);
            const unsigned g = unsigned((R + 255) / 256);
            k_u<false><<<g, 256>>>(m1, n1, P.l1, dLast, dF, cnt, nullptr, nullptr, nullptr);
            KR_CK_LAUNCH();
            const auto ptr = exclusive(download(cnt, R));
            int64_t* dptr = D.up(ptr);
            int32_t* in = D.alloc<int32_t>(ptr.back());
            double* va = D.alloc<double>(ptr.back());
            k_u<true><<<g, 256>>>(m1, n1, P.l1, dLast, dF, nullptr, dptr, in, va);
            KR_CK_LAUNCH();
            fetch(out, 1, ptr, in, va);
        }
        // --- M (CSC k x k): unit diagonal, -1 to the next kept column of the chain ---
        {
            const int64_t nAlive = int64_t(aliveRows.size());
            const int64_t links = KS > 0 ? KS - nS : 0;  // every S column but a chain's last row
            out->outer[2].alloc(k + 1);
            out->inner[2].alloc(k + links);
            out->val[2].alloc(k + links);
            int64_t q = 0;
            out->outer[2].p[0] = 0;
            for (int64_t c = 0; c < k; ++c) {
                out->inner[2].p[q] = int32_t(c);
                out->val[2].p[q++] = 1.0;
                if (c < KS && c / nS + 1 < nAlive) {
                    out->inner[2].p[q] = int32_t(c + nS);
                    out->val[2].p[q++] = -1.0;
                }
                out->outer[2].p[c + 1] = q;
            }
        }
        // --- V (CSC cols x k): S-part columns, then the F-part ---
        {
            int64_t* cnt = D.alloc<int64_t>(k);
            int32_t* dRows = D.up(aliveRows);
            int32_t* dSR = D.up(sRank);
            int32_t* dFR = D.up(fRankD);
            const size_t sm = sizeof(int) * size_t(m2);
            if (!aliveRows.empty() && nS)
                k_vs<false><<<unsigned(aliveRows.size()), 256, sm>>>(P, dRows, dSR, nS, cnt, nullptr, nullptr, nullptr);
            if (!fRankD.empty())
                k_vf<false><<<unsigned(fRankD.size()), 32>>>(P, dFR, KS, cnt, nullptr, nullptr, nullptr);
            KR_CK_LAUNCH();
            const auto ptr = exclusive(download(cnt, k));
            int64_t* dptr = D.up(ptr);
            int32_t* in = D.alloc<int32_t>(ptr.back());
            double* va = D.alloc<double>(ptr.back());
            if (!aliveRows.empty() && nS)
                k_vs<true><<<unsigned(aliveRows.size()), 256, sm>>>(P, dRows, dSR, nS, nullptr, dptr, in, va);
            if (!fRankD.empty()) k_vf<true><<<unsigned(fRankD.size()), 32>>>(P, dFR, KS, nullptr, dptr, in, va);
            KR_CK_LAUNCH();
            fetch(out, 3, ptr, in, va);
        }
        KR_CK(cudaEventRecord(e1));
        KR_CK(cudaEventSynchronize(e1));
        float ms = 0;
        KR_CK(cudaEventElapsedTime(&ms, e0, e1));
        out->seconds = ms / 1e3;
    } catch (...) {
        delete out;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        throw;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return out;
}

}  // namespace
}  // namespace krb

extern "C" {

int kr_factors_build_device(const kr_kron_board* b, int device, kr_devfactors** out) {
    return krb::guarded([&] {
        if (!b || !out) throw krb::Fail{KR_INVALID_INPUT, "null argument"};
        *out = krb::build(*b, device);
    });
}

int kr_devfactors_view(const kr_devfactors* f, kr_factors* out) {
    return krb::guarded([&] {
        if (!f || !out) throw krb::Fail{KR_INVALID_INPUT, "null argument"};
        auto view = [](const kr_devfactors* g, int w, int64_t outerSize) {
            return kr_compressed{outerSize, g->outer[w].data(), g->inner[w].data(), g->val[w].data()};
        };
        *out = kr_factors{f->rows, f->cols, f->k, view(f, 0, f->rows), view(f, 1, f->rows), view(f, 2, f->k),
                          view(f, 3, f->k), f->n1, f->n2};
    });
}

double kr_devfactors_seconds(const kr_devfactors* f) { return f ? f->seconds : 0.0; }

void kr_devfactors_free(kr_devfactors* f) { delete f; }

}  // extern "C"
