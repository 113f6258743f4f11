// kr_kfengine.cu — the Kronecker-factored engine: Technique B with
// postprocessing (sparsify.hpp:246-406) evaluated from its Kronecker factors,
// never from the expanded Â, U, M, V.
//
// Technique B writes the factors as Kronecker products of hand-space pieces
// with the betting tree's F and S (sparsify.hpp:255-275):
//   Â = −(Λ₁ H× Λ₂) ⊗ F        U = [Λ₁ ⊗ I | λ₁ ⊗ I]
//   M = blockdiag(D ⊗ I, I)     V = [(Λ₂ Yᵀ) ⊗ Sᵀ | λ₂ ⊗ Fᵀ],  Y = D W.
// This engine keeps only the hand-space pieces (λ₁, λ₂, the blocked-hand lists
// of H×, the sparsity of Y with its small-integer values, which postprocess
// leaves as chains over the "alive" rows) and the tree's F and S, a few hundred
// KB per board instead of ~150 MB, and expands each ⊗ on the fly.
//
// BITWISE contract: every output is the sum of the same terms, in the same
// order, as the reference's matvec / matvecTranspose (engine.hpp:58-133) over
// the postprocessed factors in Eigen storage order, each term produced by the
// host builder's expressions (kr_devengine.cu rows_vt / rows_ua / rows_ut /
// rows_av restate them):
//   t(r,a)  = Σ_j↑ Σ_{e∈S_a}  ((λ2_j·Y_ij)·S_e)·x[j,col_e]           (Vᵀ row)
//   t_f(a)  = Σ_j↑ Σ_{e∈F_a}  (λ2_j·F_e)·x[j,col_e]                  (Vᵀ F row)
//   z       = M⁻¹ t: z(r) = t(r) + z(r−1) along each chain             (engine.hpp:31-41)
//   y[i,a]  = λ1_i·z(prev alive(i), a) + λ1_i·z_f(a)                  (U, then)
//             + Σ_{j∈blk(i)↑} Σ_{e∈F_a} ((−λ1_i)·λ2_j·F_e)·x[j,col_e]  (Â, engine.hpp:81-89)
// and the transposed chain for Aᵀy (engine.hpp:96-133).  Contraction is off
// (-fmad=false), so each a·b + c rounds twice as on the reference's x86-64.
//
// One exact rewrite is used on the Y terms: with Y_ij ∈ {±1, ±2} (an exact
// power-of-two scale), ((λ2·Y)·S)·x == Y·((λ2·S)·x) in IEEE arithmetic as long
// as no product is subnormal or overflows.  The per-(j, e) product
// Q = (λ2_j·S_e)·x[j,col_e] is then formed once per CTA and each Vᵀ term is one
// fused Y·Q + acc (exact: Y·Q needs no rounding).  The kernels check the
// premise per CTA (every staged x / z either 0 or within [2^-900, 2^900], every
// λ2·S within [2^-100, 2^100]) and otherwise evaluate the literal expressions.
//
// Work decomposes by sequence: y[:, a] depends only on row a of F and S, and
// Aᵀy[:, b] only on column b.  So one CTA computes one output column of one
// board end to end — stage the input columns it needs, the Vᵀ (Uᵀ) rows of its
// chain, the chain solve (one thread; the order is fixed), then the output rows
// — with every intermediate in shared memory and one launch per product.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "kr_common.cuh"

namespace krb {

namespace {

constexpr int kKfThreads = 256;
constexpr int kKfMaxHands = 2047;   // 11-bit hand / alive-rank indices in the packed lists
constexpr int kKfMaxSeq = 1024;     // F / S CSR rows and columns

// One list-of-lists in SELL-32 layout: entry k of row r lives at
// ptr[r / 32] + 32 k + r % 32, so a warp's 32 rows load 64 contiguous bytes
// per step.  Entries are 16-bit: an index (11 bits) and, for the Y lists,
// Y + 2 in bits 11-13.
struct KfList {
    const int32_t* ptr = nullptr;   // per slice of 32 rows
    const int32_t* len = nullptr;   // per row
    const uint16_t* ent = nullptr;
};

struct KfBoard {
    int m1, m2, n1, n2;
    int nAlive, fast;                 // fast: every λ2·S in [2^-100, 2^100] (or 0)
    int64_t rowOff, colOff;           // y / x offsets of the board
    const double *l1, *l2;
    const int32_t* aliveRows;         // [nAlive]
    const int32_t* aliveEnd;          // [nAlive]: next alive row, or m1 (Uᵀ row range)
    const int32_t* rankPrev;          // [m1]: alive rank of the last alive row <= i, or -1
    const int32_t *fptr, *fcol;       // F CSR (n1 + 1), and CSC (n2 + 1)
    const double* fval;
    const int32_t *fcptr, *fcrow;
    const double* fcval;
    const int32_t *sptr, *scol;       // S CSR, CSC
    const double* sval;
    const int32_t *scptr, *scrow;
    const double* scval;
    const uint8_t* hasF;              // [n1]: F row d is a kept U/V column (fcolOf >= 0)
    KfList yr;                        // alive r -> (j, Y) with λ2_j·Y ≠ 0, j asc   (Vᵀ rows)
    KfList yc;                        // j -> (alive r, Y) with λ2_j·Y ≠ 0, r asc   (V rows)
    KfList b2;                        // i -> blocked j asc                          (Â rows)
    KfList b1;                        // j -> blocked i asc                          (Âᵀ rows)
};

__device__ __forceinline__ int kf_idx(uint16_t e) { return int(e & 0x7FF); }
__device__ __forceinline__ double kf_y(uint16_t e) { return double(int(e >> 11) - 2); }

// staged value admissible for the Y-factoring rewrite
__device__ __forceinline__ bool kf_ok(double v) {
    const double a = fabs(v);
    return a == 0.0 || (a >= 0x1p-900 && a <= 0x1p900);
}

// Ordered fold of n values (the sum order is fixed: one thread, one chain of
// dependent adds); loads are issued ahead of the adds.
__device__ __forceinline__ double kf_fold(const double* v, int n) {
    double acc = 0.0;
    int i = 0;
    for (; i + 8 <= n; i += 8) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = v[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = acc + t[u];
    }
    for (; i < n; ++i) acc = acc + v[i];
    return acc;
}

// In-place chain solve with −1 multipliers: z(r) = t(r) + z(r∓1)
// (solveUnitLower / solveUnitLowerT, engine.hpp:31-54: z_r -= (−1)·z_prev is
// bitwise t_r + z_prev).  The first element keeps t (t + (−0) == t).
template <int DIR>
__device__ __forceinline__ void kf_chain(double* tz, int n) {
    double z = -0.0;
    if (DIR > 0) {
        int r = 0;
        for (; r + 8 <= n; r += 8) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = tz[r + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                z = t[u] + z;
                tz[r + u] = z;
            }
        }
        for (; r < n; ++r) {
            z = tz[r] + z;
            tz[r] = z;
        }
    } else {
        int r = n - 1;
        for (; r - 8 >= -1; r -= 8) {
            double t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = tz[r - u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                z = t[u] + z;
                tz[r - u] = z;
            }
        }
        for (; r >= 0; --r) {
            z = tz[r] + z;
            tz[r] = z;
        }
    }
}

// ---------------------------------------------------------------------------
// A x: one CTA per (player-1 sequence a, board).
// shared: l2[m2] | xF[nFa][m2] | Q[nSa][m2] | fprod[m2 * nFa] | tz[nAlive] | zf
// ---------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(T) k_kf_ax(const KfBoard* __restrict__ boards, int b0,
                                              const double* __restrict__ x, double* __restrict__ y) {
    pdl_entry();
    extern __shared__ double sm[];
    __shared__ int okAll;
    __shared__ double zf;
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int a = blockIdx.x;
    const int m1 = B.m1, m2 = B.m2, n1 = B.n1, n2 = B.n2;
    const int f0 = B.fptr[a], nFa = B.fptr[a + 1] - f0;
    const int s0 = B.sptr[a], nSa = B.sptr[a + 1] - s0;
    const bool chain = nSa > 0 && B.nAlive > 0;
    const bool fA = B.hasF[a] != 0;
    double* l2s = sm;
    double* xF = l2s + m2;
    double* Q = xF + size_t(nFa) * m2;
    double* fprod = Q + size_t(nSa) * m2;
    double* tz = fprod + size_t(nFa) * m2;
    const double* xb = x + B.colOff;
    if (threadIdx.x == 0) okAll = 1;
    __syncthreads();
    int ok = B.fast;
    for (int j = threadIdx.x; j < m2; j += T) {
        const double l2 = B.l2[j];
        l2s[j] = l2;
        for (int e = 0; e < nFa; ++e) {
            const double xv = xb[int64_t(j) * n2 + B.fcol[f0 + e]];
            xF[size_t(e) * m2 + j] = xv;
            fprod[size_t(j) * nFa + e] = (l2 * B.fval[f0 + e]) * xv;   // Vᵀ F row term (rows_vt)
        }
        for (int e = 0; e < nSa; ++e) {
            const double xv = xb[int64_t(j) * n2 + B.scol[s0 + e]];
            ok &= kf_ok(xv);
            Q[size_t(e) * m2 + j] = (l2 * B.sval[s0 + e]) * xv;
        }
    }
    if (!ok) okAll = 0;  // benign race: every writer stores 0
    __syncthreads();
    const bool fast = okAll != 0;
    // Vᵀ rows of chain a: t(r) = Σ_j↑ Σ_e ((λ2_j·Y)·S_e)·x[j, col_e]
    if (chain) {
        for (int r = threadIdx.x; r < B.nAlive; r += T) {
            const int len = B.yr.len[r];
            const uint16_t* p = B.yr.ent + B.yr.ptr[r >> 5] + (r & 31);
            double acc = 0.0;
            if (fast) {
                if (nSa == 1) {
                    int k = 0;
                    for (; k + 4 <= len; k += 4) {
                        uint16_t ee[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) ee[u] = p[32 * (k + u)];
                        double q[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) q[u] = Q[kf_idx(ee[u])];
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc = fma(kf_y(ee[u]), q[u], acc);
                    }
                    for (; k < len; ++k) {
                        const uint16_t ee = p[32 * k];
                        acc = fma(kf_y(ee), Q[kf_idx(ee)], acc);
                    }
                } else {
                    for (int k = 0; k < len; ++k) {
                        const uint16_t ee = p[32 * k];
                        const int j = kf_idx(ee);
                        const double yv = kf_y(ee);
                        for (int e = 0; e < nSa; ++e) acc = fma(yv, Q[size_t(e) * m2 + j], acc);
                    }
                }
            } else {
                for (int k = 0; k < len; ++k) {
                    const uint16_t ee = p[32 * k];
                    const int j = kf_idx(ee);
                    const double scale = l2s[j] * kf_y(ee);
                    for (int e = 0; e < nSa; ++e) {
                        const double v = scale * B.sval[s0 + e];
                        acc = acc + v * xb[int64_t(j) * n2 + B.scol[s0 + e]];
                    }
                }
            }
            tz[r] = acc;
        }
    }
    __syncthreads();
    // the two ordered folds: the chain solve (warp 0) and the F row (warp 1)
    if (threadIdx.x == 0 && chain) kf_chain<1>(tz, B.nAlive);
    if (threadIdx.x == 32 && fA) zf = kf_fold(fprod, m2 * nFa);
    __syncthreads();
    // [U | Â] rows (i, a): U terms, then the blocked hands in order
    const double zfa = fA ? zf : 0.0;
    double* yb = y + B.rowOff;
    for (int i = threadIdx.x; i < m1; i += T) {
        const double v = B.l1[i];
        double acc = 0.0;
        if (v != 0.0) {
            const int rp = B.rankPrev[i];
            if (chain && rp >= 0) acc = acc + v * tz[rp];
            if (fA) acc = acc + v * zfa;
        }
        if (nFa > 0) {
            const int len = B.b2.len[i];
            const uint16_t* p = B.b2.ent + B.b2.ptr[i >> 5] + (i & 31);
            const double nv = -v;
            if (nFa == 1) {
                const double fv = B.fval[f0];
                int k = 0;
                for (; k + 4 <= len; k += 4) {
                    int jj[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) jj[u] = kf_idx(p[32 * (k + u)]);
                    double l[4], xv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        l[u] = l2s[jj[u]];
                        xv[u] = xF[jj[u]];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double w = (nv * l[u]) * fv;
                        acc = acc + w * xv[u];
                    }
                }
                for (; k < len; ++k) {
                    const int j = kf_idx(p[32 * k]);
                    const double w = (nv * l2s[j]) * fv;
                    acc = acc + w * xF[j];
                }
            } else {
                for (int k = 0; k < len; ++k) {
                    const int j = kf_idx(p[32 * k]);
                    const double scale = nv * l2s[j];
                    for (int e = 0; e < nFa; ++e) {
                        const double w = scale * B.fval[f0 + e];
                        acc = acc + w * xF[size_t(e) * m2 + j];
                    }
                }
            }
        }
        yb[int64_t(i) * n1 + a] = acc;
    }
}

// ---------------------------------------------------------------------------
// Aᵀ y: one CTA per (player-2 sequence b, board).
// shared: l1[m1] | yF[nFb][m1] | fprod[nFb][m1] | sz[nSb][nAlive] | yS[nSb][m1] | zf[nFb]
// ---------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(T) k_kf_atx(const KfBoard* __restrict__ boards, int b0,
                                               const double* __restrict__ y, double* __restrict__ x) {
    pdl_entry();
    extern __shared__ double sm[];
    __shared__ int okAll;
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int b = blockIdx.x;
    const int m1 = B.m1, m2 = B.m2, n1 = B.n1, n2 = B.n2;
    const int f0 = B.fcptr[b], nFb = B.fcptr[b + 1] - f0;
    const int s0 = B.scptr[b], nSb = B.scptr[b + 1] - s0;
    const int nA = B.nAlive;
    double* l1s = sm;
    double* yF = l1s + m1;
    double* fprod = yF + size_t(nFb) * m1;
    double* sz = fprod + size_t(nFb) * m1;
    double* yS = sz + size_t(nSb) * nA;
    double* zf = yS + size_t(nSb) * m1;
    const double* yb = y + B.rowOff;
    if (threadIdx.x == 0) okAll = 1;
    for (int i = threadIdx.x; i < m1; i += T) {
        const double l1 = B.l1[i];
        l1s[i] = l1;
        for (int e = 0; e < nFb; ++e) {
            const double yv = yb[int64_t(i) * n1 + B.fcrow[f0 + e]];
            yF[size_t(e) * m1 + i] = yv;
            fprod[size_t(e) * m1 + i] = l1 * yv;   // Uᵀ F-column row terms (rows_ut)
        }
        for (int e = 0; e < nSb; ++e) yS[size_t(e) * m1 + i] = yb[int64_t(i) * n1 + B.scrow[s0 + e]];
    }
    __syncthreads();
    // Uᵀ rows of each chain d ∈ S column b: s(r) = Σ_{i ∈ [alive r, alive r+1)} λ1_i·y[i, d]
    int ok = 1;
    for (int e = 0; e < nSb; ++e)
        for (int r = threadIdx.x; r < nA; r += T) {
            double acc = 0.0;
            for (int i = B.aliveRows[r]; i < B.aliveEnd[r]; ++i) acc = acc + l1s[i] * yS[size_t(e) * m1 + i];
            sz[size_t(e) * nA + r] = acc;
        }
    __syncthreads();
    {   // ordered folds: the backward chains, then the F-column sums
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int task = w; task < nSb + nFb; task += T / 32)
            if (lane == 0) {
                if (task < nSb) kf_chain<-1>(sz + size_t(task) * nA, nA);
                else if (B.hasF[B.fcrow[f0 + task - nSb]]) zf[task - nSb] = kf_fold(fprod + size_t(task - nSb) * m1, m1);
            }
    }
    __syncthreads();
    for (int e = 0; e < nSb; ++e)
        for (int r = threadIdx.x; r < nA; r += T) ok &= kf_ok(sz[size_t(e) * nA + r]);
    if (!ok) okAll = 0;
    __syncthreads();
    const bool zok = okAll != 0 && B.fast;
    double* xb = x + B.colOff;
    for (int j = threadIdx.x; j < m2; j += T) {
        const double l2 = B.l2[j];
        double acc = 0.0;
        if (nFb > 0) {   // Âᵀ: blocked i ascending, F column b
            const int len = B.b1.len[j];
            const uint16_t* p = B.b1.ent + B.b1.ptr[j >> 5] + (j & 31);
            if (nFb == 1) {
                const double fv = B.fcval[f0];
                int k = 0;
                for (; k + 4 <= len; k += 4) {
                    int ii[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) ii[u] = kf_idx(p[32 * (k + u)]);
                    double l[4], yv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        l[u] = l1s[ii[u]];
                        yv[u] = yF[ii[u]];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double w = (-l[u] * l2) * fv;
                        acc = acc + w * yv[u];
                    }
                }
                for (; k < len; ++k) {
                    const int i = kf_idx(p[32 * k]);
                    const double w = (-l1s[i] * l2) * fv;
                    acc = acc + w * yF[i];
                }
            } else {
                for (int k = 0; k < len; ++k) {
                    const int i = kf_idx(p[32 * k]);
                    const double scale = -l1s[i] * l2;
                    for (int e = 0; e < nFb; ++e) {
                        const double w = scale * B.fcval[f0 + e];
                        acc = acc + w * yF[size_t(e) * m1 + i];
                    }
                }
            }
        }
        if (nSb > 0 && nA > 0) {   // V, S columns: alive r ascending, S column b
            const int len = B.yc.len[j];
            const uint16_t* p = B.yc.ent + B.yc.ptr[j >> 5] + (j & 31);
            if (zok && nSb == 1) {
                const double P = l2 * B.scval[s0];
                int k = 0;
                for (; k + 4 <= len; k += 4) {
                    uint16_t ee[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) ee[u] = p[32 * (k + u)];
                    double z[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) z[u] = sz[kf_idx(ee[u])];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc = fma(kf_y(ee[u]), P * z[u], acc);
                }
                for (; k < len; ++k) {
                    const uint16_t ee = p[32 * k];
                    acc = fma(kf_y(ee), P * sz[kf_idx(ee)], acc);
                }
            } else {
                for (int k = 0; k < len; ++k) {
                    const uint16_t ee = p[32 * k];
                    const int r = kf_idx(ee);
                    const double scale = l2 * kf_y(ee);
                    for (int e = 0; e < nSb; ++e) {
                        const double w = scale * B.scval[s0 + e];
                        acc = acc + w * sz[size_t(e) * nA + r];
                    }
                }
            }
        }
        if (l2 != 0.0)   // V, F columns
            for (int e = 0; e < nFb; ++e)
                if (B.hasF[B.fcrow[f0 + e]]) acc = acc + (l2 * B.fcval[f0 + e]) * zf[e];
        xb[int64_t(j) * n2 + b] = acc;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct HostList {
    std::vector<int32_t> ptr, len;
    std::vector<uint16_t> ent;
    void build(const std::vector<std::vector<uint16_t>>& rows) {
        const int R = int(rows.size());
        const int S = (R + 31) / 32;
        ptr.assign(size_t(S) + 1, 0);
        len.assign(size_t(R), 0);
        for (int s = 0; s < S; ++s) {
            int w = 0;
            for (int l = 0; l < 32 && 32 * s + l < R; ++l) w = std::max<int>(w, int(rows[size_t(32 * s + l)].size()));
            ptr[size_t(s) + 1] = ptr[size_t(s)] + 32 * w;
        }
        ent.assign(size_t(std::max(ptr.back(), 1)), 0);
        for (int r = 0; r < R; ++r) {
            len[size_t(r)] = int32_t(rows[size_t(r)].size());
            for (size_t k = 0; k < rows[size_t(r)].size(); ++k)
                ent[size_t(ptr[size_t(r / 32)]) + 32 * k + size_t(r % 32)] = rows[size_t(r)][k];
        }
    }
};

struct HostBoard {
    int m1 = 0, m2 = 0, n1 = 0, n2 = 0, nAlive = 0, nS = 0, nF = 0, fast = 1;
    std::vector<double> l1, l2;
    std::vector<int32_t> aliveRows, aliveEnd, rankPrev;
    std::vector<int32_t> fptr, fcol, fcptr, fcrow, sptr, scol, scptr, scrow;
    std::vector<double> fval, fcval, sval, scval;
    std::vector<uint8_t> hasF;
    HostList yr, yc, b2, b1;
    int64_t nnzA = 0, nnzU = 0, nnzV = 0, nnzM = 0, K = 0;
    int maxFa = 0, maxSa = 0, maxFb = 0, maxSb = 0;
};

void csr_copy(const kr_compressed& A, int rows, int cols, const char* name, int b, std::vector<int32_t>& ptr,
              std::vector<int32_t>& idx, std::vector<double>& val, std::vector<int32_t>& cptr,
              std::vector<int32_t>& cidx, std::vector<double>& cval) {
    const std::string at = "board " + std::to_string(b) + ": ";
    if (A.outer_size != rows || !A.outer) throw Fail{KR_INVALID_INPUT, at + name + " has the wrong shape"};
    if (A.outer[0] != 0) throw Fail{KR_INVALID_INPUT, at + name + " outer[0] must be 0"};
    const int64_t nnz = A.outer[rows];
    if (nnz > 0 && (!A.inner || !A.val)) throw Fail{KR_INVALID_INPUT, at + name + " has null arrays"};
    ptr.assign(size_t(rows) + 1, 0);
    for (int r = 0; r < rows; ++r) {
        if (A.outer[r + 1] < A.outer[r]) throw Fail{KR_INVALID_INPUT, at + name + " outer not monotone"};
        ptr[size_t(r) + 1] = int32_t(A.outer[r + 1]);
        for (int64_t e = A.outer[r]; e < A.outer[r + 1]; ++e) {
            if (A.inner[e] < 0 || A.inner[e] >= cols || (e > A.outer[r] && A.inner[e] <= A.inner[e - 1]))
                throw Fail{KR_INVALID_INPUT, at + name + " inner indices out of range or not ascending"};
            if (!std::isfinite(A.val[e])) throw Fail{KR_INVALID_INPUT, at + name + " has a non-finite value"};
        }
    }
    idx.assign(A.inner, A.inner + nnz);
    val.assign(A.val, A.val + nnz);
    // CSC by a stable counting sort (rows ascending within a column)
    cptr.assign(size_t(cols) + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) cptr[size_t(A.inner[e]) + 1]++;
    for (int c = 0; c < cols; ++c) cptr[size_t(c) + 1] += cptr[size_t(c)];
    cidx.resize(size_t(nnz));
    cval.resize(size_t(nnz));
    std::vector<int32_t> pos(cptr.begin(), cptr.end() - 1);
    for (int r = 0; r < rows; ++r)
        for (int64_t e = A.outer[r]; e < A.outer[r + 1]; ++e) {
            const int32_t q = pos[size_t(A.inner[e])]++;
            cidx[size_t(q)] = r;
            cval[size_t(q)] = A.val[e];
        }
}

// Technique B post in Kronecker form for one board (the closed form the
// device enumerators of kr_devengine.cu follow; sparsify.hpp:246-406).
void build_host_board(const kr_kron_board& K, int b, HostBoard& H) {
    const std::string at = "board " + std::to_string(b) + ": ";
    const int m1 = K.m1, m2 = K.m2, n1 = K.n1, n2 = K.n2;
    if (m1 < 1 || m2 < 1 || n1 < 1 || n2 < 1) throw Fail{KR_INVALID_INPUT, at + "empty board"};
    if (m1 > kKfMaxHands || m2 > kKfMaxHands)
        throw Fail{KR_INVALID_INPUT, at + "more than 2047 hands per side (use the factored engine)"};
    if (n1 > kKfMaxSeq || n2 > kKfMaxSeq) throw Fail{KR_INVALID_INPUT, at + "tree too large"};
    if (!K.key1 || !K.key2 || !K.cards1 || !K.cards2 || !K.lambda1 || !K.lambda2)
        throw Fail{KR_INVALID_INPUT, at + "null hand arrays"};
    for (int p = 0; p < 2; ++p) {
        const int m = p ? m2 : m1;
        const uint32_t* key = p ? K.key2 : K.key1;
        const uint8_t* c = p ? K.cards2 : K.cards1;
        const double* l = p ? K.lambda2 : K.lambda1;
        for (int i = 0; i < m; ++i) {
            if (i > 0 && key[i] < key[i - 1])
                throw Fail{KR_INVALID_INPUT, at + "hands must be strength-sorted ascending (kron.hpp:74-83)"};
            if (c[2 * i] >= 52 || c[2 * i + 1] >= 52 || c[2 * i] == c[2 * i + 1])
                throw Fail{KR_INVALID_INPUT, at + "bad hand cards"};
            if (!std::isfinite(l[i])) throw Fail{KR_INVALID_INPUT, at + "non-finite lambda"};
        }
    }
    H.m1 = m1;
    H.m2 = m2;
    H.n1 = n1;
    H.n2 = n2;
    H.l1.assign(K.lambda1, K.lambda1 + m1);
    H.l2.assign(K.lambda2, K.lambda2 + m2);
    csr_copy(K.F, n1, n2, "F", b, H.fptr, H.fcol, H.fval, H.fcptr, H.fcrow, H.fcval);
    csr_copy(K.S, n1, n2, "S", b, H.sptr, H.scol, H.sval, H.scptr, H.scrow, H.scval);
    auto compat = [&](int i, int j) {
        const int a0 = K.cards1[2 * i], a1 = K.cards1[2 * i + 1], b0 = K.cards2[2 * j], b1 = K.cards2[2 * j + 1];
        return a0 != b0 && a0 != b1 && a1 != b0 && a1 != b1;
    };
    auto wsign = [&](int i, int j) {
        if (!compat(i, j)) return 0;
        const uint32_t a = K.key1[i], c = K.key2[j];
        return a > c ? 1 : (a < c ? -1 : 0);
    };
    // Y = D W over (i, j), kept where λ2_j·Y_ij ≠ 0 (V's entries, rows_vt / rows_av)
    std::vector<std::vector<uint16_t>> yrows(static_cast<size_t>(m1));
    std::vector<int> prev(static_cast<size_t>(m2), 0), cur(static_cast<size_t>(m2), 0);
    std::vector<char> alive(static_cast<size_t>(m1), 0);
    for (int i = 0; i < m1; ++i) {
        for (int j = 0; j < m2; ++j) cur[size_t(j)] = wsign(i, j);
        for (int j = 0; j < m2; ++j) {
            const int yd = i == 0 ? cur[size_t(j)] : cur[size_t(j)] - prev[size_t(j)];
            if (H.l2[size_t(j)] * double(yd) != 0.0) yrows[size_t(i)].push_back(uint16_t(j | ((yd + 2) << 11)));
        }
        alive[size_t(i)] = !yrows[size_t(i)].empty();
        std::swap(prev, cur);
    }
    std::vector<int32_t> aliveRank(static_cast<size_t>(m1), -1);
    for (int i = 0; i < m1; ++i)
        if (alive[size_t(i)]) {
            aliveRank[size_t(i)] = int32_t(H.aliveRows.size());
            H.aliveRows.push_back(i);
        }
    H.nAlive = int(H.aliveRows.size());
    H.rankPrev.assign(size_t(m1), -1);
    for (int i = 0, last = -1; i < m1; ++i) {
        if (alive[size_t(i)]) last = aliveRank[size_t(i)];
        H.rankPrev[size_t(i)] = last;
    }
    H.aliveEnd.resize(size_t(H.nAlive));
    for (int r = 0; r < H.nAlive; ++r) H.aliveEnd[size_t(r)] = r + 1 < H.nAlive ? H.aliveRows[size_t(r) + 1] : m1;
    std::vector<std::vector<uint16_t>> yr(static_cast<size_t>(H.nAlive)), yc(static_cast<size_t>(m2));
    for (int r = 0; r < H.nAlive; ++r) {
        yr[size_t(r)] = yrows[size_t(H.aliveRows[size_t(r)])];
        for (uint16_t e : yr[size_t(r)]) yc[size_t(e & 0x7FF)].push_back(uint16_t(r | (e & 0x3800)));
    }
    // chains and F columns (kr_devengine.cu pass 0)
    bool anyL2 = false;
    for (double v : H.l2) anyL2 |= v != 0.0;
    H.hasF.assign(size_t(n1), 0);
    for (int d = 0; d < n1; ++d) {
        if (H.sptr[size_t(d) + 1] > H.sptr[size_t(d)]) H.nS++;
        if (H.fptr[size_t(d) + 1] > H.fptr[size_t(d)] && anyL2) {
            H.hasF[size_t(d)] = 1;
            H.nF++;
        }
    }
    // blocked lists (H× = 1 - compat)
    std::vector<std::vector<uint16_t>> b2(static_cast<size_t>(m1)), b1(static_cast<size_t>(m2));
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j)
            if (!compat(i, j)) {
                b2[size_t(i)].push_back(uint16_t(j));
                b1[size_t(j)].push_back(uint16_t(i));
            }
    H.yr.build(yr);
    H.yc.build(yc);
    H.b2.build(b2);
    H.b1.build(b1);
    // the products' fast path premise: every λ2·S in [2^-100, 2^100] or 0
    for (int j = 0; j < m2; ++j)
        for (double s : H.sval) {
            const double p = std::fabs(H.l2[size_t(j)] * s);
            if (p != 0.0 && (p < 0x1p-100 || p > 0x1p100)) H.fast = 0;
        }
    // factor sizes (the flop rule of engine.hpp:72-131), counted as the
    // reference's builder prunes: an entry exists iff its value is nonzero
    for (int d = 0; d < n1; ++d) {
        H.maxFa = std::max(H.maxFa, H.fptr[size_t(d) + 1] - H.fptr[size_t(d)]);
        H.maxSa = std::max(H.maxSa, H.sptr[size_t(d) + 1] - H.sptr[size_t(d)]);
    }
    for (int c = 0; c < n2; ++c) {
        H.maxFb = std::max(H.maxFb, H.fcptr[size_t(c) + 1] - H.fcptr[size_t(c)]);
        H.maxSb = std::max(H.maxSb, H.scptr[size_t(c) + 1] - H.scptr[size_t(c)]);
    }
    for (int r = 0; r < H.nAlive; ++r)
        for (uint16_t e : yr[size_t(r)]) {
            const double scale = H.l2[size_t(e & 0x7FF)] * double(int(e >> 11) - 2);
            for (int d = 0; d < n1; ++d)
                for (int q = H.sptr[size_t(d)]; q < H.sptr[size_t(d) + 1]; ++q) H.nnzV += scale * H.sval[size_t(q)] != 0.0;
        }
    for (int d = 0; d < n1; ++d)
        if (H.hasF[size_t(d)])
            for (int j = 0; j < m2; ++j)
                for (int q = H.fptr[size_t(d)]; q < H.fptr[size_t(d) + 1]; ++q)
                    H.nnzV += H.l2[size_t(j)] != 0.0 && H.l2[size_t(j)] * H.fval[size_t(q)] != 0.0;
    for (int i = 0; i < m1; ++i) {
        const double v = H.l1[size_t(i)];
        for (int a = 0; a < n1; ++a) {
            if (v != 0.0) {
                H.nnzU += (H.sptr[size_t(a) + 1] > H.sptr[size_t(a)] && H.rankPrev[size_t(i)] >= 0) ? 1 : 0;
                H.nnzU += H.hasF[size_t(a)] ? 1 : 0;
            }
            for (uint16_t j : b2[size_t(i)]) {
                const double scale = -v * H.l2[size_t(j)];
                for (int q = H.fptr[size_t(a)]; q < H.fptr[size_t(a) + 1]; ++q) H.nnzA += scale * H.fval[size_t(q)] != 0.0;
            }
        }
    }
    H.K = int64_t(H.nAlive) * H.nS + H.nF;
    H.nnzM = H.K + (H.nAlive > 0 ? int64_t(H.nAlive - 1) * H.nS : 0);
}

template <class T>
T* up(std::vector<void*>& keep, const std::vector<T>& v) {
    T* p = dev_alloc<T>(std::max<int64_t>(int64_t(v.size()), 1));
    keep.push_back(p);
    if (!v.empty()) KR_CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return p;
}

KfList up_list(std::vector<void*>& keep, const HostList& h) {
    KfList l;
    l.ptr = up(keep, h.ptr);
    l.len = up(keep, h.len);
    l.ent = up(keep, h.ent);
    return l;
}

}  // namespace

struct KfState {
    KfBoard* dBoards = nullptr;    // device array
    std::vector<void*> keep;       // every device table
    size_t smem[2] = {0, 0};
    int nb = 0, nSeq[2] = {0, 0};
};

void kf_destroy(KfState* k) {
    if (!k) return;
    for (void* p : k->keep) cudaFree(p);
    delete k;
}

void kf_product(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0, int b1) {
    KfState* k = e->kf;
    if (b1 < 0) b1 = k->nb;
    if (b1 <= b0 || k->nSeq[dir] == 0) return;
    const dim3 grid(unsigned(k->nSeq[dir]), unsigned(b1 - b0));
    if (dir == 0)
        krb::launch(k_kf_ax<kKfThreads>, grid, kKfThreads, k->smem[0], s, k->dBoards, b0, in, out);
    else
        krb::launch(k_kf_atx<kKfThreads>, grid, kKfThreads, k->smem[1], s, k->dBoards, b0, in, out);
    KR_CK_LAUNCH();
    e->launches++;
}

kr_engine* create_kf_engine(const kr_kron_board* boards, int nb, int device, uint32_t flags) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Fail{KR_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    }
    if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
    if (!boards || nb < 1) throw Fail{KR_INVALID_INPUT, "at least one board is required"};
    const int n1 = boards[0].n1, n2 = boards[0].n2;
    for (int b = 0; b < nb; ++b)
        if (boards[b].n1 != n1 || boards[b].n2 != n2)
            throw Fail{KR_INVALID_INPUT, "board " + std::to_string(b) + ": boards must share one betting tree"};
    // host tables, one thread per board group
    std::vector<HostBoard> hb(static_cast<size_t>(nb));
    {
        const int nt = std::max(1, std::min<int>(nb, int(std::thread::hardware_concurrency())));
        std::vector<std::thread> th;
        std::vector<Fail> err(static_cast<size_t>(nt), Fail{KR_OK, ""});
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                try {
                    for (int b = t; b < nb; b += nt) build_host_board(boards[b], b, hb[size_t(b)]);
                } catch (const Fail& f) {
                    err[size_t(t)] = f;
                } catch (const std::exception& x) {
                    err[size_t(t)] = Fail{KR_INVALID_INPUT, x.what()};
                }
            });
        for (auto& t : th) t.join();
        for (auto& f : err)
            if (f.code != KR_OK) throw f;
    }
    int64_t R = 0, C = 0;
    for (auto& H : hb) {
        R += int64_t(H.m1) * n1;
        C += int64_t(H.m2) * n2;
    }
    if (R > INT32_MAX || C > INT32_MAX) throw Fail{KR_INVALID_INPUT, "dimensions exceed 32-bit indices"};
    KR_CK(cudaSetDevice(device));
    kr_engine* e = new kr_engine();
    try {
        e->device = device;
        KR_CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->rows = R;
        e->cols = C;
        e->n1 = n1;
        e->n2 = n2;
        e->mkind = 1;
        e->kf = new KfState();
        KfState& k = *e->kf;
        k.nb = nb;
        k.nSeq[0] = n1;
        k.nSeq[1] = n2;
        std::vector<KfBoard> db(static_cast<size_t>(nb));
        int64_t rowOff = 0, colOff = 0, K = 0;
        size_t sm0 = 0, sm1 = 0;
        for (int b = 0; b < nb; ++b) {
            HostBoard& H = hb[size_t(b)];
            KfBoard& B = db[size_t(b)];
            B.m1 = H.m1;
            B.m2 = H.m2;
            B.n1 = n1;
            B.n2 = n2;
            B.nAlive = H.nAlive;
            B.fast = H.fast;
            B.rowOff = rowOff;
            B.colOff = colOff;
            rowOff += int64_t(H.m1) * n1;
            colOff += int64_t(H.m2) * n2;
            B.l1 = up(k.keep, H.l1);
            B.l2 = up(k.keep, H.l2);
            B.aliveRows = up(k.keep, H.aliveRows);
            B.aliveEnd = up(k.keep, H.aliveEnd);
            B.rankPrev = up(k.keep, H.rankPrev);
            B.fptr = up(k.keep, H.fptr);
            B.fcol = up(k.keep, H.fcol);
            B.fval = up(k.keep, H.fval);
            B.fcptr = up(k.keep, H.fcptr);
            B.fcrow = up(k.keep, H.fcrow);
            B.fcval = up(k.keep, H.fcval);
            B.sptr = up(k.keep, H.sptr);
            B.scol = up(k.keep, H.scol);
            B.sval = up(k.keep, H.sval);
            B.scptr = up(k.keep, H.scptr);
            B.scrow = up(k.keep, H.scrow);
            B.scval = up(k.keep, H.scval);
            B.hasF = up(k.keep, H.hasF);
            B.yr = up_list(k.keep, H.yr);
            B.yc = up_list(k.keep, H.yc);
            B.b2 = up_list(k.keep, H.b2);
            B.b1 = up_list(k.keep, H.b1);
            sm0 = std::max(sm0, 8 * (size_t(H.m2) * (1 + 2 * size_t(H.maxFa) + size_t(H.maxSa)) + size_t(H.nAlive)));
            sm1 = std::max(sm1, 8 * (size_t(H.m1) * (1 + 2 * size_t(H.maxFb) + size_t(H.maxSb)) +
                                     size_t(H.maxSb) * size_t(H.nAlive) + size_t(H.maxFb)));
            e->nnzA += H.nnzA;
            e->nnzU += H.nnzU;
            e->nnzV += H.nnzV;
            e->nnzM += H.nnzM;
            K += H.K;
        }
        e->k = K;
        e->flops_per_product = e->nnzV + e->nnzU + e->nnzA + (e->nnzM - K);
        const size_t limit = 227 * 1024 - 1024;
        if (sm0 > limit || sm1 > limit)
            throw Fail{KR_INVALID_INPUT, "board too large for the Kronecker-factored engine's shared memory"};
        k.smem[0] = sm0;
        k.smem[1] = sm1;
        raise_smem_limit(k_kf_ax<kKfThreads>, sm0);
        raise_smem_limit(k_kf_atx<kKfThreads>, sm1);
        k.dBoards = up(k.keep, db);
        e->d_in = dev_alloc<double>(std::max<int64_t>(std::max(R, C), 1));
        e->d_out = dev_alloc<double>(std::max<int64_t>(std::max(R, C), 1));
        // board groups for the pipelined host-buffer calls (as the implicit engine)
        int G = 8;
        if (const char* env = std::getenv("KR_GROUPS")) G = std::atoi(env);
        G = (flags & KR_FLAG_SINGLE_PART) ? 1 : std::max(1, std::min(nb, G));
        for (int g = 0; g < G; ++g) {
            const int g0 = int(int64_t(nb) * g / G), g1 = int(int64_t(nb) * (g + 1) / G);
            int64_t r = 0, c = 0;
            for (int b = g0; b < g1; ++b) {
                r += int64_t(hb[size_t(b)].m1) * n1;
                c += int64_t(hb[size_t(b)].m2) * n2;
            }
            e->grpBoard.push_back(g1);
            e->grpRow.push_back(e->grpRow.back() + r);
            e->grpCol.push_back(e->grpCol.back() + c);
        }
        engine_make_pipeline(e);
        KR_CK(cudaDeviceSynchronize());
    } catch (...) {
        kr_engine_destroy(e);
        throw;
    }
    return e;
}

}  // namespace krb

extern "C" int kr_engine_create_kfactored(const kr_kron_board* boards, int nboards, int device, uint32_t flags,
                                          kr_engine** out) {
    return krb::guarded([&] {
        if (!out) throw krb::Fail{KR_INVALID_INPUT, "null output handle"};
        *out = krb::create_kf_engine(boards, nboards, device, flags);
    });
}
