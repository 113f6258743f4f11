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
// as no product is subnormal or overflows.  So Aᵀ's per-(j, e) product
// Q = (λ2_j·S_e)·x[j,col_e] is formed once per CTA in its four signed
// variants Y·Q, and each Vᵀ term is one load and one add; Aᵀy's V terms scale
// the chain values the same way.  The kernels check the premise per CTA (every
// staged x / z either 0 or within [2^-900, 2^900], every λ2·S within
// [2^-100, 2^100]) and otherwise evaluate the literal expressions.
//
// Work decomposes by sequence: y[:, a] depends only on row a of F and S, and
// Aᵀy[:, b] only on column b.  So one CTA computes one output column of one
// board end to end — stage the input columns it needs, the Vᵀ (Uᵀ) rows of its
// chain, the chain solve (one thread; the order is fixed), then the output rows
// — with every intermediate in shared memory and one launch per product.
//
// Lists (Y rows, Y columns, blocked hands) are stored as 16-bit entries that
// are already shared-memory byte offsets of the value they select (the signed
// Y·Q / Y·z variant, or the {λ, value} pair of a blocked hand), in a
// SELL-8x32 layout: rows sorted by length, cut into slices of 32, each lane's
// entries in 16-byte vectors of 8 (one load per 8 entries, a warp's 32 vectors
// contiguous).  Padding entries select a zero slot, so every lane of a warp
// runs to the slice width without branches and the padding adds +0.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "kr_common.cuh"

namespace krb {

namespace {

#ifndef KR_KF_WARPS
#define KR_KF_WARPS 8
#endif
constexpr int kKfWarps = KR_KF_WARPS;   // warps (SELL slices) per row-kernel CTA
constexpr int kKfMaxSeq = 1024;     // F / S CSR rows and columns
constexpr int kKfMaxHands = 1364;   // list entries address up to 48 (m + 1) bytes of shared memory (< 64 KB)
constexpr int kKfLong = 256;        // longer list rows take the warp-cooperative path
// fold kernels: one CTA per sequence, all threads stage, two fold (a
// warp-per-fold layout with 4 folds per CTA measured slower: its staging is
// latency-bound, profiles/r02/kf_launches_r02t_warp_folds_rejected.txt)
constexpr int kKfFoldThreads = 256;

// One list-of-lists in SELL-8x32 layout: slice s holds 32 rows (perm[32 s + l]
// = row of lane l, -1 past the end); vector q (8 entries) of lane l is
// ent[ptr[s] + 32 q + l]; the slice's width in vectors is (ptr[s+1]-ptr[s])/32.
struct KfList {
    const int32_t* ptr = nullptr;
    const int32_t* perm = nullptr;
    const uint4* ent = nullptr;
    int nsl = 0;
    // rows longer than kKfLong entries (the strongest hands' Y rows: ~1,000
    // entries against ~100 typical), kept out of the slices: row id, first
    // vector, vector count, contiguous 16-byte vectors of 8 entries
    int nlong = 0;
    const int32_t* lrow = nullptr;
    const int32_t* lptr = nullptr;
    const uint4* lent = nullptr;
};

struct KfBoard {
    int m1, m2, n1, n2;
    int nAlive, fast;                 // fast: every λ2·S in [2^-100, 2^100] (or 0)
    int maxSa, maxSb;                 // largest S row / S column (shared-memory layout)
    int64_t rowOff, colOff;           // y / x offsets of the board
    int64_t zOff, zfOff;              // t / z buffer [n1][nAlive] and z_f buffer [n1] offsets
    int64_t h1Off, h2Off;             // first player-1 / player-2 hand over all boards (sequence-major inputs)
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
    const uint8_t* hasF;              // [n1]: F row d is a kept U/V column
    KfList yr;   // A x,  alive r -> (j, Y), j asc: byte offset of QY[v(Y)][j]        (Vᵀ rows)
    KfList b2;   // A x,  i -> blocked j asc: byte offset of the pair {λ2_j, x_j}      (Â rows)
    KfList b1;   // Aᵀy, j -> blocked i asc: byte offset of the pair {λ1_i, y_i}     (Âᵀ rows)
    KfList yc;   // Aᵀy, j -> (alive r, Y), r asc: byte offset of ZY[v(Y)][r]          (V rows)
                 // (b1 and yc share one row order: an AV row is Âᵀ then V, one sum)
};

// staged value admissible for the Y-factoring rewrite
__device__ __forceinline__ bool kf_ok(double v) {
    const double a = fabs(v);
    return a == 0.0 || (a >= 0x1p-900 && a <= 0x1p900);
}

// Y in {-2, -1, +1, +2} is stored as the variant index v in {0, 1, 2, 3}
__device__ __forceinline__ double kf_yval(int v) { return v < 2 ? double(v - 2) : double(v - 1); }

__device__ __forceinline__ double smd(const char* smb, uint32_t off) {
    KR_SMEM_CHECK(off, 8);
    return *reinterpret_cast<const double*>(smb + off);
}
__device__ __forceinline__ double2 smd2(const char* smb, uint32_t off) {
    KR_SMEM_CHECK(off, 16);
    return *reinterpret_cast<const double2*>(smb + off);
}

// Stream one lane's vectors of a slice (KR_KF_DEPTH loads in flight),
// calling f(entry) for the 8 entries of each vector in order.
#ifndef KR_KF_DEPTH
#define KR_KF_DEPTH 2
#endif
template <class F>
__device__ __forceinline__ void kf_stream(const uint4* __restrict__ src, int nv, F&& f) {
    constexpr int D = KR_KF_DEPTH;
    const uint4 z = make_uint4(0, 0, 0, 0);
    uint4 c[D];
#pragma unroll
    for (int d = 0; d < D; ++d) c[d] = nv > d ? __ldg(src + 32 * d) : z;
    for (int q = 0; q < nv; ++q) {
        const uint4 cur = c[0];
#pragma unroll
        for (int d = 0; d + 1 < D; ++d) c[d] = c[d + 1];
        c[D - 1] = q + D < nv ? __ldg(src + 32 * (q + D)) : z;
        f(cur.x & 0xFFFFu);
        f(cur.x >> 16);
        f(cur.y & 0xFFFFu);
        f(cur.y >> 16);
        f(cur.z & 0xFFFFu);
        f(cur.z >> 16);
        f(cur.w & 0xFFFFu);
        f(cur.w >> 16);
    }
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
// Kernels.  Per product direction: the output-row kernels (one warp per SELL
// slice of 32 rows, all rows of a board's sequence over a few CTAs that stage
// the columns they gather from in shared memory) and one kernel of ordered
// folds (the chain solves and the long F rows / columns: one warp per fold).
//   A x : k_kfa_vt (Vᵀ rows -> t) ; k_kfa_fold (chains t -> z, F rows -> z_f) ;
//         k_kfa_ua ([U | Â] rows -> y)
//   Aᵀy : k_kft_fold (Uᵀ rows + backward chains -> z, F columns -> z_f) ;
//         k_kft_av ([Âᵀ | V] rows -> x)
// t / z live in a per-board [sequence][alive rank] buffer, z_f in [sequence].
//
// Shared-memory layouts (bytes); list entries address the first 64 KB:
//   k_kfa_vt : QY[maxSa][4][m2+1]  (Y·Q for Y = -2, -1, +1, +2; slot m2 = 0) | long-row buffers
//   k_kfa_ua : PR[m2+1] {λ2_j, x[j, col(F_a,0)]} | xF[nFa-1][m2]
//   k_kft_av : PR[m1+1] {λ1_i, y[i, row(F_b,0)]} | ZY[maxSb][4][nA+1] | yF[nFb-1][m1]
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ size_t kf_vt_bytes(int m2, int maxSa, int warps) {
    const size_t S = size_t(maxSa > 0 ? maxSa : 1);
    return 32 * (size_t(m2) + 1) * S + 8 * 256 * S * size_t(warps);   // QY | long-row buffers
}
__host__ __device__ __forceinline__ size_t kf_ua_bytes(int m2, int maxFa) {
    return 16 * (size_t(m2) + 1) + 8 * size_t(m2) * size_t(maxFa > 1 ? maxFa - 1 : 0);
}
__host__ __device__ __forceinline__ size_t kf_av_bytes(int m1, int nA, int maxSb, int maxFb) {
    return 16 * (size_t(m1) + 1) + 32 * (size_t(nA) + 1) * size_t(maxSb > 0 ? maxSb : 1) +
           8 * size_t(m1) * size_t(maxFb > 1 ? maxFb - 1 : 0);
}

// Ordered left fold of v[0..n) (DESC: v[n-1] down to v[0]) by ONE thread
// from shared memory: acc = v + acc is the only dependency chain.  Whole
// batches of 16 are loaded first and added without predicates, which keeps
// the loop at the DADD latency (tools/fold_bench.cu: 9.8 cycles per element
// against 26 for a predicated double-buffered loop).  With out != nullptr
// the running sum after each element is stored there (the chain solves: z in
// place of t).  Returns the final sum.
template <bool DESC>
__device__ __forceinline__ double kf_fold(double* v, int n, double acc, bool store) {
    int k0 = 0;
    for (; k0 + 16 <= n; k0 += 16) {
        double t[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = v[DESC ? n - 1 - k0 - u : k0 + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            acc = t[u] + acc;
            if (store) v[DESC ? n - 1 - k0 - u : k0 + u] = acc;
        }
    }
    for (; k0 < n; ++k0) {
        acc = v[DESC ? n - 1 - k0 : k0] + acc;
        if (store) v[DESC ? n - 1 - k0 : k0] = acc;
    }
    return acc;
}

// ---- input transpose -------------------------------------------------------
// The row kernels stage whole input columns (one sequence, every hand of a
// board); a sequence-major copy of the input, out[s M + J] = in[J n + s] over
// all boards' hands J (hands [J0, J1) of a board-group launch), makes those
// loads contiguous.  32 hands per block through shared memory: both the loads
// (32 n contiguous doubles) and the stores (32 per sequence) are coalesced.
__global__ void __launch_bounds__(256) k_kf_seqmajor(const double* __restrict__ in, int64_t M, int n, int64_t J0,
                                                     int64_t J1, double* __restrict__ out) {
    pdl_entry();
    extern __shared__ double tile[];  // [32][n]
    const int64_t h0 = J0 + int64_t(blockIdx.x) * 32;
    const int nh = int(lmin(32, J1 - h0));
    if (nh <= 0) return;
    KR_SMEM_CHECK(0, size_t(8) * 32 * n);
    for (int q = threadIdx.x; q < nh * n; q += blockDim.x) tile[q] = in[h0 * n + q];
    __syncthreads();
    for (int q = threadIdx.x; q < n * 32; q += blockDim.x) {
        const int s = q >> 5, l = q & 31;
        if (l < nh) out[int64_t(s) * M + h0 + l] = tile[l * n + s];
    }
}

// Slices [lo, hi) of CTA g out of gs for a list of nsl slices (balanced).
__device__ __forceinline__ void kf_range(int g, int gs, int nsl, int& lo, int& hi) {
    lo = int(int64_t(g) * nsl / gs);
    hi = int(int64_t(g + 1) * nsl / gs);
}

// ---- A x -------------------------------------------------------------------
// One Vᵀ entry's terms added to acc in order (S entries of the row), for rows
// with several S entries or inputs outside the rewrite's premise (literal
// expressions of rows_vt); kept out of line so the common path stays lean.
// xs: the board's sequence-major input, column c at xs + c * M2.
__device__ __noinline__ double kf_vt_add(const KfBoard& B, const char* smb, const double* xs, int64_t M2,
                                         uint32_t off, int s0, int nSa, int m2p, bool fast, double acc) {
    if (fast) {
        for (int e = 0; e < nSa; ++e) acc = acc + smd(smb, off + uint32_t(e) * 32u * uint32_t(m2p));
        return acc;
    }
    const int q = int(off >> 3), v = q / m2p, j = q - v * m2p;
    if (j >= B.m2) return acc;
    const double scale = B.l2[j] * kf_yval(v);
    for (int e = 0; e < nSa; ++e) acc = acc + (scale * B.sval[s0 + e]) * xs[B.scol[s0 + e] * M2 + j];
    return acc;
}
// The terms of 8 entries (one vector), in order, into o[8 * nSa].
__device__ __noinline__ void kf_vt_terms8(const KfBoard& B, const char* smb, const double* xs, int64_t M2, uint4 c,
                                          int s0, int nSa, int m2p, bool fast, double* o) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    for (int u = 0; u < 8; ++u) {
        const uint32_t off = u & 1 ? w[u >> 1] >> 16 : w[u >> 1] & 0xFFFFu;
        if (fast) {
            for (int e = 0; e < nSa; ++e) o[u * nSa + e] = smd(smb, off + uint32_t(e) * 32u * uint32_t(m2p));
            continue;
        }
        const int q = int(off >> 3), v = q / m2p, j = q - v * m2p;
        if (j >= B.m2) {
            for (int e = 0; e < nSa; ++e) o[u * nSa + e] = 0.0;
            continue;
        }
        const double scale = B.l2[j] * kf_yval(v);
        for (int e = 0; e < nSa; ++e) o[u * nSa + e] = (scale * B.sval[s0 + e]) * xs[B.scol[s0 + e] * M2 + j];
    }
}

// Vᵀ rows of chain a: t(r) = Σ_j↑ Σ_e ((λ2_j·Y)·S_e)·x[j, col_e]  (rows_vt).
// CTAs g < gs take a balanced range of slices (warps loop over them); CTA gs
// takes the long rows, one warp per row: each round the 32 lanes load 256
// entries, produce their terms in order into the warp's buffer, and all lanes
// add them in order (warp-uniform adds).  xT: sequence-major input.
template <int W>
__global__ void __launch_bounds__(32 * W, 32 / W) k_kfa_vt(const KfBoard* __restrict__ boards, int b0, int gy, int gs,
                                                            const double* __restrict__ xT, int64_t M2,
                                                            double* __restrict__ tz) {
    pdl_entry();
    extern __shared__ __align__(16) double sm[];
    const char* smb = reinterpret_cast<const char*>(sm);
    __shared__ int okAll;
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int a = blockIdx.x / gy, g = blockIdx.x - a * gy;
    const int s0 = B.sptr[a], nSa = B.sptr[a + 1] - s0;
    const int nA = B.nAlive, m2 = B.m2, m2p = m2 + 1;
    const bool longCta = g == gs;
    int lo = 0, hi = 0;
    if (!longCta) kf_range(g, gs, B.yr.nsl, lo, hi);
    if (nSa == 0 || nA == 0 || (longCta ? B.yr.nlong == 0 : lo >= hi)) return;
    const double* xs = xT + B.h2Off;
    if (threadIdx.x == 0) okAll = 1;
    __syncthreads();
    int ok = B.fast;
    KR_DCHECK(nSa <= B.maxSa && m2 <= M2);
    KR_SMEM_CHECK(0, size_t(32) * m2p * nSa);
    for (int e = 0; e < nSa; ++e) {
        KR_DCHECK(unsigned(B.scol[s0 + e]) < unsigned(B.n2));
        double* QY = sm + size_t(e) * 4 * m2p;
        const double* col = xs + B.scol[s0 + e] * M2;
        const double sv = B.sval[s0 + e];
        for (int j = threadIdx.x; j < m2p; j += 32 * W) {
            double q = 0.0;
            if (j < m2) {
                const double xv = col[j];
                ok &= kf_ok(xv);
                q = (B.l2[j] * sv) * xv;
            }
            QY[j] = -2.0 * q;   // exact scalings (premise checked below)
            QY[m2p + j] = -q;
            QY[2 * m2p + j] = q;
            QY[3 * m2p + j] = 2.0 * q;
        }
    }
    if (!ok) okAll = 0;
    __syncthreads();
    const bool fast = okAll != 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (longCta) {
        double* buf = sm + size_t(4) * m2p * size_t(B.maxSa) + size_t(warp) * 256 * size_t(B.maxSa);
        KR_SMEM_CHECK(8 * (size_t(4) * m2p * B.maxSa + (size_t(warp) + 1) * 256 * B.maxSa), 0);
        for (int L = warp; L < B.yr.nlong; L += W) {
            const int v0 = B.yr.lptr[L], nvec = B.yr.lptr[L + 1] - v0;
            double acc = 0.0;
            for (int q0 = 0; q0 < nvec; q0 += 32) {
                const int cnt = min(32, nvec - q0);
                __syncwarp();
                if (lane < cnt) {
                    const uint4 c = __ldg(B.yr.lent + v0 + q0 + lane);
                    double* o = buf + size_t(lane) * 8 * nSa;
                    if (fast && nSa == 1) {
                        o[0] = smd(smb, c.x & 0xFFFFu);
                        o[1] = smd(smb, c.x >> 16);
                        o[2] = smd(smb, c.y & 0xFFFFu);
                        o[3] = smd(smb, c.y >> 16);
                        o[4] = smd(smb, c.z & 0xFFFFu);
                        o[5] = smd(smb, c.z >> 16);
                        o[6] = smd(smb, c.w & 0xFFFFu);
                        o[7] = smd(smb, c.w >> 16);
                    } else {
                        kf_vt_terms8(B, smb, xs, M2, c, s0, nSa, m2p, fast, o);
                    }
                }
                __syncwarp();
                const int nt = cnt * 8 * nSa;
                for (int k = 0; k < nt; ++k) acc = acc + buf[k];
            }
            KR_DCHECK(unsigned(B.yr.lrow[L]) < unsigned(nA));
            if (lane == 0) tz[B.zOff + int64_t(a) * nA + B.yr.lrow[L]] = acc;
        }
        return;
    }
    for (int s = lo + warp; s < hi; s += W) {
        const int p0 = B.yr.ptr[s], nv = (B.yr.ptr[s + 1] - p0) >> 5;
        const int r = B.yr.perm[32 * s + lane];
        const uint4* src = B.yr.ent + p0 + lane;
        double acc = 0.0;
        if (fast && nSa == 1) {
            kf_stream(src, nv, [&](uint32_t off) { acc = acc + smd(smb, off); });
        } else {
            kf_stream(src, nv, [&](uint32_t off) { acc = kf_vt_add(B, smb, xs, M2, off, s0, nSa, m2p, fast, acc); });
        }
        KR_DCHECK(r < nA);
        if (r >= 0) tz[B.zOff + int64_t(a) * nA + r] = acc;
    }
}

// The ordered folds of A x for player-1 sequence a: all threads stage the
// fold inputs in shared memory, then thread 0 runs the chain solve
// (z(r) = t(r) + z(r-1), engine.hpp:31-41) and thread 32 the F row
// t_f(a) = Σ_j↑ Σ_e (λ2_j·F_e)·x[j, col_e] (rows_vt), side by side.
// shared: v[nAlive] | f[m2 · nFa]
__global__ void __launch_bounds__(kKfFoldThreads) k_kfa_fold(const KfBoard* __restrict__ boards, int b0,
                                                              const double* __restrict__ xT, int64_t M2,
                                                              double* __restrict__ tz, double* __restrict__ zf) {
    pdl_entry();
    extern __shared__ __align__(16) double sm[];
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int a = blockIdx.x;
    const int nA = B.nAlive, m2 = B.m2;
    const bool chain = B.sptr[a + 1] > B.sptr[a] && nA > 0;
    const bool fA = B.hasF[a] != 0;
    if (!chain && !fA) return;
    const int f0 = B.fptr[a], nFa = B.fptr[a + 1] - f0;
    double* v = sm;
    double* f = sm + nA;
    double* t = tz + B.zOff + int64_t(a) * nA;
    const double* xs = xT + B.h2Off;
    KR_SMEM_CHECK(0, 8 * (size_t(nA) + size_t(fA ? m2 : 0) * nFa));
    if (chain)
        for (int r = threadIdx.x; r < nA; r += kKfFoldThreads) v[r] = t[r];
    if (fA)
        for (int k = threadIdx.x; k < m2 * nFa; k += kKfFoldThreads) {
            const int j = nFa == 1 ? k : k / nFa, e = k - j * nFa;
            KR_DCHECK(unsigned(B.fcol[f0 + e]) < unsigned(B.n2));
            f[k] = (B.l2[j] * B.fval[f0 + e]) * xs[B.fcol[f0 + e] * M2 + j];
        }
    __syncthreads();
    if (threadIdx.x == 0 && chain) kf_fold<false>(v, nA, -0.0, true);
    if (threadIdx.x == 32 && fA) zf[B.zfOff + a] = kf_fold<false>(f, m2 * nFa, 0.0, false);
    __syncthreads();
    if (chain)
        for (int r = threadIdx.x; r < nA; r += kKfFoldThreads) t[r] = v[r];
}

// [U | Â] rows (i, a): λ1_i·z(prev alive(i), a) + λ1_i·z_f(a), then the
// blocked hands j ascending: ((−λ1_i)·λ2_j·F_e)·x[j, col_e]  (rows_ua)
template <int W>
__global__ void __launch_bounds__(32 * W) k_kfa_ua(const KfBoard* __restrict__ boards, int b0, int gu,
                                                    const double* __restrict__ xT, int64_t M2,
                                                    const double* __restrict__ tz, const double* __restrict__ zf,
                                                    double* __restrict__ y) {
    pdl_entry();
    extern __shared__ __align__(16) double sm[];
    const char* smb = reinterpret_cast<const char*>(sm);
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int a = blockIdx.x / gu, g = blockIdx.x - a * gu;
    int lo, hi;
    kf_range(g, gu, B.b2.nsl, lo, hi);
    if (lo >= hi) return;
    const int m2 = B.m2, n1 = B.n1, nA = B.nAlive;
    const int f0 = B.fptr[a], nFa = B.fptr[a + 1] - f0;
    double2* PR = reinterpret_cast<double2*>(sm);
    double* xF1 = sm + 2 * (m2 + 1);
    KR_SMEM_CHECK(0, 8 * (2 * (size_t(m2) + 1) + size_t(nFa > 1 ? nFa - 1 : 0) * m2));
    if (nFa > 0) {
        const double* xs = xT + B.h2Off;
        const double* c0 = xs + B.fcol[f0] * M2;
        for (int j = threadIdx.x; j <= m2; j += 32 * W) {
            if (j == m2) {
                PR[m2] = make_double2(0.0, 0.0);
                continue;
            }
            PR[j] = make_double2(B.l2[j], c0[j]);
            for (int e = 1; e < nFa; ++e) xF1[size_t(e - 1) * m2 + j] = xs[B.fcol[f0 + e] * M2 + j];
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool chain = B.sptr[a + 1] > B.sptr[a] && nA > 0;
    const bool fA = B.hasF[a] != 0;
    const double zfa = fA ? zf[B.zfOff + a] : 0.0;
    const double fv = nFa > 0 ? B.fval[f0] : 0.0;
    for (int s = lo + warp; s < hi; s += W) {
        const int i = B.b2.perm[32 * s + lane];
        KR_DCHECK(i < B.m1);
        const double v = i >= 0 ? B.l1[i] : 0.0;
        double acc = 0.0;
        if (i >= 0 && v != 0.0) {
            const int rp = B.rankPrev[i];
            KR_DCHECK(rp < nA);
            if (chain && rp >= 0) acc = acc + v * tz[B.zOff + int64_t(a) * nA + rp];
            if (fA) acc = acc + v * zfa;
        }
        if (nFa > 0) {
            const int p0 = B.b2.ptr[s], nv = (B.b2.ptr[s + 1] - p0) >> 5;
            const uint4* src = B.b2.ent + p0 + lane;
            const double nv1 = -v;
            if (nFa == 1) {
                kf_stream(src, nv, [&](uint32_t off) {
                    const double2 p = smd2(smb, off);
                    const double w = (nv1 * p.x) * fv;
                    acc = acc + w * p.y;
                });
            } else {
                kf_stream(src, nv, [&](uint32_t off) {
                    const int j = int(off >> 4);
                    if (j >= m2) return;
                    const double scale = nv1 * PR[j].x;
                    for (int e = 0; e < nFa; ++e) {
                        const double w = scale * B.fval[f0 + e];
                        acc = acc + w * (e == 0 ? PR[j].y : xF1[size_t(e - 1) * m2 + j]);
                    }
                });
            }
        }
        if (i >= 0) y[B.rowOff + int64_t(i) * n1 + a] = acc;
    }
}

// ---- Aᵀ y ------------------------------------------------------------------
// The ordered folds of Aᵀy for player-1 sequence d: all threads compute the
// Uᵀ rows of chain d, s(r) = Σ_{i ∈ [alive r, alive r+1)} λ1_i·y[i, d], and
// the F-column terms λ1_i·y[i, d] (rows_ut) into shared memory; thread 0 then
// solves the chain backward (z(r) = s(r) + z(r+1), engine.hpp:44-54) and
// thread 32 folds the F column Σ_i↑, side by side.  yT: sequence-major input.
// shared: v[nAlive] | f[m1]
__global__ void __launch_bounds__(kKfFoldThreads) k_kft_fold(const KfBoard* __restrict__ boards, int b0,
                                                              const double* __restrict__ yT, int64_t M1,
                                                              double* __restrict__ tz, double* __restrict__ zf) {
    pdl_entry();
    extern __shared__ __align__(16) double sm[];
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int d = blockIdx.x;
    const int nA = B.nAlive, m1 = B.m1;
    const bool chain = B.sptr[d + 1] > B.sptr[d] && nA > 0;
    const bool fD = B.hasF[d] != 0;
    if (!chain && !fD) return;
    const double* yd = yT + d * M1 + B.h1Off;
    double* v = sm;
    double* f = sm + nA;
    KR_SMEM_CHECK(0, 8 * (size_t(nA) + (fD ? m1 : 0)));
    if (chain)
        for (int r = threadIdx.x; r < nA; r += kKfFoldThreads) {
            KR_DCHECK(B.aliveRows[r] >= 0 && B.aliveEnd[r] <= m1);
            double acc = 0.0;
            for (int i = B.aliveRows[r]; i < B.aliveEnd[r]; ++i) acc = acc + B.l1[i] * yd[i];
            v[r] = acc;
        }
    if (fD)
        for (int i = threadIdx.x; i < m1; i += kKfFoldThreads) f[i] = B.l1[i] * yd[i];
    __syncthreads();
    if (threadIdx.x == 0 && chain) kf_fold<true>(v, nA, -0.0, true);
    if (threadIdx.x == 32 && fD) zf[B.zfOff + d] = kf_fold<false>(f, m1, 0.0, false);
    __syncthreads();
    if (chain) {
        double* z = tz + B.zOff + int64_t(d) * nA;
        for (int r = threadIdx.x; r < nA; r += kKfFoldThreads) z[r] = v[r];
    }
}

// [Âᵀ | V] rows (j, b): the blocked hands i ascending, ((−λ1_i)·λ2_j·F_e)·y[i, row_e];
// then V: alive r ascending, ((λ2_j·Y)·S_e)·z(r, row_e); then λ2_j·F_e·z_f  (rows_av)
template <int W>
__global__ void __launch_bounds__(32 * W) k_kft_av(const KfBoard* __restrict__ boards, int b0, int gv,
                                                    const double* __restrict__ yT, int64_t M1,
                                                    const double* __restrict__ tz, const double* __restrict__ zf,
                                                    double* __restrict__ x) {
    pdl_entry();
    extern __shared__ __align__(16) double sm[];
    const char* smb = reinterpret_cast<const char*>(sm);
    __shared__ int okAll;
    const KfBoard& B = boards[b0 + blockIdx.y];
    const int b = blockIdx.x / gv, g = blockIdx.x - b * gv;
    int lo, hi;
    kf_range(g, gv, B.b1.nsl, lo, hi);
    if (lo >= hi) return;
    const int m1 = B.m1, n2 = B.n2, nA = B.nAlive;
    const int m1p = m1 + 1, nAp = nA + 1;
    const int f0 = B.fcptr[b], nFb = B.fcptr[b + 1] - f0;
    const int s0 = B.scptr[b], nSb = B.scptr[b + 1] - s0;
    double2* PR = reinterpret_cast<double2*>(sm);
    double* ZY = sm + 2 * m1p;                                   // [maxSb][4][nAp]
    double* yF1 = ZY + size_t(4) * nAp * (B.maxSb > 0 ? B.maxSb : 1);
    const double* ys = yT + B.h1Off;
    KR_DCHECK(nSb <= (B.maxSb > 0 ? B.maxSb : 1) || nA == 0);
    KR_SMEM_CHECK(0, 8 * (2 * size_t(m1p) + size_t(4) * nAp * (B.maxSb > 0 ? B.maxSb : 1) +
                          size_t(nFb > 1 ? nFb - 1 : 0) * m1));
    if (threadIdx.x == 0) okAll = 1;
    __syncthreads();
    if (nFb > 0) {
        const double* c0 = ys + B.fcrow[f0] * M1;
        for (int i = threadIdx.x; i <= m1; i += 32 * W) {
            if (i == m1) {
                PR[m1] = make_double2(0.0, 0.0);
                continue;
            }
            PR[i] = make_double2(B.l1[i], c0[i]);
            for (int e = 1; e < nFb; ++e) yF1[size_t(e - 1) * m1 + i] = ys[B.fcrow[f0 + e] * M1 + i];
        }
    }
    int ok = B.fast;
    if (nA > 0)
        for (int e = 0; e < nSb; ++e) {
            KR_DCHECK(unsigned(B.scrow[s0 + e]) < unsigned(B.n1));
            const double* z = tz + B.zOff + int64_t(B.scrow[s0 + e]) * nA;
            double* Z = ZY + size_t(e) * 4 * nAp;
            for (int r = threadIdx.x; r < nAp; r += 32 * W) {
                const double v = r < nA ? z[r] : 0.0;
                ok &= kf_ok(v);
                Z[r] = -2.0 * v;
                Z[nAp + r] = -v;
                Z[2 * nAp + r] = v;
                Z[3 * nAp + r] = 2.0 * v;
            }
        }
    if (!ok) okAll = 0;
    __syncthreads();
    const bool zok = okAll != 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double fv = nFb > 0 ? B.fcval[f0] : 0.0;
    for (int s = lo + warp; s < hi; s += W) {
        const int j = B.b1.perm[32 * s + lane];
        KR_DCHECK(j < B.m2);
        const double l2 = j >= 0 ? B.l2[j] : 0.0;
        double acc = 0.0;
        if (nFb > 0) {   // Âᵀ
            const int p0 = B.b1.ptr[s], nv = (B.b1.ptr[s + 1] - p0) >> 5;
            const uint4* src = B.b1.ent + p0 + lane;
            if (nFb == 1) {
                kf_stream(src, nv, [&](uint32_t off) {
                    const double2 p = smd2(smb, off);
                    const double w = (-p.x * l2) * fv;
                    acc = acc + w * p.y;
                });
            } else {
                kf_stream(src, nv, [&](uint32_t off) {
                    const int i = int(off >> 4);
                    if (i >= m1) return;
                    const double scale = -PR[i].x * l2;
                    for (int e = 0; e < nFb; ++e) {
                        const double w = scale * B.fcval[f0 + e];
                        acc = acc + w * (e == 0 ? PR[i].y : yF1[size_t(e - 1) * m1 + i]);
                    }
                });
            }
        }
        if (nSb > 0 && nA > 0) {   // V, S columns
            const int p0 = B.yc.ptr[s], nv = (B.yc.ptr[s + 1] - p0) >> 5;
            const uint4* src = B.yc.ent + p0 + lane;
            if (zok && nSb == 1) {
                // ((λ2·Y)·S)·z == (λ2·S)·(Y·z): one multiply, one add
                const double P0 = l2 * B.scval[s0];
                kf_stream(src, nv, [&](uint32_t off) { acc = acc + P0 * smd(smb, off); });
            } else if (zok) {
                kf_stream(src, nv, [&](uint32_t off) {
                    for (int e = 0; e < nSb; ++e)
                        acc = acc + (l2 * B.scval[s0 + e]) * smd(smb, off + uint32_t(e) * 32u * uint32_t(nAp));
                });
            } else {
                kf_stream(src, nv, [&](uint32_t off) {
                    const int q = int(off >> 3) - 2 * m1p, v = q / nAp, r = q - v * nAp;
                    if (r >= nA) return;
                    const double scale = l2 * kf_yval(v);
                    for (int e = 0; e < nSb; ++e) {
                        const double w = scale * B.scval[s0 + e];
                        acc = acc + w * tz[B.zOff + int64_t(B.scrow[s0 + e]) * nA + r];
                    }
                });
            }
        }
        if (j >= 0) {
            if (l2 != 0.0)   // V, F columns
                for (int e = 0; e < nFb; ++e) {
                    const int d = B.fcrow[f0 + e];
                    if (B.hasF[d]) acc = acc + (l2 * B.fcval[f0 + e]) * zf[B.zfOff + d];
                }
            x[B.colOff + int64_t(j) * n2 + b] = acc;
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// SELL-8x32 list (KfList) on the host: rows in `order` (or by length,
// longest first), slices of 32, each slice padded to a multiple of 8 entries
// with `pad`; with longCut > 0, rows longer than longCut go to the long-row
// list instead (contiguous, padded to whole vectors).
struct HostList {
    std::vector<int32_t> ptr, perm, lrow, lptr;
    std::vector<uint16_t> ent, lent;   // 8 per uint4
    int nsl = 0;
    void build(const std::vector<std::vector<uint16_t>>& rows, uint16_t pad, const std::vector<int32_t>* order,
               size_t longCut = 0) {
        const int R = int(rows.size());
        std::vector<int32_t> ord;
        if (order) {
            ord = *order;
        } else {
            ord.resize(size_t(R));
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(),
                             [&](int32_t u, int32_t v) { return rows[size_t(u)].size() > rows[size_t(v)].size(); });
        }
        std::vector<int32_t> kept;
        lptr.assign(1, 0);
        for (int32_t r : ord) {
            if (longCut > 0 && rows[size_t(r)].size() > longCut) {
                lrow.push_back(r);
                const size_t nv = (rows[size_t(r)].size() + 7) / 8;
                lptr.push_back(lptr.back() + int32_t(nv));
                for (size_t k = 0; k < nv * 8; ++k) lent.push_back(k < rows[size_t(r)].size() ? rows[size_t(r)][k] : pad);
            } else {
                kept.push_back(r);
            }
        }
        if (lent.empty()) lent.assign(8, pad);
        const int K = int(kept.size());
        nsl = (K + 31) / 32;
        perm.assign(size_t(std::max(nsl, 1)) * 32, -1);
        for (int q = 0; q < K; ++q) perm[size_t(q)] = kept[size_t(q)];
        ptr.assign(size_t(nsl) + 1, 0);
        for (int sl = 0; sl < nsl; ++sl) {
            size_t w = 0;
            for (int l = 0; l < 32; ++l) {
                const int r = perm[size_t(32 * sl + l)];
                if (r >= 0) w = std::max(w, rows[size_t(r)].size());
            }
            ptr[size_t(sl) + 1] = ptr[size_t(sl)] + int32_t(32 * ((w + 7) / 8));
        }
        ent.assign(size_t(std::max(ptr.back(), 1)) * 8, pad);
        for (int sl = 0; sl < nsl; ++sl)
            for (int l = 0; l < 32; ++l) {
                const int r = perm[size_t(32 * sl + l)];
                if (r < 0) continue;
                const auto& row = rows[size_t(r)];
                for (size_t k = 0; k < row.size(); ++k)
                    ent[(size_t(ptr[size_t(sl)]) + 32 * (k / 8) + size_t(l)) * 8 + k % 8] = row[k];
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
// device enumerators of kr_devengine.cu follow; sparsify.hpp:246-406).  List
// entries are the kernels' shared-memory byte offsets (kf_ax_bytes /
// kf_atx_bytes layouts), so they depend on m1, m2 and the alive count.
void build_host_board(const kr_kron_board& K, int b, HostBoard& H) {
    const std::string at = "board " + std::to_string(b) + ": ";
    const int m1 = K.m1, m2 = K.m2, n1 = K.n1, n2 = K.n2;
    if (m1 < 1 || m2 < 1 || n1 < 1 || n2 < 1) throw Fail{KR_INVALID_INPUT, at + "empty board"};
    if (m1 > kKfMaxHands || m2 > kKfMaxHands)
        throw Fail{KR_INVALID_INPUT, at + "more than 1364 hands per side (use the factored engine)"};
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
    // Y rows (alive r -> j) and columns (j -> alive r), as (index, Y)
    std::vector<std::vector<std::pair<uint16_t, int8_t>>> yrl(static_cast<size_t>(H.nAlive)), ycl(static_cast<size_t>(m2));
    for (int r = 0; r < H.nAlive; ++r)
        for (uint16_t e : yrows[size_t(H.aliveRows[size_t(r)])]) {
            const int j = e & 0x7FF, yd = int(e >> 11) - 2;
            yrl[size_t(r)].push_back({uint16_t(j), int8_t(yd)});
            ycl[size_t(j)].push_back({uint16_t(r), int8_t(yd)});
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
    std::vector<std::vector<int>> b2i(static_cast<size_t>(m1));
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j)
            if (!compat(i, j)) b2i[size_t(i)].push_back(j);
    // byte offsets into the kernels' shared memory (see kf_ax_bytes / kf_atx_bytes)
    const int m1p = m1 + 1, m2p = m2 + 1, nAp = H.nAlive + 1;
    auto vidx = [](int yd) { return yd < 0 ? yd + 2 : yd + 1; };   // Y -> variant 0..3
    {
        std::vector<std::vector<uint16_t>> rows(static_cast<size_t>(H.nAlive));
        for (int r = 0; r < H.nAlive; ++r)
            for (auto [j, yd] : yrl[size_t(r)]) rows[size_t(r)].push_back(uint16_t((vidx(yd) * m2p + j) * 8));
        H.yr.build(rows, uint16_t((2 * m2p + m2) * 8), nullptr, kKfLong);
        for (int i = 0; i < m1; ++i)
            for (int j : b2i[size_t(i)]) b2[size_t(i)].push_back(uint16_t(16 * j));
        H.b2.build(b2, uint16_t(16 * m2), nullptr);
    }
    {
        std::vector<std::vector<uint16_t>> yc(static_cast<size_t>(m2));
        for (int i = 0; i < m1; ++i)
            for (int j : b2i[size_t(i)]) b1[size_t(j)].push_back(uint16_t(16 * i));
        for (int j = 0; j < m2; ++j)
            for (auto [r, yd] : ycl[size_t(j)]) yc[size_t(j)].push_back(uint16_t(16 * m1p + (vidx(yd) * nAp + r) * 8));
        // one row order for both (an AV row is its Âᵀ part then its V part)
        std::vector<int32_t> ord(static_cast<size_t>(m2));
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t u, int32_t v) {
            return b1[size_t(u)].size() + yc[size_t(u)].size() > b1[size_t(v)].size() + yc[size_t(v)].size();
        });
        H.b1.build(b1, uint16_t(16 * m1), &ord);
        H.yc.build(yc, uint16_t(16 * m1p + (2 * nAp + H.nAlive) * 8), &ord);
    }
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
        for (auto [j, yd] : yrl[size_t(r)]) {
            const double scale = H.l2[size_t(j)] * double(yd);
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
            for (int j : b2i[size_t(i)]) {
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
    l.perm = up(keep, h.perm);
    uint4* e = dev_alloc<uint4>(int64_t(h.ent.size() / 8));
    keep.push_back(e);
    KR_CK(cudaMemcpy(e, h.ent.data(), 2 * h.ent.size(), cudaMemcpyHostToDevice));
    l.ent = e;
    l.nsl = h.nsl;
    l.nlong = int(h.lrow.size());
    l.lrow = up(keep, h.lrow);
    l.lptr = up(keep, h.lptr);
    uint4* le = dev_alloc<uint4>(int64_t(h.lent.size() / 8));
    keep.push_back(le);
    KR_CK(cudaMemcpy(le, h.lent.data(), 2 * h.lent.size(), cudaMemcpyHostToDevice));
    l.lent = le;
    return l;
}

}  // namespace

struct KfState {
    KfBoard* dBoards = nullptr;    // device array
    std::vector<void*> keep;       // every device table
    size_t smVT = 0, smUA = 0, smAV = 0, smFA = 0, smFT = 0;
    int nb = 0, n1 = 0, n2 = 0;
    int gy = 1, gs = 0, gu = 1, gv = 1;    // row-kernel CTAs per sequence (gs: slice CTAs of the Vᵀ rows)
    double* tz[2] = {nullptr, nullptr};   // t / z per direction (A x, Aᵀy may run concurrently)
    double* zf[2] = {nullptr, nullptr};
    double* inT[2] = {nullptr, nullptr};  // sequence-major input per direction
    int64_t M1 = 0, M2 = 0;               // hands of each player over all boards
    std::vector<int64_t> hOff1, hOff2;    // per board (+ total)
};

void kf_destroy(KfState* k) {
    if (!k) return;
    for (void* p : k->keep) krb::dev_free(p);
    delete k;
}

// Boards [b0, b1) of one product: the input made sequence-major, then
// A x = Vᵀ rows, folds, [U|Â] rows; Aᵀy = folds (Uᵀ rows and chains), [Âᵀ|V] rows.
// The engine's staging layout: the input sequence-major over all of the
// direction's hands, out[s M + J] = in[J n + s] (hands [J0, J1)).
void kf_stage(kr_engine* e, int dir, const double* in, double* inT, int64_t J0, int64_t J1, cudaStream_t s) {
    KfState* k = e->kf;
    const int64_t M = dir == 0 ? k->M2 : k->M1;
    const int n = dir == 0 ? k->n2 : k->n1;
    if (J1 <= J0) return;
    krb::launch(k_kf_seqmajor, unsigned((J1 - J0 + 31) / 32), 256, size_t(32) * n * sizeof(double), s, in, M, n, J0, J1,
                inT);
    KR_CK_LAUNCH();
    e->launches++;
}

void kf_kernels(kr_engine* e, int dir, const double* inT, double* out, cudaStream_t s, int b0, int b1);

void kf_product(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0, int b1) {
    KfState* k = e->kf;
    if (b1 < 0) b1 = k->nb;
    if (b1 <= b0) return;
    const int64_t J0 = (dir == 0 ? k->hOff2 : k->hOff1)[size_t(b0)], J1 = (dir == 0 ? k->hOff2 : k->hOff1)[size_t(b1)];
    kf_stage(e, dir, in, k->inT[dir], J0, J1, s);
    kf_kernels(e, dir, k->inT[dir], out, s, b0, b1);
}

// The products on an input already in the staging layout (the DCFR solver
// writes its strategies that way: no transpose per product).
void kf_product_staged(kr_engine* e, int dir, const double* inT, double* out, cudaStream_t s) {
    kf_kernels(e, dir, inT, out, s, 0, e->kf->nb);
}

void kf_stage_all(kr_engine* e, int dir, const double* in, double* inT, cudaStream_t s) {
    KfState* k = e->kf;
    kf_stage(e, dir, in, inT, 0, (dir == 0 ? k->hOff2 : k->hOff1)[size_t(k->nb)], s);
}

void kf_kernels(kr_engine* e, int dir, const double* inT, double* out, cudaStream_t s, int b0, int b1) {
    KfState* k = e->kf;
    const unsigned nb = unsigned(b1 - b0);
    constexpr int T = 32 * kKfWarps;
    const int64_t M = dir == 0 ? k->M2 : k->M1;
    if (dir == 0) {
        krb::launch(k_kfa_vt<kKfWarps>, dim3(unsigned(k->n1 * k->gy), nb), T, k->smVT, s, k->dBoards, b0, k->gy, k->gs,
                    inT, M, k->tz[0]);
        KR_CK_LAUNCH();
        krb::launch(k_kfa_fold, dim3(unsigned(k->n1), nb), kKfFoldThreads, k->smFA, s, k->dBoards, b0, inT, M, k->tz[0],
                    k->zf[0]);
        KR_CK_LAUNCH();
        krb::launch(k_kfa_ua<kKfWarps>, dim3(unsigned(k->n1 * k->gu), nb), T, k->smUA, s, k->dBoards, b0, k->gu, inT,
                    M, k->tz[0], k->zf[0], out);
        KR_CK_LAUNCH();
        e->launches += 3;
    } else {
        krb::launch(k_kft_fold, dim3(unsigned(k->n1), nb), kKfFoldThreads, k->smFT, s, k->dBoards, b0, inT, M, k->tz[1],
                    k->zf[1]);
        KR_CK_LAUNCH();
        krb::launch(k_kft_av<kKfWarps>, dim3(unsigned(k->n2 * k->gv), nb), T, k->smAV, s, k->dBoards, b0, k->gv, inT,
                    M, k->tz[1], k->zf[1], out);
        KR_CK_LAUNCH();
        e->launches += 2;
    }
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
        k.n1 = n1;
        k.n2 = n2;
        std::vector<KfBoard> db(static_cast<size_t>(nb));
        int64_t rowOff = 0, colOff = 0, K = 0, zOff = 0;
        int slY = 0, slB2 = 0, slB1 = 0;
        bool anyLong = false;
        for (int b = 0; b < nb; ++b) {
            HostBoard& H = hb[size_t(b)];
            KfBoard& B = db[size_t(b)];
            B.m1 = H.m1;
            B.m2 = H.m2;
            B.n1 = n1;
            B.n2 = n2;
            B.nAlive = H.nAlive;
            B.fast = H.fast;
            B.maxSa = H.maxSa;
            B.maxSb = H.maxSb;
            B.rowOff = rowOff;
            B.colOff = colOff;
            B.h1Off = k.M1;
            B.h2Off = k.M2;
            k.hOff1.push_back(k.M1);
            k.hOff2.push_back(k.M2);
            k.M1 += H.m1;
            k.M2 += H.m2;
            B.zOff = zOff;
            B.zfOff = int64_t(b) * n1;
            zOff += int64_t(n1) * H.nAlive;
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
            k.smVT = std::max(k.smVT, kf_vt_bytes(H.m2, H.maxSa, kKfWarps));
            anyLong |= H.yr.lrow.size() > 0;
            k.smUA = std::max(k.smUA, kf_ua_bytes(H.m2, H.maxFa));
            k.smAV = std::max(k.smAV, kf_av_bytes(H.m1, H.nAlive, H.maxSb, H.maxFb));
            k.smFA = std::max(k.smFA, 8 * (size_t(H.nAlive) + size_t(H.m2) * size_t(std::max(H.maxFa, 1))));
            k.smFT = std::max(k.smFT, 8 * (size_t(H.nAlive) + size_t(H.m1)));
            slY = std::max(slY, H.yr.nsl);
            slB2 = std::max(slB2, H.b2.nsl);
            slB1 = std::max(slB1, H.b1.nsl);
            e->nnzA += H.nnzA;
            e->nnzU += H.nnzU;
            e->nnzV += H.nnzV;
            e->nnzM += H.nnzM;
            K += H.K;
        }
        e->k = K;
        e->flops_per_product = e->nnzV + e->nnzU + e->nnzA + (e->nnzM - K);
        const size_t limit = 227 * 1024 - 1024;
        if (k.smVT > limit || k.smUA > limit || k.smAV > limit || k.smFA > limit || k.smFT > limit)
            throw Fail{KR_INVALID_INPUT, "board too large for the Kronecker-factored engine's shared memory"};
        raise_smem_limit(k_kfa_vt<kKfWarps>, k.smVT);
        raise_smem_limit(k_kfa_ua<kKfWarps>, k.smUA);
        raise_smem_limit(k_kft_av<kKfWarps>, k.smAV);
        raise_smem_limit(k_kfa_fold, k.smFA);
        raise_smem_limit(k_kft_fold, k.smFT);
        raise_smem_limit(k_kf_seqmajor, size_t(32) * std::max(n1, n2) * sizeof(double));
        k.hOff1.push_back(k.M1);
        k.hOff2.push_back(k.M2);
        // CTAs per sequence: one slice per warp, or several rounds of slices
        // per CTA when the grid would exceed ~6 waves (fewer CTAs stage the
        // same input columns); slices spread evenly (kf_range).  Rounds
        // capped at 8 for the A x row kernels and 2 for A^T y's (config 3,
        // one box: A x 310 -> 306 us from 4 to 8, A^T y 351 -> 347 from 4 to
        // 2; KR_KF_ROUNDS_A / KR_KF_ROUNDS_T override)
        auto ctas = [&](int slices, int seqs, const char* env, int capDefault) {
            const int base = (slices + kKfWarps - 1) / kKfWarps;
            const int64_t total = int64_t(base) * seqs * nb;
            const char* re = std::getenv(env);
            const int64_t cap = re ? std::max(1, std::atoi(re)) : capDefault;
            const int rounds = int(std::min<int64_t>(cap, std::max<int64_t>(1, total / (6 * 148))));
            return std::max(1, (slices + kKfWarps * rounds - 1) / (kKfWarps * rounds));
        };
        k.gs = slY > 0 ? ctas(slY, n1, "KR_KF_ROUNDS_A", 8) : 0;
        k.gy = k.gs + (anyLong ? 1 : 0);
        if (k.gy == 0) k.gy = 1;
        k.gu = ctas(slB2, n1, "KR_KF_ROUNDS_A", 8);
        k.gv = ctas(slB1, n2, "KR_KF_ROUNDS_T", 2);
        for (int d = 0; d < 2; ++d) {
            k.inT[d] = dev_alloc<double>(std::max<int64_t>(d == 0 ? C : R, 1));
            k.keep.push_back(k.inT[d]);
            k.tz[d] = dev_alloc<double>(std::max<int64_t>(zOff, 1));
            k.zf[d] = dev_alloc<double>(int64_t(nb) * n1);
            k.keep.push_back(k.tz[d]);
            k.keep.push_back(k.zf[d]);
        }
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
