// kr_kron.cu — the implicit Kronecker engine.
//
// The payoff of one river board is A = Σ_ij π_ij (F + W_ij S) ⊗ e_i e_jᵀ with
// π_ij = λ1_i λ2_j [hands i, j disjoint] and W_ij = sign(key1_i − key2_j)
// (kron.hpp:104-132; referenceMatvec / referenceMatvecT, kron.hpp:211-254).
// Nothing of A is materialised.  For an output hand i on side O (player 1
// for A x, player 2 for Aᵀ y), summing over the hands j of side Σ:
//
//   out[i·n_O + a] = λ_O(i) · ( Σ_{j disj i} WF_j[a]  +  σ Σ_{j disj i} W_ij WS_j[a] )
//   WF_j[a] = λ_Σ(j) (F_d v_j)[a],   WS_j[a] = λ_Σ(j) (S_d v_j)[a]
//
// with F_d = F (A x) or Fᵀ (Aᵀ y), σ = +1 (A x) or −1 (Aᵀ y).  Hands of each
// side are strength-sorted ascending, so "key_j < key_i" is a prefix of the
// summing side: the W-weighted sum is (prefix below) − (suffix above), and
// the disjointness constraint is inclusion–exclusion over the two cards of i
// (all − hands holding c1 − hands holding c2 + the hand holding both), each
// card list again strength-sorted so its part is a prefix of the list.
//
// One fused kernel per product, one CTA per (sequence a, board b); every
// intermediate lives in shared memory (≈ 5 m_Σ doubles + 2 m_Σ ints):
//   1. wf[j], ws[j] for every summing hand j (gathers of v, L2-resident)
//   2. one block scan giving the prefix of ws in strength order, the prefix
//      of ws inside each of the 52 card lists, TF = Σ wf and the per-card
//      sums CF[c] of wf (see k_kron_fused)
//   3. every output hand i of the board: out = λ_O (TF − CF[c1] − CF[c2]
//      + wf[dup] + σ (lower − upper)), lookups from a 16-byte per-hand table
// so HBM sees only v, the output, and the small per-board tables.  The
// lookups (key ranks lt / le, their per-card-list counterparts, the
// duplicate-hand index) depend only on the keys and are built once on the
// host at create time.  Results equal referenceMatvec(T) up to rounding
// (different summation order): tests hold them to 1e-12 normwise.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kr_common.cuh"

namespace krb {

namespace {

constexpr int kCards = 52;
#ifndef KR_K7_THREADS
#define KR_K7_THREADS 256
#endif
constexpr int kThreads = KR_K7_THREADS;  // threads per CTA (compile-time: A/B builds)

// Lookup table of one output hand, packed in 16 bytes (positions in the
// kernel's virtual prefix array; list starts and ends come from the staged
// list pointers):
//   x = lt | le << 16          (ranks of the hand's key on the summing side)
//   y = (dup + 1) | c1 << 16 | c2 << 24
//   z = p1lt | p1le << 16      (m + the same ranks inside the list of c1)
//   w = p2lt | p2le << 16      (m + ... inside the list of c2)
// Hands per side per board are at most C(52,2) = 1326, so 3 m < 2^16.
constexpr int kMaxHands = 1536;            // hands per side and board; a thread takes kMaxHands / T
constexpr bool kKronSeqDefault = false;    // KR_KRON_SEQ, see kron_seq_major
constexpr int64_t kSmallGrid = 148;        // K7 grids up to this many CTAs run 512-thread CTAs
constexpr int kScanT = 256;                // block-scan chunks (fixed: bits independent of the CTA size)
static_assert(kMaxHands % 512 == 0, "512-thread K7 CTAs");

// Device view of one direction (0: A x, 1: Aᵀ y).
struct KronDir {
    int nO = 0, nS = 0, nb = 0, sign = 1;
    int64_t mO = 0, mS = 0;
    int maxMS = 0;
    int maxMO = 0;
    int64_t* sumOff = nullptr;    // [nb+1] global summing-hand offsets
    int64_t* outOff = nullptr;    // [nb+1] global output-hand offsets
    double* lamS = nullptr;       // [mS]
    double* lamO = nullptr;       // [mO]
    int64_t* fptr = nullptr;      // [nb*(nO+1)] global positions into fcol/fval
    int32_t* fcol = nullptr;
    double* fval = nullptr;
    int64_t* sptr = nullptr;
    int32_t* scol = nullptr;
    double* sval = nullptr;
    int32_t* listPtr = nullptr;   // [nb*53] offsets in the board's card-list space
    int64_t* listBase = nullptr;  // [nb] base of the board's lists in listHands
    int32_t* listHands = nullptr; // local summing-hand ids, list-major, ascending
    int4* otab = nullptr;         // [mO] packed lookups
    int64_t flops = 0;
};

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Dynamic shared memory for a board of maxMS summing hands: (ws, wf) pairs
// (2 m doubles), the virtual prefix P (3 m + 1), the list-boundary prefixes
// of wf (56) and the per-card terms G, CF (2 x 56), then the list hands
// (2 m int32) and list pointers (56 int32).  (Staging the output table too,
// and looping over several sequences per CTA, was measured slower: the
// larger footprint halves the resident CTAs per SM.)
size_t fused_smem(int maxMS) {
    return sizeof(double) * (5 * size_t(maxMS) + 1 + 3 * 56) + sizeof(int32_t) * (2 * size_t(maxMS) + 56);
}

// One CTA per (sequence a, board b); see the file header for the algebra.
//
// The prefix sums run over one virtual array of 3 m entries: the m values
// ws[j] (strength order), then the 2 m values ws[h] of the 52 card lists laid
// end to end.  Its exclusive prefix P gives ps = P[0..m] directly and every
// per-card prefix as a difference P[m + pos] − P[m + start(c)], so a single
// block scan replaces 53 segmented ones.  The same scan carries wf, whose
// prefix is only kept at the 53 list boundaries (QB): TF = QB[0] and the
// per-card sums CF[c] = QB[c+1] − QB[c].  With B_c / E_c the start / end of
// card c's list in P, the W-weighted part of an output is
//   lower − upper = (P[lt] + P[le] − TS) − (P[p1lt] + P[p1le])
//                   − (P[p2lt] + P[p2le]) + G[c1] + G[c2],   G[c] = P[B_c] + P[E_c].
//
// SEQ: v and out are sequence-major per board (board b's block of m_b·n
// values starts where it does hand-major, laid out [seq][hand]), so the
// gathers of step 1 and the stores of step 3 are coalesced across the CTA;
// k_board_transpose converts around the kernel.
template <bool SEQ, int T>
__global__ void __launch_bounds__(T) k_kron_fused(KronDir d, int b0, const double* __restrict__ in,
                                                         double* __restrict__ out) {
    constexpr int kPerT = kMaxHands / T;
    static_assert(T >= kScanT, "K7 CTAs hold at least the scan's threads");
    krb::pdl_entry();
    extern __shared__ double sm[];
    __shared__ double warpV[kScanT / 32], warpW[kScanT / 32];
    const int a = blockIdx.x, b = b0 + int(blockIdx.y);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t sBase = d.sumOff[b];
    const int mSb = int(d.sumOff[b + 1] - sBase);
    const int N = 3 * mSb;
    double2* W = reinterpret_cast<double2*>(sm);  // [mSb] (ws, wf)
    double* P = sm + 2 * mSb;                     // [N + 1]
    double* QB = P + N + 1;                       // [53]
    double* G = QB + 56;                          // [52]
    double* CF = G + 56;                          // [52]
    int32_t* lhand = reinterpret_cast<int32_t*>(CF + 56);  // [2 mSb]
    int32_t* lptr = lhand + 2 * mSb;                       // [53]
    KR_SMEM_CHECK(0, sizeof(double) * (5 * size_t(mSb) + 1 + 3 * 56) + sizeof(int32_t) * (2 * size_t(mSb) + 56));
    KR_DCHECK(mSb <= d.maxMS && mSb <= kMaxHands);

    // 1. weights of every summing hand for sequence a: the few F/S entries of
    // row a are uniform across the CTA, so each thread issues the gathers of
    // all its kPerT hands back to back.  The card lists are staged meanwhile.
    {
        const int32_t* lb = d.listPtr + int64_t(b) * (kCards + 1);
        if (tid <= kCards) lptr[tid] = __ldg(lb + tid);
        const int32_t* hands = d.listHands + d.listBase[b];
#pragma unroll
        for (int q = 0; q < 2 * kPerT; ++q)
            if (tid + q * T < 2 * mSb) {
                lhand[tid + q * T] = __ldg(hands + tid + q * T);
                KR_DCHECK(unsigned(lhand[tid + q * T]) < unsigned(mSb));
            }
        KR_DCHECK(tid > kCards || (lptr[tid] >= 0 && lptr[tid] <= 2 * mSb));

        const int64_t* fp = d.fptr + int64_t(b) * (d.nO + 1) + a;
        const int64_t* sp = d.sptr + int64_t(b) * (d.nO + 1) + a;
        const int64_t f0 = fp[0], f1 = fp[1], s0 = sp[0], s1 = sp[1];
        const int64_t nS = d.nS;
        const double* v0 = SEQ ? in + sBase * nS + tid : in + (sBase + tid) * nS;
        const int64_t step = SEQ ? int64_t(T) : int64_t(T) * nS;
        const int64_t colMul = SEQ ? int64_t(mSb) : 1;
        double f[kPerT], s[kPerT];
#pragma unroll
        for (int q = 0; q < kPerT; ++q) f[q] = s[q] = 0.0;
        for (int64_t e = f0; e < f1; ++e) {
            const double val = __ldg(d.fval + e);
            KR_DCHECK(unsigned(__ldg(d.fcol + e)) < unsigned(nS));
            const double* vc = v0 + __ldg(d.fcol + e) * colMul;
#pragma unroll
            for (int q = 0; q < kPerT; ++q)
                if (tid + q * T < mSb) f[q] += val * __ldg(vc + q * step);
        }
        for (int64_t e = s0; e < s1; ++e) {
            const double val = __ldg(d.sval + e);
            KR_DCHECK(unsigned(__ldg(d.scol + e)) < unsigned(nS));
            const double* vc = v0 + __ldg(d.scol + e) * colMul;
#pragma unroll
            for (int q = 0; q < kPerT; ++q)
                if (tid + q * T < mSb) s[q] += val * __ldg(vc + q * step);
        }
#pragma unroll
        for (int q = 0; q < kPerT; ++q) {
            const int j = tid + q * T;
            if (j < mSb) {
                const double lam = __ldg(d.lamS + sBase + j);
                W[j] = make_double2(lam * s[q], lam * f[q]);
            }
        }
    }
    __syncthreads();

    // 2. one block scan over the virtual array, in kScanT contiguous chunks
    // whatever the CTA size: the summation order (and so the bits) of a
    // board's product does not depend on the engine's launch shape, which
    // depends on its board count (a shard of boards on one rank sums exactly
    // as the whole turn on one GPU).  With T = 512 the upper half idles here.
    constexpr int kWarpsS = kScanT / 32;
    const bool scanner = tid < kScanT;
    const int chunk = (N + kScanT - 1) / kScanT;
    const int j0 = scanner ? min(N, tid * chunk) : N, j1 = scanner ? min(N, j0 + chunk) : N;
    double sv = 0.0, sw = 0.0;
#pragma unroll 4
    for (int p = j0; p < j1; ++p) {
        const double2 w = W[p < mSb ? p : lhand[p - mSb]];
        P[p] = w.x;  // staged; replaced by its prefix below
        sv += w.x;
        sw += w.y;
    }
    const double iv = warp_incl_scan(sv, lane);
    const double iw = warp_incl_scan(sw, lane);
    if (lane == 31 && warp < kWarpsS) {
        warpV[warp] = iv;
        warpW[warp] = iw;
    }
    // output tables are independent of the scan: load them before the barrier
    // (measured: loading them in step 3 instead frees registers for a fourth
    // resident CTA but is 15% slower)
    const int64_t oBase = d.outOff[b];
    const int mOb = int(d.outOff[b + 1] - oBase);
    int4 tb[kPerT];
    double lo[kPerT];
#pragma unroll
    for (int q = 0; q < kPerT; ++q) {
        const int i = tid + q * T;
        if (i < mOb) {
            tb[q] = __ldg(d.otab + oBase + i);
            lo[q] = __ldg(d.lamO + oBase + i);
        }
    }
    __syncthreads();
    if (scanner) {
        double run = iv - sv, runQ = iw - sw;
        for (int w = 0; w < warp; ++w) {
            run += warpV[w];
            runQ += warpW[w];
        }
        {
            // wf prefix at the list boundaries inside [j0, j1): B_c = mSb + lptr[c]
            int nc = 0;
            {
                int hi = kCards + 1;  // first c with mSb + lptr[c] >= j0
                while (nc < hi) {
                    const int mid = (nc + hi) >> 1;
                    if (mSb + lptr[mid] < j0) nc = mid + 1; else hi = mid;
                }
            }
            int p = j0;
            for (; nc <= kCards; ++nc) {
                const int B = mSb + lptr[nc];
                if (B >= j1) break;
                for (; p < B; ++p) runQ += W[p < mSb ? p : lhand[p - mSb]].y;
                QB[nc] = runQ;
            }
            if (tid == kScanT - 1) {
                for (; p < j1; ++p) runQ += W[p < mSb ? p : lhand[p - mSb]].y;
                for (; nc <= kCards; ++nc) QB[nc] = runQ;  // lists ending at N
            }
        }
#pragma unroll 4
        for (int p = j0; p < j1; ++p) {
            const double v = P[p];
            P[p] = run;
            run += v;
        }
        if (tid == kScanT - 1) P[N] = run;
    }
    __syncthreads();
    if (tid < kCards) {  // per-card terms
        G[tid] = P[mSb + lptr[tid]] + P[mSb + lptr[tid + 1]];
        CF[tid] = QB[tid + 1] - QB[tid];
    }
    __syncthreads();

    // 3. outputs of every hand of the board for sequence a
    const double TF = QB[0];
    const double TS = P[mSb];
    const double sg = double(d.sign);
#pragma unroll
    for (int q = 0; q < kPerT; ++q) {
        const int i = tid + q * T;
        if (i < mOb) {
            const int4 t = tb[q];
            const int lt = t.x & 0xffff, le = t.x >> 16;
            const int dup = (t.y & 0xffff) - 1, c1 = (t.y >> 16) & 0xff, c2 = t.y >> 24;
            const int p1lt = t.z & 0xffff, p1le = t.z >> 16, p2lt = t.w & 0xffff, p2le = t.w >> 16;
            KR_DCHECK(lt <= N && le <= N && p1lt <= N && p1le <= N && p2lt <= N && p2le <= N);
            KR_DCHECK(dup < mSb && c1 < kCards && c2 < kCards);
            double fpart = TF - CF[c1] - CF[c2];
            if (dup >= 0) fpart += W[dup].y;
            const double wsum = (P[lt] + P[le] - TS) - (P[p1lt] + P[p1le]) - (P[p2lt] + P[p2le]) + G[c1] + G[c2];
            const double r = lo[q] * (fpart + sg * wsum);
            if (SEQ) out[oBase * d.nO + int64_t(a) * mOb + i] = r;
            else out[(oBase + i) * d.nO + a] = r;
        }
    }
}

// Per-board transpose between hand-major [hand][seq] and sequence-major
// [seq][hand] (board b's block starts at off[b]·n either way).  32×32 tiles
// through shared memory, so both the loads and the stores are coalesced.
// grid = (hand tiles × sequence tiles, boards).
__global__ void __launch_bounds__(256) k_board_transpose(const double* __restrict__ src, double* __restrict__ dst,
                                                         const int64_t* __restrict__ off, int n, int b0,
                                                         int toSeq) {
    krb::pdl_entry();
    __shared__ double t[32][33];
    const int b = b0 + int(blockIdx.y);
    const int64_t base = off[b] * n;
    const int m = int(off[b + 1] - off[b]);
    const int tilesS = (n + 31) >> 5;
    const int h0 = int(blockIdx.x / unsigned(tilesS)) * 32, s0 = int(blockIdx.x % unsigned(tilesS)) * 32;
    if (h0 >= m) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    if (toSeq) {  // read rows h (contiguous s), write rows s (contiguous h)
#pragma unroll
        for (int r = ty; r < 32; r += 8)
            if (h0 + r < m && s0 + tx < n) t[r][tx] = src[base + int64_t(h0 + r) * n + s0 + tx];
        __syncthreads();
#pragma unroll
        for (int r = ty; r < 32; r += 8)
            if (s0 + r < n && h0 + tx < m) dst[base + int64_t(s0 + r) * m + h0 + tx] = t[tx][r];
    } else {
#pragma unroll
        for (int r = ty; r < 32; r += 8)
            if (s0 + r < n && h0 + tx < m) t[tx][r] = src[base + int64_t(s0 + r) * m + h0 + tx];
        __syncthreads();
#pragma unroll
        for (int r = ty; r < 32; r += 8)
            if (h0 + r < m && s0 + tx < n) dst[base + int64_t(h0 + r) * n + s0 + tx] = t[r][tx];
    }
}

template <class T>
T* upload(const std::vector<T>& v) {
    T* p = dev_alloc<T>(int64_t(v.size()));
    if (!v.empty()) KR_CK(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return p;
}

void check_csr(const kr_compressed& m, int rows, int cols, const char* name) {
    if (m.outer_size != rows || !m.outer) throw Fail{KR_INVALID_INPUT, std::string(name) + ": wrong outer size"};
    if (m.outer[0] != 0) throw Fail{KR_INVALID_INPUT, std::string(name) + ": outer[0] != 0"};
    for (int r = 0; r < rows; ++r)
        if (m.outer[r + 1] < m.outer[r]) throw Fail{KR_INVALID_INPUT, std::string(name) + ": outer not monotone"};
    const int64_t nnz = m.outer[rows];
    if (nnz > 0 && (!m.inner || !m.val)) throw Fail{KR_INVALID_INPUT, std::string(name) + ": null arrays"};
    for (int64_t e = 0; e < nnz; ++e) {
        if (m.inner[e] < 0 || m.inner[e] >= cols)
            throw Fail{KR_INVALID_INPUT, std::string(name) + ": column index out of range"};
        if (!std::isfinite(m.val[e])) throw Fail{KR_INVALID_INPUT, std::string(name) + ": non-finite value"};
    }
}

struct HostCsr {
    std::vector<int64_t> ptr;
    std::vector<int32_t> col;
    std::vector<double> val;
};

// F (n1 x n2) as given, or its transpose (stable counting sort: columns of
// each transposed row ascending).
HostCsr csr_dir(const kr_compressed& m, int n1, int n2, bool transpose) {
    HostCsr h;
    const int64_t nnz = m.outer[n1];
    if (!transpose) {
        h.ptr.assign(m.outer, m.outer + n1 + 1);
        h.col.assign(m.inner, m.inner + nnz);
        h.val.assign(m.val, m.val + nnz);
        return h;
    }
    h.ptr.assign(static_cast<size_t>(n2) + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) h.ptr[size_t(m.inner[e]) + 1]++;
    for (int c = 0; c < n2; ++c) h.ptr[size_t(c) + 1] += h.ptr[size_t(c)];
    h.col.resize(static_cast<size_t>(nnz));
    h.val.resize(static_cast<size_t>(nnz));
    std::vector<int64_t> pos(h.ptr.begin(), h.ptr.end() - 1);
    for (int r = 0; r < n1; ++r)
        for (int64_t e = m.outer[r]; e < m.outer[r + 1]; ++e) {
            const int64_t q = pos[size_t(m.inner[e])]++;
            h.col[size_t(q)] = r;
            h.val[size_t(q)] = m.val[e];
        }
    return h;
}

struct Side {
    int m;
    const uint32_t* key;
    const uint8_t* cards;
    const double* lam;
};

void build_dir(KronDir& d, const kr_kron_board* boards, int nb, int dir) {
    const int O = dir == 0 ? 0 : 1;
    d.nb = nb;
    d.sign = dir == 0 ? 1 : -1;
    d.nO = O == 0 ? boards[0].n1 : boards[0].n2;
    d.nS = O == 0 ? boards[0].n2 : boards[0].n1;
    const size_t NB = static_cast<size_t>(nb);
    std::vector<int64_t> sumOff(NB + 1, 0), outOff(NB + 1, 0), listBase(NB);
    std::vector<int32_t> listPtr, listHands;
    std::vector<int4> otab;
    std::vector<double> lamS, lamO;
    std::vector<int64_t> fptr, sptr;
    std::vector<int32_t> fcol, scol;
    std::vector<double> fval, sval;
    int64_t nnzFS = 0;
    d.maxMS = 0;
    for (int b = 0; b < nb; ++b) {
        const kr_kron_board& B = boards[b];
        const Side sO = O == 0 ? Side{B.m1, B.key1, B.cards1, B.lambda1} : Side{B.m2, B.key2, B.cards2, B.lambda2};
        const Side sS = O == 0 ? Side{B.m2, B.key2, B.cards2, B.lambda2} : Side{B.m1, B.key1, B.cards1, B.lambda1};
        const int mS = sS.m;
        if (mS > kMaxHands || sO.m > kMaxHands)
            throw Fail{KR_INVALID_INPUT, "more than 1536 hands on one side of a board"};
        d.maxMS = std::max(d.maxMS, mS);
        d.maxMO = std::max(d.maxMO, sO.m);
        sumOff[size_t(b) + 1] = sumOff[size_t(b)] + mS;
        outOff[size_t(b) + 1] = outOff[size_t(b)] + sO.m;
        lamS.insert(lamS.end(), sS.lam, sS.lam + mS);
        lamO.insert(lamO.end(), sO.lam, sO.lam + sO.m);
        // F_d / S_d of this board, positions global
        const HostCsr F = csr_dir(B.F, B.n1, B.n2, O == 1), S = csr_dir(B.S, B.n1, B.n2, O == 1);
        for (int a = 0; a <= d.nO; ++a) {
            fptr.push_back(int64_t(fcol.size()) + F.ptr[size_t(a)]);
            sptr.push_back(int64_t(scol.size()) + S.ptr[size_t(a)]);
        }
        nnzFS += int64_t(F.col.size() + S.col.size()) * mS;
        fcol.insert(fcol.end(), F.col.begin(), F.col.end());
        fval.insert(fval.end(), F.val.begin(), F.val.end());
        scol.insert(scol.end(), S.col.begin(), S.col.end());
        sval.insert(sval.end(), S.val.begin(), S.val.end());
        // card lists of the summing side (hands ascending = keys ascending)
        std::vector<int32_t> cnt(kCards + 1, 0);
        for (int j = 0; j < mS; ++j)
            for (int s = 0; s < 2; ++s) cnt[size_t(sS.cards[2 * j + s]) + 1]++;
        for (int c = 0; c < kCards; ++c) cnt[size_t(c) + 1] += cnt[size_t(c)];
        listBase[size_t(b)] = int64_t(listHands.size());
        listPtr.insert(listPtr.end(), cnt.begin(), cnt.end());
        std::vector<int32_t> lh(static_cast<size_t>(2 * mS));
        {
            std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
            for (int j = 0; j < mS; ++j)
                for (int s = 0; s < 2; ++s) lh[size_t(pos[size_t(sS.cards[2 * j + s])]++)] = j;
        }
        listHands.insert(listHands.end(), lh.begin(), lh.end());
        // output-side lookups
        const uint32_t* kS = sS.key;
        for (int i = 0; i < sO.m; ++i) {
            const uint32_t k = sO.key[i];
            const int c1 = sO.cards[2 * i], c2 = sO.cards[2 * i + 1];
            int32_t lt = int32_t(std::lower_bound(kS, kS + mS, k) - kS);
            int32_t le = int32_t(std::upper_bound(kS, kS + mS, k) - kS);
            int32_t dup = -1, plt[2], ple[2];
            for (int s = 0; s < 2; ++s) {
                const int c = s == 0 ? c1 : c2;
                const int p0 = cnt[size_t(c)], p1 = cnt[size_t(c) + 1];
                auto keyAt = [&](int p) { return kS[lh[size_t(p)]]; };
                int lo = p0, hi = p1;  // first list position with key >= k
                while (lo < hi) {
                    const int mid = (lo + hi) / 2;
                    if (keyAt(mid) < k) lo = mid + 1; else hi = mid;
                }
                int lo2 = lo, hi2 = p1;  // first with key > k
                while (lo2 < hi2) {
                    const int mid = (lo2 + hi2) / 2;
                    if (keyAt(mid) <= k) lo2 = mid + 1; else hi2 = mid;
                }
                plt[s] = mS + lo;  // position in the kernel's virtual prefix array
                ple[s] = mS + lo2;
                if (s == 0)
                    for (int p = p0; p < p1; ++p) {
                        const int j = lh[size_t(p)];
                        const int d1 = sS.cards[2 * j], d2 = sS.cards[2 * j + 1];
                        if ((d1 == c1 && d2 == c2) || (d1 == c2 && d2 == c1)) dup = j;
                    }
            }
            int4 t;
            t.x = lt | (le << 16);
            t.y = (dup + 1) | (c1 << 16) | (c2 << 24);
            t.z = plt[0] | (ple[0] << 16);
            t.w = plt[1] | (ple[1] << 16);
            otab.push_back(t);
        }
    }
    d.mO = outOff[NB];
    d.mS = sumOff[NB];
    // weights (2 flops per F/S entry per summing hand), scans (6 per summing
    // hand and sequence), combine (14 per output)
    d.flops = 2 * int64_t(nnzFS) + 6 * int64_t(d.nO) * d.mS + 14 * d.mO * d.nO;
    d.sumOff = upload(sumOff);
    d.outOff = upload(outOff);
    d.lamS = upload(lamS);
    d.lamO = upload(lamO);
    d.fptr = upload(fptr);
    d.fcol = upload(fcol);
    d.fval = upload(fval);
    d.sptr = upload(sptr);
    d.scol = upload(scol);
    d.sval = upload(sval);
    d.listPtr = upload(listPtr);
    d.listBase = upload(listBase);
    d.listHands = upload(listHands);
    d.otab = upload(otab);
}

void free_dir(KronDir& d) {
    void* ps[] = {d.sumOff, d.outOff, d.lamS, d.lamO, d.fptr, d.fcol, d.fval, d.sptr, d.scol, d.sval,
                  d.listPtr, d.listBase, d.listHands, d.otab};
    for (void* p : ps) krb::dev_free(p);
    d = KronDir{};
}

void validate_board(const kr_kron_board& B, const kr_kron_board& B0, int b) {
    const std::string at = "board " + std::to_string(b) + ": ";
    if (B.m1 < 0 || B.m2 < 0) throw Fail{KR_INVALID_INPUT, at + "negative hand count"};
    if (B.n1 < 1 || B.n2 < 1) throw Fail{KR_INVALID_INPUT, at + "empty sequence space"};
    if (B.n1 != B0.n1 || B.n2 != B0.n2) throw Fail{KR_INVALID_INPUT, at + "boards must share one betting tree"};
    check_csr(B.F, B.n1, B.n2, "F");
    check_csr(B.S, B.n1, B.n2, "S");
    const Side sides[2] = {{B.m1, B.key1, B.cards1, B.lambda1}, {B.m2, B.key2, B.cards2, B.lambda2}};
    for (const Side& s : sides) {
        if (s.m > 0 && (!s.key || !s.cards || !s.lam)) throw Fail{KR_INVALID_INPUT, at + "null hand arrays"};
        for (int i = 0; i < s.m; ++i) {
            if (i > 0 && s.key[i] < s.key[i - 1])
                throw Fail{KR_INVALID_INPUT, at + "hands must be strength-sorted ascending (kron.hpp:74-83)"};
            const int c1 = s.cards[2 * i], c2 = s.cards[2 * i + 1];
            if (c1 >= kCards || c2 >= kCards || c1 == c2) throw Fail{KR_INVALID_INPUT, at + "bad hand cards"};
            if (!std::isfinite(s.lam[i])) throw Fail{KR_INVALID_INPUT, at + "non-finite lambda"};
        }
    }
}

}  // namespace

struct KronState {
    KronDir dir[2];
    size_t smem[2] = {0, 0};
    // sequence-major copies of each direction's input and output (one pair
    // per direction: kr_engine_pair_device runs the two concurrently)
    double* seqIn[2] = {nullptr, nullptr};
    double* seqOut[2] = {nullptr, nullptr};
};

void kron_destroy(KronState* k) {
    if (!k) return;
    free_dir(k->dir[0]);
    free_dir(k->dir[1]);
    for (int i = 0; i < 2; ++i) {
        krb::dev_free(k->seqIn[i]);
        krb::dev_free(k->seqOut[i]);
    }
    delete k;
}

// KR_KRON_SEQ=1: the product runs sequence-major (transpose in, K7<SEQ>,
// transpose out); read per launch so a process can switch.
bool kron_seq_major() {
    const char* env = std::getenv("KR_KRON_SEQ");
    return env ? std::atoi(env) != 0 : kKronSeqDefault;
}

// The product on sequence-major vectors (per board [seq][hand]) with no
// transposes: the DCFR solver keeps the strategies and gradients of a K7
// engine sequence-major (kr_solver.cu, k7seq), so the coalesced kernel runs
// alone.  Same bits as kron_product (the layout changes only addresses).
void kron_product_seq(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s) {
    KronState* k = e->kron;
    KronDir& d = k->dir[dir];
    if (d.mO * d.nO == 0) return;
    const bool wide = int64_t(d.nO) * d.nb <= kSmallGrid;
    if (wide)
        krb::launch(k_kron_fused<true, 512>, dim3(unsigned(d.nO), unsigned(d.nb)), 512, k->smem[dir], s, d, 0, in,
                    out);
    else
        krb::launch(k_kron_fused<true, kThreads>, dim3(unsigned(d.nO), unsigned(d.nb)), kThreads, k->smem[dir], s, d,
                    0, in, out);
    KR_CK_LAUNCH();
    e->launches++;
}

// Hand-major <-> sequence-major per board for direction dir's input side
// (side 0: the summing hands, n = nS) or output side (side 1: n = nO).
void kron_transpose(kr_engine* e, int dir, int side, const double* src, double* dst, bool toSeq, cudaStream_t s) {
    KronState* k = e->kron;
    KronDir& d = k->dir[dir];
    const int n = side == 0 ? d.nS : d.nO;
    const int maxM = side == 0 ? d.maxMS : d.maxMO;
    if (n == 0 || d.nb == 0) return;
    const unsigned tiles = unsigned((maxM + 31) / 32) * unsigned((n + 31) / 32);
    krb::launch(k_board_transpose, dim3(tiles, unsigned(d.nb)), 256, 0, s, src, dst, side == 0 ? d.sumOff : d.outOff, n,
                0, toSeq ? 1 : 0);
    KR_CK_LAUNCH();
    e->launches++;
}

void kron_product(kr_engine* e, int dir, const double* in, double* out, cudaStream_t s, int b0, int b1) {
    KronState* k = e->kron;
    KronDir& d = k->dir[dir];
    if (b1 < 0) b1 = d.nb;
    if (d.mO * d.nO == 0 || b1 <= b0) return;
    // Engines whose whole grid has at most one CTA per SM (single boards) run
    // 512-thread CTAs: that shortens each CTA, which is the whole launch.
    // Larger grids keep 256 (measured: config 2 14.5 -> 13.3 us per pair,
    // config 3 110 -> 123 us with 512).  Decided per engine, not per launch,
    // so board-group sub-launches sum in the same order as whole-range ones.
    const bool wide = int64_t(d.nO) * d.nb <= kSmallGrid;
    if (!kron_seq_major()) {
        if (wide)
            krb::launch(k_kron_fused<false, 512>, dim3(unsigned(d.nO), unsigned(b1 - b0)), 512, k->smem[dir], s, d,
                        b0, in, out);
        else
            krb::launch(k_kron_fused<false, kThreads>, dim3(unsigned(d.nO), unsigned(b1 - b0)), kThreads,
                        k->smem[dir], s, d, b0, in, out);
        KR_CK_LAUNCH();
        e->launches++;
        return;
    }
    const unsigned nb = unsigned(b1 - b0);
    const unsigned tilesS = unsigned((d.nS + 31) / 32), tilesO = unsigned((d.nO + 31) / 32);
    krb::launch(k_board_transpose, dim3(unsigned((d.maxMS + 31) / 32) * tilesS, nb), 256, 0, s, in, k->seqIn[dir],
                d.sumOff, d.nS, b0, 1);
    KR_CK_LAUNCH();
    if (wide)
        krb::launch(k_kron_fused<true, 512>, dim3(unsigned(d.nO), nb), 512, k->smem[dir], s, d, b0, k->seqIn[dir],
                    k->seqOut[dir]);
    else
        krb::launch(k_kron_fused<true, kThreads>, dim3(unsigned(d.nO), nb), kThreads, k->smem[dir], s, d, b0,
                    k->seqIn[dir], k->seqOut[dir]);
    KR_CK_LAUNCH();
    krb::launch(k_board_transpose, dim3(unsigned((d.maxMO + 31) / 32) * tilesO, nb), 256, 0, s, k->seqOut[dir], out,
                d.outOff, d.nO, b0, 0);
    KR_CK_LAUNCH();
    e->launches += 3;
}

int64_t kron_flops(const kr_engine* e, int dir) { return e->kron->dir[dir].flops; }
int kron_boards(const kr_engine* e) { return e->kron->dir[0].nb; }

kr_engine* create_kron_engine(const kr_kron_board* boards, int nb, int device, uint32_t flags) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Fail{KR_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    }
    if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
    if (!boards || nb < 1) throw Fail{KR_INVALID_INPUT, "at least one board is required"};
    int64_t R = 0, C = 0;
    for (int b = 0; b < nb; ++b) {
        validate_board(boards[b], boards[0], b);
        R += int64_t(boards[b].m1) * boards[b].n1;
        C += int64_t(boards[b].m2) * boards[b].n2;
    }
    if (R > INT32_MAX || C > INT32_MAX) throw Fail{KR_INVALID_INPUT, "dimensions exceed 32-bit indices"};
    KR_CK(cudaSetDevice(device));
    kr_engine* e = new kr_engine();
    try {
        e->device = device;
        KR_CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->rows = R;
        e->cols = C;
        e->n1 = boards[0].n1;
        e->n2 = boards[0].n2;
        e->kron = new KronState();
        size_t smMax = 0;
        for (int dir = 0; dir < 2; ++dir) {
            KronDir& d = e->kron->dir[dir];
            build_dir(d, boards, nb, dir);
            e->kron->smem[dir] = fused_smem(d.maxMS);
            smMax = std::max(smMax, e->kron->smem[dir]);
        }
        if (smMax > 227 * 1024) throw Fail{KR_INVALID_INPUT, "board has too many hands for the implicit engine"};
        raise_smem_limit(k_kron_fused<false, kThreads>, smMax);
        raise_smem_limit(k_kron_fused<false, 512>, smMax);
        raise_smem_limit(k_kron_fused<true, kThreads>, smMax);
        raise_smem_limit(k_kron_fused<true, 512>, smMax);
        for (int dir = 0; dir < 2; ++dir) {
            e->kron->seqIn[dir] = dev_alloc<double>(dir == 0 ? C : R);
            e->kron->seqOut[dir] = dev_alloc<double>(dir == 0 ? R : C);
        }
        e->flops_per_product = e->kron->dir[0].flops;
        e->d_in = dev_alloc<double>(std::max(R, C));
        e->d_out = dev_alloc<double>(std::max(R, C));
        // board groups for the pipelined host-buffer calls
        // (eight: the kernel is short next to the copies, so finer groups
        // shorten the unhidden first input copy and last output copy)
        int G = 8;
        if (const char* env = std::getenv("KR_GROUPS")) G = std::atoi(env);
        G = (flags & KR_FLAG_SINGLE_PART) ? 1 : std::max(1, std::min(nb, G));
        for (int g = 0; g < G; ++g) {
            const int g0 = int(int64_t(nb) * g / G), g1 = int(int64_t(nb) * (g + 1) / G);
            int64_t r = 0, c = 0;
            for (int b = g0; b < g1; ++b) {
                r += int64_t(boards[b].m1) * boards[b].n1;
                c += int64_t(boards[b].m2) * boards[b].n2;
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

extern "C" int kr_engine_create_kron(const kr_kron_board* boards, int nboards, int device, uint32_t flags,
                                     kr_engine** out) {
    return krb::guarded([&] {
        if (!out) throw krb::Fail{KR_INVALID_INPUT, "null output handle"};
        *out = krb::create_kron_engine(boards, nboards, device, flags);
    });
}
