// kr_engine.cu — B200 factored gradient oracle: y = A x and x = A^T y with
// A = Ahat + U M^-1 V^T (arXiv 2112.03804; reference engine.hpp:58-133).
//
// Design:
//  * Every product is "ordered": each output row is accumulated by ONE thread
//    in the reference's storage order (engine.hpp:67-70, 82-88, 104-108,
//    118-129), so results are bitwise equal to the reference (compiled with
//    -fmad=false: no contraction, as in the reference's x86-64 build).
//  * The scatter loops of matvecTranspose become gathers over precomputed
//    transposed layouts built once at create time (no atomics, deterministic).
//  * Ax = [V^T x] -> [M solve] -> [[U|Ahat] over [z|x]]; the U and Ahat rows
//    are merged so one pass reproduces the single accumulator of
//    engine.hpp:83-89.  ATx = [U^T y] -> [M^T solve] -> [[Ahat^T|V] over [y|z]].
//  * SpMV kernel: row blocks of <= 256 rows and ~4K entries; each tile of
//    column indices and values is streamed with coalesced loads, the products
//    are staged in shared memory, then each thread folds its own row's
//    products in order.  Technique B's M is a set of chains (segmented
//    recurrences over strength-sorted hands), solved one chain per thread.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <thread>

#include "kr_common.cuh"

namespace krb {

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

namespace {
thread_local int g_code = 0;
thread_local std::string g_msg;
}  // namespace

void set_error(int code, const std::string& msg) {
    g_code = code;
    g_msg = msg;
}

namespace {

constexpr int kThreads = 256;        // threads per SpMV block == max rows per block
constexpr int kTile = 2048;          // entries staged per tile (16 KB of products)
constexpr int kPer = kTile / kThreads;
constexpr int64_t kNnzPerBlock = 4096;

// ------------------------------------------------------------- kernels ----

// y[r] = sum over row r of val * src[col], in storage order.  src is the
// concatenation [xa (split entries) | xb] when TWO is set.
template <bool TWO>
__global__ void __launch_bounds__(kThreads) k_ordered_spmv(const int64_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ val,
                                                           const int32_t* __restrict__ blk,
                                                           const double* __restrict__ xa,
                                                           const double* __restrict__ xb, int32_t split,
                                                           double* __restrict__ y) {
    __shared__ double P[kTile];
    const int32_t r0 = blk[blockIdx.x], r1 = blk[blockIdx.x + 1];
    const int64_t e0 = rowptr[r0], e1 = rowptr[r1];
    const int tid = threadIdx.x;
    const int32_t r = r0 + tid;
    int64_t rs = 0, re = 0;
    if (r < r1) {
        rs = rowptr[r];
        re = rowptr[r + 1];
    }
    double acc = 0.0;
    for (int64_t t0 = e0; t0 < e1; t0 += kTile) {
        const int n = int(lmin(kTile, e1 - t0));
        int32_t cc[kPer];
        double vv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int q = tid + u * kThreads;
            if (q < n) {
                cc[u] = __ldcs(col + t0 + q);
                vv[u] = __ldcs(val + t0 + q);
            }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int q = tid + u * kThreads;
            if (q < n) {
                double xv;
                if (TWO) xv = cc[u] < split ? __ldg(xa + cc[u]) : __ldg(xb + (cc[u] - split));
                else xv = __ldg(xa + cc[u]);
                P[q] = vv[u] * xv;
            }
        }
        __syncthreads();
        const int64_t s = max(rs, t0), en = min(re, t0 + n);
        for (int64_t e = s; e < en; ++e) acc += P[e - t0];
        __syncthreads();
    }
    if (r < r1) y[r] = acc;
}

// Forward solve M z = t along chains (engine.hpp:31-41 restricted to <=1
// off-diagonal per row/column): z_r = t_r - M(r,p) z_p, skipped when z_p == 0.
__global__ void k_chain_forward(const int64_t* __restrict__ cptr, const int32_t* __restrict__ cidx,
                                const double* __restrict__ cmul, int64_t nchains, double* __restrict__ z) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchains) return;
    const int64_t a = cptr[c], b = cptr[c + 1];
    double prev = 0.0;
    for (int64_t k0 = a; k0 < b; k0 += 8) {
        const int n = int(lmin(8, b - k0));
        int32_t rr[8];
        double mm[8], tt[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < n) {
                rr[u] = cidx[k0 + u];
                mm[u] = cmul[k0 + u];
            }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < n) tt[u] = z[rr[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < n) {
                double zr = tt[u];
                if (k0 + u != a && prev != 0.0) zr = tt[u] - mm[u] * prev;
                z[rr[u]] = zr;
                prev = zr;
            }
    }
}

// Backward solve M^T z = s along chains (engine.hpp:44-54): visiting each
// chain in reverse, z_r = s_r - (0 + M(next, r) z_next).
__global__ void k_chain_backward(const int64_t* __restrict__ cptr, const int32_t* __restrict__ cidx,
                                 const double* __restrict__ cmul, int64_t nchains, double* __restrict__ z) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchains) return;
    const int64_t a = cptr[c], b = cptr[c + 1];
    double next = 0.0, mulNext = 0.0;
    bool have = false;
    for (int64_t k1 = b; k1 > a; k1 -= 8) {
        const int n = int(lmin(8, k1 - a));
        int32_t rr[8];
        double mm[8], ss[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < n) {
                rr[u] = cidx[k1 - 1 - u];
                mm[u] = cmul[k1 - 1 - u];
            }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < n) ss[u] = z[rr[u]];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < n) {
                double acc = 0.0;
                if (have) acc += mulNext * next;
                const double zr = ss[u] - acc;
                z[rr[u]] = zr;
                next = zr;
                mulNext = mm[u];
                have = true;
            }
    }
}

// General unit-lower forward solve, one level: row-oriented gathers in
// ascending column order == the column-oriented order of engine.hpp:33-40.
__global__ void k_level_forward(const int32_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ ptr,
                                const int32_t* __restrict__ col, const double* __restrict__ val,
                                double* __restrict__ z) {
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
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t j = cols[q];
    double acc = 0.0;
    for (int64_t e = ptr[j]; e < ptr[j + 1]; ++e) acc += val[e] * z[row[e]];
    z[j] -= acc;
}

// ------------------------------------------------------- host building ----

struct HostRows {  // row-ordered matrix under construction (one board)
    std::vector<int64_t> ptr;
    std::vector<int32_t> col;
    std::vector<double> val;
};

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

void partition_rows(const std::vector<int64_t>& ptr, int32_t rowOff, std::vector<int32_t>& blk) {
    const int64_t n = int64_t(ptr.size()) - 1;
    int64_t r = 0;
    while (r < n) {
        const int64_t start = r;
        int64_t nnz = 0;
        while (r < n && r - start < kThreads) {
            const int64_t len = ptr[r + 1] - ptr[r];
            if (r > start && nnz + len > kNnzPerBlock) break;
            nnz += len;
            ++r;
        }
        blk.push_back(int32_t(rowOff + start));
    }
}

void check_compressed(const kr_compressed& c, int64_t outerN, int64_t innerN, const char* name) {
    if (c.outer_size != outerN)
        throw Fail{KR_CONTRACT, std::string(name) + " dimensions do not match Ahat/M"};
    if (outerN > 0 && (!c.outer)) throw Fail{KR_INVALID_INPUT, std::string(name) + ": null outer array"};
    if (outerN == 0 && !c.outer) return;
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
    const kr_factors* f;
    int64_t rowOff, colOff, kOff;
    int64_t nnzVT, nnzUA, nnzUT, nnzAV;  // offsets into the combined arrays
    int mkind;
    std::string why;
};

void upload_rows(const HostRows& h, int64_t rowBase, int64_t nnzBase, krb::DevRows& d, cudaStream_t s) {
    const int64_t n = int64_t(h.ptr.size()) - 1;
    std::vector<int64_t> p(h.ptr.begin(), h.ptr.end() - 1);
    for (auto& x : p) x += nnzBase;
    if (n > 0) KR_CK(cudaMemcpyAsync(d.rowptr + rowBase, p.data(), 8 * size_t(n), cudaMemcpyHostToDevice, s));
    if (!h.col.empty()) {
        KR_CK(cudaMemcpyAsync(d.col + nnzBase, h.col.data(), 4 * h.col.size(), cudaMemcpyHostToDevice, s));
        KR_CK(cudaMemcpyAsync(d.val + nnzBase, h.val.data(), 8 * h.val.size(), cudaMemcpyHostToDevice, s));
    }
    KR_CK(cudaStreamSynchronize(s));
}

void alloc_rows(krb::DevRows& d, int64_t nrows, int64_t nnz) {
    d.nrows = nrows;
    d.nnz = nnz;
    d.rowptr = dev_alloc<int64_t>(nrows + 1);
    d.col = dev_alloc<int32_t>(std::max<int64_t>(nnz, 1));
    d.val = dev_alloc<double>(std::max<int64_t>(nnz, 1));
    KR_CK(cudaMemcpy(d.rowptr + nrows, &nnz, 8, cudaMemcpyHostToDevice));
}

void free_rows(krb::DevRows& d) {
    cudaFree(d.rowptr);
    cudaFree(d.col);
    cudaFree(d.val);
    cudaFree(d.blk);
    d = krb::DevRows{};
}

void finish_blocks(krb::DevRows& d, std::vector<int32_t>& blk) {
    blk.push_back(int32_t(d.nrows));
    d.nblk = int32_t(blk.size()) - 1;
    d.blk = dev_alloc<int32_t>(int64_t(blk.size()));
    KR_CK(cudaMemcpy(d.blk, blk.data(), 4 * blk.size(), cudaMemcpyHostToDevice));
}

void destroy_engine(kr_engine* e) {
    if (!e) return;
    cudaSetDevice(e->device);
    free_rows(e->VT);
    free_rows(e->UA);
    free_rows(e->UT);
    free_rows(e->AV);
    cudaFree(e->chain_ptr);
    cudaFree(e->chain_idx);
    cudaFree(e->chain_mul);
    cudaFree(e->lvl_fwd_rows);
    cudaFree(e->lvl_bwd_cols);
    cudaFree(e->mr_ptr);
    cudaFree(e->mr_col);
    cudaFree(e->mr_val);
    cudaFree(e->mc_ptr);
    cudaFree(e->mc_row);
    cudaFree(e->mc_val);
    cudaFree(e->d_tz);
    cudaFree(e->d_in);
    cudaFree(e->d_out);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

kr_engine* create_engine(const kr_factors* boards, int nb, int device, uint32_t flags) {
    (void)flags;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Fail{KR_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    }
    if (device < 0 || device >= ndev) throw Fail{KR_INVALID_INPUT, "device index out of range"};
    if (!boards || nb < 1) throw Fail{KR_INVALID_INPUT, "at least one factor set is required"};
    KR_CK(cudaSetDevice(device));

    std::vector<BoardPlan> plan(static_cast<size_t>(nb));
    int64_t R = 0, Cc = 0, K = 0, nVT = 0, nUA = 0, nUT = 0, nAV = 0, nM = 0;
    int32_t n1 = boards[0].n1, n2 = boards[0].n2;
    for (int b = 0; b < nb; ++b) {
        const kr_factors& f = boards[b];
        if (f.rows < 0 || f.cols < 0 || f.k < 0) throw Fail{KR_INVALID_INPUT, "negative dimension"};
        check_compressed(f.ahat, f.rows, f.cols, "Ahat");
        check_compressed(f.u, f.rows, f.k, "U");
        check_compressed(f.m, f.k, f.k, "M");
        check_compressed(f.v, f.k, f.cols, "V");
        if (f.n1 != n1 || f.n2 != n2) n1 = n2 = 0;
        BoardPlan& p = plan[b];
        p.f = &f;
        p.rowOff = R;
        p.colOff = Cc;
        p.kOff = K;
        p.nnzVT = nVT;
        p.nnzUA = nUA;
        p.nnzUT = nUT;
        p.nnzAV = nAV;
        const int64_t a = f.ahat.outer[f.rows], u = f.u.outer[f.rows], v = f.v.outer[f.k];
        nVT += v;
        nUA += u + a;
        nUT += u;
        nAV += a + v;
        nM += f.m.outer[f.k];
        R += f.rows;
        Cc += f.cols;
        K += f.k;
        p.mkind = classify_m(f.m, f.k, p.why);
    }
    if (R > INT32_MAX || Cc > INT32_MAX || K > INT32_MAX || R + K > INT32_MAX || Cc + K > INT32_MAX)
        throw Fail{KR_INVALID_INPUT, "dimensions exceed 32-bit indices"};

    kr_engine* e = new kr_engine();
    try {
        e->device = device;
        KR_CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
        e->rows = R;
        e->cols = Cc;
        e->k = K;
        e->nnzA = nUA - nUT;
        e->nnzU = nUT;
        e->nnzV = nVT;
        e->nnzM = nM;
        e->n1 = n1;
        e->n2 = n2;
        int worst = 0;
        bool anyGeneral = false, allIdentity = true;
        for (auto& p : plan) {
            if (p.mkind == 3 && worst != 3) {
                worst = 3;
                e->mfail = p.why;
            }
            if (p.mkind == 2) anyGeneral = true;
            if (p.mkind != 0) allIdentity = false;
        }
        e->mkind = worst == 3 ? 3 : allIdentity ? 0 : anyGeneral ? 2 : 1;
        // flop rule (engine.hpp:72,77,90-91): the combined M is the identity
        // iff every board's is.
        e->flops_per_product = e->nnzV + e->nnzU + e->nnzA + (e->mkind == 0 ? 0 : e->nnzM - K);

        alloc_rows(e->VT, K, nVT);
        alloc_rows(e->UA, R, nUA);
        alloc_rows(e->UT, K, nUT);
        alloc_rows(e->AV, Cc, nAV);
        e->d_tz = dev_alloc<double>(std::max<int64_t>(K, 1));
        e->d_in = dev_alloc<double>(std::max<int64_t>(std::max(R, Cc), 1));
        e->d_out = dev_alloc<double>(std::max<int64_t>(std::max(R, Cc), 1));

        std::vector<std::vector<int32_t>> bVT(static_cast<size_t>(nb)), bUA(static_cast<size_t>(nb)), bUT(static_cast<size_t>(nb)), bAV(static_cast<size_t>(nb));
        std::atomic<int> next{0};
        std::mutex mu;
        Fail firstFail{KR_OK, ""};
        auto worker = [&] {
            try {
                KR_CK(cudaSetDevice(device));
                cudaStream_t s;
                KR_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
                for (int b; (b = next.fetch_add(1)) < nb;) {
                    const BoardPlan& p = plan[size_t(b)];
                    const kr_factors& f = *p.f;
                    HostRows h;
                    // VT: V's CSC columns as rows, entries index x.
                    h.ptr.assign(f.v.outer, f.v.outer + f.k + 1);
                    const int64_t nv = f.v.outer[f.k];
                    h.col.resize(size_t(nv));
                    for (int64_t q = 0; q < nv; ++q) h.col[q] = int32_t(p.colOff + f.v.inner[q]);
                    h.val.assign(f.v.val, f.v.val + nv);
                    upload_rows(h, p.kOff, p.nnzVT, e->VT, s);
                    partition_rows(h.ptr, int32_t(p.kOff), bVT[size_t(b)]);
                    // UA: [U row | Ahat row] over [z (K) | x].
                    h.ptr.assign(size_t(f.rows) + 1, 0);
                    h.col.clear();
                    h.val.clear();
                    for (int64_t i = 0; i < f.rows; ++i) {
                        for (int64_t q = f.u.outer[i]; q < f.u.outer[i + 1]; ++q) {
                            h.col.push_back(int32_t(p.kOff + f.u.inner[q]));
                            h.val.push_back(f.u.val[q]);
                        }
                        for (int64_t q = f.ahat.outer[i]; q < f.ahat.outer[i + 1]; ++q) {
                            h.col.push_back(int32_t(K + p.colOff + f.ahat.inner[q]));
                            h.val.push_back(f.ahat.val[q]);
                        }
                        h.ptr[size_t(i) + 1] = int64_t(h.col.size());
                    }
                    upload_rows(h, p.rowOff, p.nnzUA, e->UA, s);
                    partition_rows(h.ptr, int32_t(p.rowOff), bUA[size_t(b)]);
                    // UT: U^T rows, entries index y.
                    std::vector<int64_t> tp;
                    std::vector<int32_t> ti;
                    std::vector<double> tv;
                    transpose_into(f.rows, f.k, f.u.outer, f.u.inner, f.u.val, tp, ti, tv);
                    for (auto& c : ti) c = int32_t(c + p.rowOff);
                    h.ptr = std::move(tp);
                    h.col = std::move(ti);
                    h.val = std::move(tv);
                    upload_rows(h, p.kOff, p.nnzUT, e->UT, s);
                    partition_rows(h.ptr, int32_t(p.kOff), bUT[size_t(b)]);
                    // AV: [Ahat^T row | V row] over [y (R) | z].
                    std::vector<int64_t> ap, vp;
                    std::vector<int32_t> ai, vi;
                    std::vector<double> av, vv;
                    transpose_into(f.rows, f.cols, f.ahat.outer, f.ahat.inner, f.ahat.val, ap, ai, av);
                    transpose_into(f.k, f.cols, f.v.outer, f.v.inner, f.v.val, vp, vi, vv);
                    h.ptr.assign(size_t(f.cols) + 1, 0);
                    h.col.clear();
                    h.val.clear();
                    h.col.reserve(ai.size() + vi.size());
                    h.val.reserve(ai.size() + vi.size());
                    for (int64_t c = 0; c < f.cols; ++c) {
                        for (int64_t q = ap[c]; q < ap[c + 1]; ++q) {
                            h.col.push_back(int32_t(p.rowOff + ai[q]));
                            h.val.push_back(av[q]);
                        }
                        for (int64_t q = vp[c]; q < vp[c + 1]; ++q) {
                            h.col.push_back(int32_t(R + p.kOff + vi[q]));
                            h.val.push_back(vv[q]);
                        }
                        h.ptr[size_t(c) + 1] = int64_t(h.col.size());
                    }
                    upload_rows(h, p.colOff, p.nnzAV, e->AV, s);
                    partition_rows(h.ptr, int32_t(p.colOff), bAV[size_t(b)]);
                }
                cudaStreamDestroy(s);
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

        auto cat = [&](std::vector<std::vector<int32_t>>& parts, krb::DevRows& d) {
            std::vector<int32_t> all;
            for (auto& v : parts) all.insert(all.end(), v.begin(), v.end());
            finish_blocks(d, all);
        };
        cat(bVT, e->VT);
        cat(bUA, e->UA);
        cat(bUT, e->UT);
        cat(bAV, e->AV);

        // M solve structures (global indices).
        if (e->mkind == 1) {
            std::vector<int64_t> cptr{0};
            std::vector<int32_t> cidx;
            std::vector<double> cmul;
            for (auto& p : plan) {
                const kr_factors& f = *p.f;
                std::vector<int64_t> nxt(static_cast<size_t>(f.k), -1);
                std::vector<double> mul(static_cast<size_t>(f.k), 0.0);
                std::vector<char> hasPrev(static_cast<size_t>(f.k), 0);
                for (int64_t j = 0; j < f.k; ++j)
                    for (int64_t q = f.m.outer[j] + 1; q < f.m.outer[j + 1]; ++q) {
                        nxt[j] = f.m.inner[q];
                        mul[size_t(f.m.inner[q])] = f.m.val[q];
                        hasPrev[size_t(f.m.inner[q])] = 1;
                    }
                for (int64_t j = 0; j < f.k; ++j) {
                    if (hasPrev[j]) continue;
                    for (int64_t r = j; r >= 0; r = nxt[r]) {
                        cidx.push_back(int32_t(p.kOff + r));
                        cmul.push_back(mul[r]);
                    }
                    cptr.push_back(int64_t(cidx.size()));
                }
            }
            e->nchains = int64_t(cptr.size()) - 1;
            e->chain_ptr = dev_alloc<int64_t>(int64_t(cptr.size()));
            e->chain_idx = dev_alloc<int32_t>(std::max<int64_t>(1, int64_t(cidx.size())));
            e->chain_mul = dev_alloc<double>(std::max<int64_t>(1, int64_t(cmul.size())));
            KR_CK(cudaMemcpy(e->chain_ptr, cptr.data(), 8 * cptr.size(), cudaMemcpyHostToDevice));
            if (!cidx.empty()) {
                KR_CK(cudaMemcpy(e->chain_idx, cidx.data(), 4 * cidx.size(), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(e->chain_mul, cmul.data(), 8 * cmul.size(), cudaMemcpyHostToDevice));
            }
        } else if (e->mkind == 2) {
            // strictly-lower parts, global indices; CSR via transpose of CSC
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
            std::vector<int32_t> lf(static_cast<size_t>(K), 0), lb(size_t(K), 0);
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
        KR_CK(cudaDeviceSynchronize());
    } catch (...) {
        destroy_engine(e);
        throw;
    }
    return e;
}

void launch_spmv(kr_engine* e, const krb::DevRows& A, const double* xa, const double* xb, int64_t split,
                 double* y, cudaStream_t s) {
    if (A.nblk == 0) return;
    if (xb) k_ordered_spmv<true><<<A.nblk, kThreads, 0, s>>>(A.rowptr, A.col, A.val, A.blk, xa, xb, int32_t(split), y);
    else k_ordered_spmv<false><<<A.nblk, kThreads, 0, s>>>(A.rowptr, A.col, A.val, A.blk, xa, nullptr, 0, y);
    KR_CK_LAUNCH();
    e->launches++;
}

void solve_forward(kr_engine* e, cudaStream_t s) {
    if (e->mkind == 1 && e->nchains > 0) {
        const int nt = 128;
        k_chain_forward<<<unsigned((e->nchains + nt - 1) / nt), nt, 0, s>>>(e->chain_ptr, e->chain_idx,
                                                                          e->chain_mul, e->nchains, e->d_tz);
        KR_CK_LAUNCH();
        e->launches++;
    } else if (e->mkind == 2) {
        for (size_t l = 0; l + 1 < e->lvl_fwd_ptr.size(); ++l) {
            const int64_t a = e->lvl_fwd_ptr[l], n = e->lvl_fwd_ptr[l + 1] - a;
            if (n == 0) continue;
            k_level_forward<<<unsigned((n + 127) / 128), 128, 0, s>>>(e->lvl_fwd_rows + a, n, e->mr_ptr, e->mr_col,
                                                                      e->mr_val, e->d_tz);
            KR_CK_LAUNCH();
            e->launches++;
        }
    }
}

void solve_backward(kr_engine* e, cudaStream_t s) {
    if (e->mkind == 1 && e->nchains > 0) {
        const int nt = 128;
        k_chain_backward<<<unsigned((e->nchains + nt - 1) / nt), nt, 0, s>>>(e->chain_ptr, e->chain_idx,
                                                                           e->chain_mul, e->nchains, e->d_tz);
        KR_CK_LAUNCH();
        e->launches++;
    } else if (e->mkind == 2) {
        for (size_t l = 0; l + 1 < e->lvl_bwd_ptr.size(); ++l) {
            const int64_t a = e->lvl_bwd_ptr[l], n = e->lvl_bwd_ptr[l + 1] - a;
            if (n == 0) continue;
            k_level_backward<<<unsigned((n + 127) / 128), 128, 0, s>>>(e->lvl_bwd_cols + a, n, e->mc_ptr,
                                                                       e->mc_row, e->mc_val, e->d_tz);
            KR_CK_LAUNCH();
            e->launches++;
        }
    }
}

}  // namespace

void engine_ax(kr_engine* e, const double* x, double* y, cudaStream_t s) {
    if (e->mkind == 3) throw Fail{KR_CONTRACT, e->mfail};
    launch_spmv(e, e->VT, x, nullptr, 0, e->d_tz, s);    // t = V^T x       engine.hpp:65-72
    solve_forward(e, s);                                 // z = M^-1 t      engine.hpp:74-78
    launch_spmv(e, e->UA, e->d_tz, x, e->k, y, s);       // y = U z + Ahat x  engine.hpp:81-89
    e->flops_last = e->flops_per_product;
    e->flops_total += e->flops_last;
}

void engine_atx(kr_engine* e, const double* y, double* x, cudaStream_t s) {
    if (e->mkind == 3) throw Fail{KR_CONTRACT, e->mfail};
    launch_spmv(e, e->UT, y, nullptr, 0, e->d_tz, s);    // s = U^T y         engine.hpp:103-110
    solve_backward(e, s);                                // z = M^-T s        engine.hpp:112-115
    launch_spmv(e, e->AV, y, e->d_tz, e->rows, x, s);    // x = Ahat^T y + V z  engine.hpp:117-130
    e->flops_last = e->flops_per_product;
    e->flops_total += e->flops_last;
}

}  // namespace krb

using krb::Fail;
using krb::guarded;

extern "C" {

const char* kr_last_error(int* code) {
    if (code) *code = krb::g_code;
    return krb::g_msg.c_str();
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
        if (nx != e->cols)
            throw Fail{KR_INVALID_INPUT,
                       "matvec input has size " + std::to_string(nx) + ", expected " + std::to_string(e->cols)};
        if (ny != e->rows) throw Fail{KR_INVALID_INPUT, "matvec output has the wrong size"};
        KR_CK(cudaSetDevice(e->device));
        if (e->mkind == 3) throw Fail{KR_CONTRACT, e->mfail};
        KR_CK(cudaMemcpyAsync(e->d_in, x, 8 * size_t(nx), cudaMemcpyHostToDevice, e->stream));
        krb::engine_ax(e, e->d_in, e->d_out, e->stream);
        KR_CK(cudaMemcpyAsync(y, e->d_out, 8 * size_t(ny), cudaMemcpyDeviceToHost, e->stream));
        KR_CK(cudaStreamSynchronize(e->stream));
    });
}

int kr_engine_atx(kr_engine* e, const double* y, int64_t ny, double* x, int64_t nx) {
    return guarded([&] {
        if (!e) throw Fail{KR_INVALID_INPUT, "null engine"};
        if (ny != e->rows)
            throw Fail{KR_INVALID_INPUT,
                       "matvec input has size " + std::to_string(ny) + ", expected " + std::to_string(e->rows)};
        if (nx != e->cols) throw Fail{KR_INVALID_INPUT, "matvec output has the wrong size"};
        KR_CK(cudaSetDevice(e->device));
        if (e->mkind == 3) throw Fail{KR_CONTRACT, e->mfail};
        KR_CK(cudaMemcpyAsync(e->d_in, y, 8 * size_t(ny), cudaMemcpyHostToDevice, e->stream));
        krb::engine_atx(e, e->d_in, e->d_out, e->stream);
        KR_CK(cudaMemcpyAsync(x, e->d_out, 8 * size_t(nx), cudaMemcpyDeviceToHost, e->stream));
        KR_CK(cudaStreamSynchronize(e->stream));
    });
}

int kr_engine_ax_device(kr_engine* e, const double* x, double* y, void* stream) {
    return guarded([&] {
        if (!e || !x || !y) throw Fail{KR_INVALID_INPUT, "null argument"};
        KR_CK(cudaSetDevice(e->device));
        krb::engine_ax(e, x, y, stream ? static_cast<cudaStream_t>(stream) : e->stream);
    });
}

int kr_engine_atx_device(kr_engine* e, const double* y, double* x, void* stream) {
    return guarded([&] {
        if (!e || !x || !y) throw Fail{KR_INVALID_INPUT, "null argument"};
        KR_CK(cudaSetDevice(e->device));
        krb::engine_atx(e, y, x, stream ? static_cast<cudaStream_t>(stream) : e->stream);
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
