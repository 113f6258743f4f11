// kr_solver.cu — DCFR solver step on the B200 (reference solver.hpp:145-414).
//
// One DCFR iteration (solver.hpp:365-388) becomes:
//   g1 = A x2                      engine (kr_engine.cu)
//   k_player_step(P1, g1)          fused: cfrSweep (222-260) -> sequenceForm
//                                  (197-218) -> discount (262-264) ->
//                                  avg = (avg + x) * shrink (381-387)
//   g2 = A^T x1                    engine
//   k_player_step(P2, -g2)         same, gradient negated (solver.hpp:370)
// Fusing the discount and the averaging of player 1 into its own step is
// exact: the reference touches rt1 / avg1 nowhere between sequenceForm(rt1)
// and those updates.  Each thread owns one hand and replays the reference's
// per-hand treeplex walks in the same order, so with bitwise-equal gradients
// the regrets, strategies, averages and exploitability trace are bitwise
// equal to the reference.  A block stages its hands' gradient / regret rows
// in shared memory with coalesced loads (hand-major rows, as KronPayoff::flat
// lays them out, kron.hpp:124-126) and walks them there.
//
// Scalars that need pow() (discount factors, shrink) are computed on the host
// with std::pow exactly as the reference does and passed as kernel arguments.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kr_common.cuh"
#include "kr_jit.cuh"

struct kr_solver {
    kr_engine* eng = nullptr;
    int device = 0;
    int nboards = 0;
    int n[2] = {0, 0};
    int nnodes[2] = {0, 0};
    int maxActs = 0;
    int64_t H[2] = {0, 0};
    std::vector<int64_t> boardStart[2];  // host copy, hands prefix per board
    double pot = 0;
    int32_t* d_tree[2] = {nullptr, nullptr};  // [parent(nn) | aptr(nn+1) | aseq(na)]
    int32_t treeLen[2] = {0, 0};
    int32_t na[2] = {0, 0};      // actions (entries of action_seq)
    bool levelled[2] = {false, false};  // level tables appended (team step kernel)
    int nlev[2] = {0, 0};
    int team[2] = {4, 4};        // lanes per hand in k_player_team (2, 4 or 8), per player
    // the step compiled for each player's tree (kr_jit.cu), for update rule
    // jitRule[p]; host copies of the trees to recompile on kr_solver_set_rule
    krb::JitStep jit[2];
    int jitRule[2] = {-1, -1};
    std::string jitWhy[2];
    std::vector<int32_t> tPar[2], tPtr[2], tSeq[2];
    // board-half pipelining of the captured iteration (overlap_ok): the
    // steps run on ovSide beside the next half's product; gB holds g2 so the
    // two players' gradients never share a buffer while both are in flight
    // implicit-engine solves keep x and the gradients sequence-major per
    // board (k7seq): kron_product_seq runs without transposes and the
    // compiled step reads / writes that layout (jitSeq)
    bool k7seq = false;          // a sequence-major solve is running (seqMode 1: implicit, 2: Kronecker-factored)
    int seqMode = 0;
    krb::JitStep jitSeq[2];
    int jitSeqRule[2] = {-1, -1};
    double* xs[2] = {nullptr, nullptr};
    cudaStream_t ovSide = nullptr;
    cudaEvent_t ovEv[8] = {};
    double* gB = nullptr;
    int teamThreads = 128;       // threads per k_player_team block (KR_TEAM_THREADS: 64, 128 or 256)
    // graph replay of whole iterations (kr_solver_run without early stop):
    // per-iteration factors pos/neg/shrink and weightSum as device tables
    // indexed by the device counter d_cnt[0] (iteration), d_cnt[1] = checkpoints
    double* d_fac = nullptr;
    double* d_ws = nullptr;
    int* d_cnt = nullptr;
    bool graphs = true;
    int rule = 0;                // KR_RULE_*
    int64_t* d_bstart[2] = {nullptr, nullptr};
    double* regret[2] = {nullptr, nullptr};
    double* avg[2] = {nullptr, nullptr};
    double* x[2] = {nullptr, nullptr};
    double* g = nullptr;        // gradient scratch, max(rows, cols)
    double* a[2] = {nullptr, nullptr};  // normalised averages at checkpoints
    double* handval = nullptr;  // per-hand best-response values
    double* boardval = nullptr; // per-board sums
    // player 2's checkpoint best response runs beside player 1's on `side`
    // (own gradient / hand scratch; the engine's A^T y has its own scratch)
    double* g2 = nullptr;
    double* handval2 = nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t evFork = nullptr, evJoin = nullptr;
    bool brSerial = false;      // KR_BR_SERIAL: one after the other on the solver stream
    int* d_flag = nullptr;
    int nt[2] = {64, 64};       // hands per block of the step kernel
    int64_t launches = 0;
    // incremental state (kr_solver_begin / iterate / checkpoint)
    bool begun = false;
    double alpha = 1.5, beta = 0.0, gamma = 2.0;
    int t = 0;                  // iterations completed
    double weightSum = 0;       // solver.hpp:354, 384-387
    // multi-GPU (kr_solver_set_comm): this rank's boards are
    // [board0, board0 + nboards) of nbTotal; checkpoint values are
    // all-gathered (ckSend -> ckRecv, world x 2 x nbMax) and scattered into
    // global board order (k_ck_scatter), so traces cover every board.
    kr_comm* comm = nullptr;
    int world = 1, rank = 0, nbTotal = 0, nbMax = 0;
    double* ckSend = nullptr;
    double* ckRecv = nullptr;
    int32_t* d_bpre = nullptr;  // [world + 1] board prefix over the ranks
    int totalBoards() const { return comm ? nbTotal : nboards; }
};

namespace krb {
namespace {

constexpr int kMaxActions = 32;

struct Tree {
    const int32_t* parent;
    const int32_t* aptr;
    const int32_t* aseq;
};

__device__ __forceinline__ Tree tree_view(const int32_t* t, int nn) { return Tree{t, t + nn, t + 2 * nn + 1}; }

// regretMatch (solver.hpp:166-194), split so no per-action array is needed:
// rm_stats scans a node's regrets once; rm_prob then yields probs[a] from the
// action's regret with the same expressions (r / sumPos, 1.0 / ties).
struct RmStats {
    bool positive;
    double sumPos;  // when positive
    double cut;     // best - tol, when not positive
    double uniform; // 1.0 / ties, when not positive
};

__device__ __forceinline__ RmStats rm_stats(const double* R, int stride, const int32_t* seqs, int count) {
    double best = R[(seqs[0] - 1) * stride];
    double maxAbs = fabs(best);
    double sumPos = best > 0 ? 0.0 + best : 0.0;  // the same additions, in action order
    for (int a = 1; a < count; ++a) {
        const double r = R[(seqs[a] - 1) * stride];
        best = (best < r) ? r : best;  // std::max
        const double ar = fabs(r);
        maxAbs = (maxAbs < ar) ? ar : maxAbs;
        if (r > 0) sumPos += r;
    }
    const double tol = 1e-9 * (1 + maxAbs);
    RmStats st;
    st.positive = best > tol;
    st.sumPos = sumPos;
    st.cut = best - tol;
    st.uniform = 0;
    if (!st.positive) {
        int ties = 0;
        for (int a = 0; a < count; ++a)
            if (R[(seqs[a] - 1) * stride] >= st.cut) ++ties;
        st.uniform = 1.0 / ties;
    }
    return st;
}

__device__ __forceinline__ double rm_prob(const RmStats& st, double r) {
    if (st.positive) return r > 0 ? r / st.sumPos : 0.0;
    return r >= st.cut ? st.uniform : 0.0;
}

// mode 0: sequence form only (initial strategy, solver.hpp:363-364)
// mode 1: full DCFR player step (sweep, sequence form, discount, average)
__global__ void k_player_step(int mode, const int32_t* __restrict__ treeBuf, int nn, int n, int64_t H, int nt,
                              const double* __restrict__ g, int negate, double* __restrict__ regret,
                              double* __restrict__ xout, double* __restrict__ avg, double pos, double neg,
                              double shrink) {
    krb::pdl_entry();
    // Shared memory per hand: its regret row and its seqVal / reach row
    // (strided so consecutive threads hit consecutive banks).  The gradient
    // row is read straight from global memory (each element once); the
    // sequence-form strategy is the reach row itself (x[s-1] = reach[s]).
    extern __shared__ double sm[];
    const int stride = nt + 1;
    double* Rg = sm;                      // n x stride     : regrets
    double* V = Rg + n * stride;          // (n+1) x stride : seqVal / reach
    int32_t* T = reinterpret_cast<int32_t*>(V + (n + 1) * stride);
    const int tl = 2 * nn + 1;  // parent + aptr
    for (int q = threadIdx.x; q < tl; q += blockDim.x) T[q] = treeBuf[q];
    const int64_t h0 = int64_t(blockIdx.x) * nt;
    const int nh = int(lmin(nt, H - h0));
    const int64_t e0 = h0 * n;
    const int ne = nh * n;
    __syncthreads();
    const int na = T[2 * nn];  // aptr[nn]
    for (int q = threadIdx.x; q < na; q += blockDim.x) T[tl + q] = treeBuf[tl + q];
    // coalesced loads, 8 in flight per thread
    for (int q0 = threadIdx.x; q0 < ne; q0 += 8 * blockDim.x) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * blockDim.x;
            v[u] = q < ne ? regret[e0 + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * blockDim.x;
            if (q < ne) {
                const int hh = q / n, s = q - hh * n;
                Rg[s * stride + hh] = v[u];
            }
        }
    }
    __syncthreads();
    const Tree tr = tree_view(T, nn);
    const int t = threadIdx.x;
    if (t < nh) {
        double* R = Rg + t;
        double* Vt = V + t;
        const double* gh = g + (h0 + t) * n;
        if (mode == 1) {
            // cfrSweep (solver.hpp:227-245): bottom-up over the player's nodes
            for (int s = 0; s <= n; ++s) Vt[s * stride] = 0.0;
            // the gradient entries of node v-1 are loaded while node v is
            // processed (up to kPre actions per node in registers)
            constexpr int kPre = 8;
            double gnext[kPre];
            auto prefetch = [&](int v, double* dst) {
                if (v < 0) return;
                const int a0 = tr.aptr[v], cnt = tr.aptr[v + 1] - a0;
#pragma unroll
                for (int u = 0; u < kPre; ++u)
                    if (u < cnt) dst[u] = __ldg(gh + tr.aseq[a0 + u] - 1);
            };
            prefetch(nn - 1, gnext);
            for (int v = nn - 1; v >= 0; --v) {
                const int a0 = tr.aptr[v], cnt = tr.aptr[v + 1] - a0;
                const int32_t* seqs = tr.aseq + a0;
                double gcur[kPre];
#pragma unroll
                for (int u = 0; u < kPre; ++u) gcur[u] = gnext[u];
                prefetch(v - 1, gnext);
                const RmStats st = rm_stats(R, stride, seqs, cnt);
                double nodeVal = 0;
#pragma unroll
                for (int a = 0; a < kPre; ++a)
                    if (a < cnt) {
                        const int sq = seqs[a];
                        const double gv = negate ? -gcur[a] : gcur[a];
                        const double ev = gv + Vt[sq * stride];
                        Vt[sq * stride] = ev;
                        nodeVal += rm_prob(st, R[(sq - 1) * stride]) * ev;
                    }
                for (int a = kPre; a < cnt; ++a) {
                    const int sq = seqs[a];
                    const double gv = negate ? -__ldg(gh + sq - 1) : __ldg(gh + sq - 1);
                    const double ev = gv + Vt[sq * stride];
                    Vt[sq * stride] = ev;
                    nodeVal += rm_prob(st, R[(sq - 1) * stride]) * ev;
                }
                for (int a = 0; a < cnt; ++a) {
                    const int sq = seqs[a];
                    R[(sq - 1) * stride] += Vt[sq * stride] - nodeVal;
                }
                Vt[tr.parent[v] * stride] += nodeVal;
            }
        }
        // sequenceForm (solver.hpp:202-215): top-down reach
        Vt[0] = 1.0;
        for (int v = 0; v < nn; ++v) {
            const int a0 = tr.aptr[v], cnt = tr.aptr[v + 1] - a0;
            const int32_t* seqs = tr.aseq + a0;
            const RmStats st = rm_stats(R, stride, seqs, cnt);
            const double mass = Vt[tr.parent[v] * stride];
            for (int a = 0; a < cnt; ++a) {
                const int sq = seqs[a];
                Vt[sq * stride] = mass * rm_prob(st, R[(sq - 1) * stride]);
            }
        }
        if (mode == 1)  // discount (solver.hpp:262-264)
            for (int s = 0; s < n; ++s) {
                const double r = R[s * stride];
                R[s * stride] = r * (r > 0 ? pos : neg);
            }
    }
    __syncthreads();
    for (int q0 = threadIdx.x; q0 < ne; q0 += 8 * blockDim.x) {
        double a[8];
        if (mode == 1) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int q = q0 + u * blockDim.x;
                a[u] = q < ne ? avg[e0 + q] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * blockDim.x;
            if (q < ne) {
                const int hh = q / n, s = q - hh * n;
                const double xv = V[(s + 1) * stride + hh];
                xout[e0 + q] = xv;
                if (mode == 1) {
                    regret[e0 + q] = Rg[s * stride + hh];
                    avg[e0 + q] = (a[u] + xv) * shrink;  // solver.hpp:382-386
                }
            }
        }
    }
}

// The same player step with a team of kTeam lanes per hand: the treeplex is
// walked level by level (its own-decision depth, 2-3 levels for river trees)
// and the lanes of a team take the nodes of a level in parallel.  Bitwise
// identical to k_player_step: every node performs the reference's per-node
// arithmetic in the same order, and the bottom-up accumulation of child node
// values into a sequence (Vt[parent] += nodeVal, solver.hpp:243, in
// descending node order) is replaced by pulling the children's values in
// that same descending order when the sequence's own node is processed.
// Needs every node's parent sequence to belong to an earlier node (true for
// the reference's skeleton); the host checks it and otherwise uses
// k_player_step.  Level tables follow the base tree in treeBuf:
//   nlev | levPtr[nlev+1] | levNodes[nn] | chPtr[n+2] | chNodes[...]
// (chNodes: per sequence its child nodes, descending).
template <int kTeam>
__global__ void __launch_bounds__(256) k_player_team(int mode, const int32_t* __restrict__ treeBuf, int nn, int n,
                                                     int na, int tlen, int64_t H, int hpb,
                                                     const double* __restrict__ g, int negate,
                                                     double* __restrict__ regret, double* __restrict__ xout,
                                                     double* __restrict__ avg, double pos, double neg, double shrink,
                                                     int rule, const double* __restrict__ fac,
                                                     const int* __restrict__ dt, int noAvg = 0,
                                                     double* __restrict__ rootOut = nullptr,
                                                     const double* __restrict__ extra = nullptr) {
    krb::pdl_entry();
    // noAvg: leave avg alone (river blocks of a turn game are averaged after
    // their reach is scaled); rootOut: each hand's root value (the sum of its
    // root nodes' values, descending node order: seqVal[0] of cfrSweep);
    // extra: values added to each sequence after its children (the river
    // subgames below a turn sequence).  Hand h, sequence s: extra[h*n + s-1].
    extern __shared__ double sm[];
    const int stride = hpb + 1;
    if (fac) {  // graph replay: this iteration's factors from the device table
        const int t = *dt;
        pos = fac[3 * t];
        neg = fac[3 * t + 1];
        shrink = fac[3 * t + 2];
    }
    double* Rg = sm;                      // n x stride      regrets
    double* V = Rg + n * stride;          // (n+1) x stride  gradient -> values -> probabilities -> reach
    double* NV = V + (n + 1) * stride;    // nn x stride     node values
    int32_t* T = reinterpret_cast<int32_t*>(NV + nn * stride);
    KR_SMEM_CHECK(0, sizeof(double) * size_t(2 * n + 1 + nn) * stride + sizeof(int32_t) * size_t(tlen));
    KR_DCHECK(int(blockDim.x) / kTeam >= hpb);
    for (int q = threadIdx.x; q < tlen; q += blockDim.x) T[q] = treeBuf[q];
    const int64_t h0 = int64_t(blockIdx.x) * hpb;
    const int nh = int(lmin(hpb, H - h0));
    const int64_t e0 = h0 * n;
    const int ne = nh * n;
    // element q = hh * n + sq of the block's rows; the thread's position is
    // advanced by blockDim.x without divisions
    const int dh = int(blockDim.x) / n, ds = int(blockDim.x) - dh * n;
    const int hh0 = int(threadIdx.x) / n, sq0 = int(threadIdx.x) - hh0 * n;
    // coalesced staging: regrets, and (mode 1) the gradient rows into V[1..n]
    {
        int hh = hh0, sq = sq0;
        for (int q0 = threadIdx.x; q0 < ne; q0 += 4 * blockDim.x) {
            double r[4], gv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // loads first: 4 (8) in flight
                const int q = q0 + u * int(blockDim.x);
                r[u] = q < ne ? regret[e0 + q] : 0.0;
                gv[u] = (mode == 1 && q < ne) ? g[e0 + q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (q0 + u * int(blockDim.x) < ne) {
                    Rg[sq * stride + hh] = r[u];
                    V[(sq + 1) * stride + hh] = gv[u];
                }
                hh += dh;
                sq += ds;
                if (sq >= n) {
                    sq -= n;
                    ++hh;
                }
            }
        }
    }
    __syncthreads();
    const Tree tr = tree_view(T, nn);
    const int32_t* lv = T + 2 * nn + 1 + na;  // nlev, levPtr, levNodes, chPtr, chNodes, levSeqPtr, levSeq, seqPar
    const int nlev = lv[0];
    const int32_t* levPtr = lv + 1;
    const int32_t* levNodes = levPtr + nlev + 1;
    const int32_t* chPtr = levNodes + nn;
    const int32_t* chNodes = chPtr + n + 2;
    const int32_t* levSeqPtr = chNodes + chPtr[n + 1];
    const int32_t* levSeq = levSeqPtr + nlev + 1;
    const int32_t* seqPar = levSeq + n;  // parent sequence of each sequence's node (by sequence id - 1)
    const int hand = threadIdx.x / kTeam, lane = threadIdx.x % kTeam;
    const bool valid = hand < nh;
    double* R = Rg + hand;
    double* Vt = V + hand;
    double* Nt = NV + hand;
    if (mode == 1) {
        // cfrSweep (solver.hpp:227-245), deepest level first.  Once a node's
        // regrets are final its sequenceForm probabilities (solver.hpp:
        // 202-215 reads exactly these regrets) replace the values in V.
        for (int l = nlev - 1; l >= 0; --l) {
            if (valid)
                for (int k = levPtr[l] + lane; k < levPtr[l + 1]; k += kTeam) {
                    const int v = levNodes[k];
                    KR_DCHECK(v >= 0 && v < nn);
                    const int a0 = tr.aptr[v], cnt = tr.aptr[v + 1] - a0;
                    const int32_t* seqs = tr.aseq + a0;
                    KR_DCHECK(cnt >= 1 && seqs[0] >= 1 && seqs[cnt - 1] <= n);
                    const RmStats st = rm_stats(R, stride, seqs, cnt);
                    double nodeVal = 0;
                    for (int a = 0; a < cnt; ++a) {
                        const int sq = seqs[a];
                        double cs = 0.0;  // Vt[sq] of the reference: children, descending
                        for (int c = chPtr[sq]; c < chPtr[sq + 1]; ++c) cs += Nt[chNodes[c] * stride];
                        if (extra) cs += extra[(h0 + hand) * n + sq - 1];
                        const double gr = Vt[sq * stride];
                        const double gv = negate ? -gr : gr;
                        const double ev = gv + cs;
                        Vt[sq * stride] = ev;
                        nodeVal += rm_prob(st, R[(sq - 1) * stride]) * ev;
                    }
                    for (int a = 0; a < cnt; ++a) {
                        const int sq = seqs[a];
                        const double d = Vt[sq * stride] - nodeVal;  // instantaneous regret
                        R[(sq - 1) * stride] += d;
                        if (rule == 2) Vt[sq * stride] = d;
                    }
                    Nt[v * stride] = nodeVal;
                    if (rule != 0)  // CFR+ / PRM+: discount before the strategy
                        for (int a = 0; a < cnt; ++a) {
                            double* rp = R + (seqs[a] - 1) * stride;
                            const double r = *rp;
                            *rp = r * (r > 0 ? pos : neg);
                        }
                    if (rule == 2) {  // PRM+: match R + d
                        for (int a = 0; a < cnt; ++a) {
                            const int sq = seqs[a];
                            Vt[sq * stride] = R[(sq - 1) * stride] + Vt[sq * stride];
                        }
                        const RmStats st2 = rm_stats(Vt + stride, stride, seqs, cnt);
                        for (int a = 0; a < cnt; ++a) {
                            const int sq = seqs[a];
                            Vt[sq * stride] = rm_prob(st2, Vt[sq * stride]);
                        }
                    } else {
                        const RmStats st2 = rm_stats(R, stride, seqs, cnt);
                        for (int a = 0; a < cnt; ++a) {
                            const int sq = seqs[a];
                            Vt[sq * stride] = rm_prob(st2, R[(sq - 1) * stride]);
                        }
                    }
                }
            __syncwarp();
        }
        if (rootOut && valid && lane == 0) {  // seqVal[0]: root nodes, descending
            double acc = 0.0;
            for (int k = levPtr[1] - 1; k >= levPtr[0]; --k) acc += Nt[levNodes[k] * stride];
            rootOut[h0 + hand] = acc;
        }
        // sequenceForm: reach = mass * prob, root level first, lanes over sequences
        if (valid && lane == 0) Vt[0] = 1.0;
        __syncwarp();
        for (int l = 0; l < nlev; ++l) {
            if (valid)
                for (int k = levSeqPtr[l] + lane; k < levSeqPtr[l + 1]; k += kTeam) {
                    const int sq = levSeq[k];
                    Vt[sq * stride] = Vt[seqPar[sq - 1] * stride] * Vt[sq * stride];
                }
            __syncwarp();
        }
        if (valid && rule == 0)  // discount (solver.hpp:262-264)
            for (int q = lane; q < n; q += kTeam) {
                const double r = R[q * stride];
                R[q * stride] = r * (r > 0 ? pos : neg);
            }
    } else {
        // sequenceForm only (initial strategy, solver.hpp:363-364)
        if (valid && lane == 0) Vt[0] = 1.0;
        __syncwarp();
        for (int l = 0; l < nlev; ++l) {
            if (valid)
                for (int k = levPtr[l] + lane; k < levPtr[l + 1]; k += kTeam) {
                    const int v = levNodes[k];
                    const int a0 = tr.aptr[v], cnt = tr.aptr[v + 1] - a0;
                    const int32_t* seqs = tr.aseq + a0;
                    const RmStats st = rm_stats(R, stride, seqs, cnt);
                    const double mass = Vt[tr.parent[v] * stride];
                    for (int a = 0; a < cnt; ++a) {
                        const int sq = seqs[a];
                        Vt[sq * stride] = mass * rm_prob(st, R[(sq - 1) * stride]);
                    }
                }
            __syncwarp();
        }
    }
    __syncthreads();
    {
        int hh = hh0, sq = sq0;
        for (int q0 = threadIdx.x; q0 < ne; q0 += 4 * blockDim.x) {
            double a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u * int(blockDim.x);
                a[u] = (mode == 1 && !noAvg && q < ne) ? avg[e0 + q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u * int(blockDim.x);
                if (q < ne) {
                    const double xv = V[(sq + 1) * stride + hh];
                    xout[e0 + q] = xv;
                    if (mode == 1) {
                        regret[e0 + q] = Rg[sq * stride + hh];
                        if (!noAvg) avg[e0 + q] = (a[u] + xv) * shrink;  // solver.hpp:382-386
                    }
                }
                hh += dh;
                sq += ds;
                if (sq >= n) {
                    sq -= n;
                    ++hh;
                }
            }
        }
    }
}

// Device-side counters of a replayed graph: c[which] += 1.
__global__ void k_tick(int* c, int which) { krb::pdl_entry(); c[which] += 1; }

size_t team_smem(int n, int nn, int hpb, int tlen) {
    return size_t(2 * n + 1 + nn) * size_t(hpb + 1) * 8 + size_t(tlen) * 4 + 16;
}

__global__ void k_normalise(const double* __restrict__ avg, int64_t n, double w, double* __restrict__ out,
                            const double* __restrict__ wsArr, const int* __restrict__ dt) {
    krb::pdl_entry();
    if (wsArr) w = wsArr[*dt];  // graph replay: weightSum of this iteration
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q < n) out[q] = avg[q] / w;  // solver.hpp:390-391
}

// Both players' averages in one launch: elements [0, n0) of avg0, then
// [0, n1) of avg1 (the same division as k_normalise).
__global__ void k_normalise2(const double* __restrict__ avg0, int64_t n0, double* __restrict__ out0,
                             const double* __restrict__ avg1, int64_t n1, double* __restrict__ out1, double w,
                             const double* __restrict__ wsArr, const int* __restrict__ dt) {
    krb::pdl_entry();
    if (wsArr) w = wsArr[*dt];
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q < n0) out0[q] = avg0[q] / w;  // solver.hpp:390-391
    else if (q < n0 + n1) out1[q - n0] = avg1[q - n0] / w;
}

// bestResponseValue per hand (solver.hpp:304-318): bottom-up max walk.
__global__ void k_best_response(const int32_t* __restrict__ treeBuf, int nn, int n, int64_t H,
                                const double* __restrict__ g, int negate, double* __restrict__ handval,
                                const double* __restrict__ extra = nullptr) {
    krb::pdl_entry();
    extern __shared__ int32_t Ts[];
    const int tl = 2 * nn + 1;
    for (int q = threadIdx.x; q < tl; q += blockDim.x) Ts[q] = treeBuf[q];
    __syncthreads();
    const int na = Ts[2 * nn];
    for (int q = threadIdx.x; q < na; q += blockDim.x) Ts[tl + q] = treeBuf[tl + q];
    double* seqVal = reinterpret_cast<double*>(Ts + ((tl + na + 1) & ~1));
    __syncthreads();
    const Tree tr = tree_view(Ts, nn);
    const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (h >= H) return;
    double* sv = seqVal + threadIdx.x;
    const int st = blockDim.x;
    for (int s = 0; s <= n; ++s) sv[s * st] = 0.0;
    const double* gh = g + h * n;
    for (int v = nn - 1; v >= 0; --v) {
        double best = 0;
        bool first = true;
        for (int a = tr.aptr[v]; a < tr.aptr[v + 1]; ++a) {
            const int sq = tr.aseq[a];
            const double gv = negate ? -gh[sq - 1] : gh[sq - 1];
            const double cs = extra ? sv[sq * st] + extra[h * n + sq - 1] : sv[sq * st];
            const double ev = gv + cs;
            if (first || ev > best) best = ev;
            first = false;
        }
        sv[tr.parent[v] * st] += best;
    }
    handval[h] = sv[0];
}

// Per-board totals in ascending hand order (solver.hpp:318 `total += ...`).
// One block per board: the block stages chunks of the board's hand values in
// shared memory with coalesced loads; thread 0 adds them in hand order.
constexpr int kSumChunk = 2048;
__global__ void __launch_bounds__(256) k_board_sums(const double* __restrict__ handval,
                                                    const int64_t* __restrict__ bstart, int nb,
                                                    double* __restrict__ out, const int* __restrict__ slot,
                                                    int64_t slotStride) {
    krb::pdl_entry();
    __shared__ double buf[kSumChunk];
    if (slot) out += int64_t(*slot) * slotStride;  // graph replay: this checkpoint's slot
    const int b = blockIdx.x;
    if (b >= nb) return;
    double total = 0;
    for (int64_t h0 = bstart[b]; h0 < bstart[b + 1]; h0 += kSumChunk) {
        const int n = int(lmin(kSumChunk, bstart[b + 1] - h0));
        for (int q = threadIdx.x; q < n; q += blockDim.x) buf[q] = handval[h0 + q];
        __syncthreads();
        if (threadIdx.x == 0) {
            int q = 0;
            for (; q + 8 <= n; q += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = buf[q + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) total += v[u];
            }
            for (; q < n; ++q) total += buf[q];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b] = total;
}

// The all-gathered checkpoint values (rank r: [2][nbMax], its first
// bpre[r+1]-bpre[r] entries valid) into global board order:
// dst[half * nbT + board], at checkpoint slot *slot when given.
__global__ void k_ck_scatter(const double* __restrict__ recv, int world, int nbMax, const int32_t* __restrict__ bpre,
                             double* __restrict__ dst, const int* __restrict__ slot, int64_t slotStride) {
    krb::pdl_entry();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= world * 2 * nbMax) return;
    const int r = q / (2 * nbMax), rem = q - r * 2 * nbMax, half = rem / nbMax, b = rem - half * nbMax;
    if (b >= bpre[r + 1] - bpre[r]) return;
    const int nbT = bpre[world];
    if (slot) dst += int64_t(*slot) * slotStride;
    dst[int64_t(half) * nbT + bpre[r] + b] = recv[q];
}

// validateSequenceStrategy (solver.hpp:266-286): flag 1 = negative entry,
// 2 = flow conservation violated.
__global__ void k_validate(const int32_t* __restrict__ treeBuf, int nn, int n, int64_t H,
                           const double* __restrict__ x, double tol, int* __restrict__ flag) {
    krb::pdl_entry();
    const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (h >= H) return;
    const Tree tr = tree_view(treeBuf, nn);
    const double* xh = x + h * n;
    for (int s = 0; s < n; ++s)
        if (xh[s] < -tol) atomicOr(flag, 1);
    for (int v = 0; v < nn; ++v) {
        const int p = tr.parent[v];
        const double parentMass = p == 0 ? 1.0 : xh[p - 1];
        double sum = 0;
        for (int a = tr.aptr[v]; a < tr.aptr[v + 1]; ++a) sum += xh[tr.aseq[a] - 1];
        if (fabs(sum - parentMass) > tol * (1 + fabs(parentMass))) atomicOr(flag, 2);
    }
}

// Level tables for k_player_team (appended to the base tree buffer), when
// every node's parent sequence belongs to an earlier node.
void append_levels(const kr_treeplex& t, std::vector<int32_t>& buf, bool& ok, int& nlev) {
    const int nn = t.n_nodes, n = t.n_seq;
    std::vector<int32_t> owner(size_t(n) + 1, -1), lev(size_t(nn), 0);
    for (int v = 0; v < nn; ++v)
        for (int a = t.node_action_ptr[v]; a < t.node_action_ptr[v + 1]; ++a) owner[size_t(t.action_seq[a])] = v;
    ok = true;
    nlev = 0;
    for (int v = 0; v < nn; ++v) {
        const int ps = t.node_parent_seq[v];
        if (ps == 0) lev[size_t(v)] = 0;
        else if (owner[size_t(ps)] >= 0 && owner[size_t(ps)] < v) lev[size_t(v)] = lev[size_t(owner[size_t(ps)])] + 1;
        else {
            ok = false;
            return;
        }
        nlev = std::max(nlev, lev[size_t(v)] + 1);
    }
    std::vector<int32_t> levPtr(size_t(nlev) + 1, 0), levNodes;
    for (int v = 0; v < nn; ++v) levPtr[size_t(lev[size_t(v)]) + 1]++;
    for (int l = 0; l < nlev; ++l) levPtr[size_t(l) + 1] += levPtr[size_t(l)];
    for (int l = 0; l < nlev; ++l)
        for (int v = 0; v < nn; ++v)
            if (lev[size_t(v)] == l) levNodes.push_back(v);
    std::vector<int32_t> chPtr(size_t(n) + 2, 0), chNodes;
    for (int sq = 0; sq <= n; ++sq) {
        chPtr[size_t(sq)] = int32_t(chNodes.size());
        for (int v = nn - 1; v >= 0; --v)
            if (t.node_parent_seq[v] == sq) chNodes.push_back(v);
    }
    chPtr[size_t(n) + 1] = int32_t(chNodes.size());
    // sequences by level of their node, and each sequence's parent sequence
    std::vector<int32_t> levSeqPtr(size_t(nlev) + 1, 0), levSeq, seqPar(size_t(n), 0);
    for (int l = 0; l < nlev; ++l) {
        for (int v : levNodes)
            if (lev[size_t(v)] == l)
                for (int a = t.node_action_ptr[v]; a < t.node_action_ptr[v + 1]; ++a) {
                    levSeq.push_back(t.action_seq[a]);
                    seqPar[size_t(t.action_seq[a]) - 1] = t.node_parent_seq[v];
                }
        levSeqPtr[size_t(l) + 1] = int32_t(levSeq.size());
    }
    buf.push_back(nlev);
    buf.insert(buf.end(), levPtr.begin(), levPtr.end());
    buf.insert(buf.end(), levNodes.begin(), levNodes.end());
    buf.insert(buf.end(), chPtr.begin(), chPtr.end());
    buf.insert(buf.end(), chNodes.begin(), chNodes.end());
    buf.insert(buf.end(), levSeqPtr.begin(), levSeqPtr.end());
    buf.insert(buf.end(), levSeq.begin(), levSeq.end());
    buf.insert(buf.end(), seqPar.begin(), seqPar.end());
}

// t^e / (t^e + 1) as the reference computes it (solver.hpp:378-379), with the
// limits 1 / 0 for e = +-inf (where std::pow would give inf / inf).
double discount_factor(int t, double e) {
    if (std::isinf(e)) return e > 0 ? 1.0 : 0.0;
    const double te = std::pow(double(t), e);
    return te / (te + 1);
}

size_t step_smem(int n, int nt, int nn, int na) {
    return size_t(2 * n + 1) * size_t(nt + 1) * 8 + size_t(2 * nn + 1 + na) * 4 + 16;
}

// Compile each player's step for the current update rule when it pays:
// grids of at least two CTAs per SM (smaller ones, single boards, keep the
// team kernel, whose lanes spread a few hundred hands over more threads);
// KR_STEP=jit forces it, KR_STEP=team / thread forbids it.
void jit_prepare(kr_solver* s) {
    const char* env = std::getenv("KR_STEP");
    const bool force = env && std::string(env) == "jit";
    for (int p = 0; p < 2; ++p) {
        if (!s->levelled[p] || s->jitRule[p] == s->rule) continue;
        s->jit[p] = JitStep{};
        s->jitRule[p] = -1;
        kr_treeplex t{};
        t.n_nodes = s->nnodes[p];
        t.n_seq = s->n[p];
        t.node_parent_seq = s->tPar[p].data();
        t.node_action_ptr = s->tPtr[p].data();
        t.action_seq = s->tSeq[p].data();
        // below two one-thread-per-hand CTAs per SM (single boards): the tree
        // split over warp groups (KR_JIT_GROUPS, 0 = the team kernel there)
        const bool small = !force && s->H[p] < int64_t(2) * 148 * kJitHands;
        int groups = 1;
        if (small) {
            const char* ge = std::getenv("KR_JIT_GROUPS");
            groups = ge ? std::atoi(ge) : 4;
            if (groups < 2) {
                s->jitWhy[p] = "grid below two CTAs per SM";
                continue;
            }
        }
        if (jit_step_compile(t, s->rule, s->jit[p], s->jitWhy[p], 0, groups)) {
            s->jitRule[p] = s->rule;
            s->jitWhy[p].clear();
            std::string why;
            s->jitSeq[p] = JitStep{};
            s->jitSeqRule[p] = -1;
            // implicit engines: sequence-major on full-GPU grids only (single
            // boards measured no gain: 26,523 -> 26,380 it/s at config 2);
            // Kronecker-factored: the staging layout at every size (config 2
            // 10,908 -> 11,708)
            const int lay = s->eng->kron ? (small ? 0 : 1) : s->eng->kf ? 2 : 0;
            if (lay && jit_step_compile(t, s->rule, s->jitSeq[p], why, lay, groups)) s->jitSeqRule[p] = s->rule;
        }
    }
}

// Sequence-major solves: the implicit engine keeps x and the gradients
// [seq][hand] per board (kron_product_seq, no transposes; KR_K7SEQ=0
// disables), the Kronecker-factored engine keeps x in its staging layout
// (kf_product_staged skips the per-product transpose; KR_KFSEQ=0 disables).
// Both players' compiled steps in the matching form; no SelfCheck (it
// compares hand-major products).
int seq_mode_for(const kr_solver* s) {
    const int mode = s->eng->kron ? 1 : s->eng->kf ? 2 : 0;
    if (!mode) return 0;
    if (const char* env = std::getenv(mode == 1 ? "KR_K7SEQ" : "KR_KFSEQ"))
        if (std::atoi(env) == 0) return 0;
    if (s->eng->scRef) return 0;
    for (int p = 0; p < 2; ++p)
        if (s->jitSeqRule[p] != s->rule || !s->jitSeq[p].kern || s->jitSeq[p].layout != mode) return 0;
    return mode;
}
bool k7seq_ok(const kr_solver* s) { return seq_mode_for(s) != 0; }

// player p's x as the input of the product that consumes it: player 1's
// feeds A^T (direction 1), player 2's feeds A (direction 0)
void enter_seq(kr_solver* s, cudaStream_t st) {
    const int mode = seq_mode_for(s);
    for (int p = 0; p < 2; ++p) {
        if (!s->xs[p]) s->xs[p] = dev_alloc<double>(std::max<int64_t>(s->H[p] * s->n[p], 1));
        const int dir = p == 0 ? 1 : 0;
        if (mode == 1) kron_transpose(s->eng, dir, 0, s->x[p], s->xs[p], true, st);
        else kf_stage_all(s->eng, dir, s->x[p], s->xs[p], st);
    }
    s->k7seq = true;
    s->seqMode = mode;
}

// the staging layout back to hand-major: out[h n + q] = in[q H + h]
__global__ void k_unstage(const double* __restrict__ in, double* __restrict__ out, int64_t H, int n) {
    pdl_entry();
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= H * n) return;
    const int64_t h = i / n;
    const int q = int(i - h * n);
    out[i] = in[int64_t(q) * H + h];
}

void leave_seq(kr_solver* s, cudaStream_t st) {
    if (!s->k7seq) return;
    for (int p = 0; p < 2; ++p) {
        if (s->seqMode == 1) {
            kron_transpose(s->eng, p == 0 ? 1 : 0, 0, s->xs[p], s->x[p], false, st);
        } else {
            const int64_t len = s->H[p] * s->n[p];
            if (len > 0) {
                krb::launch(k_unstage, unsigned((len + 255) / 256), 256, 0, st, s->xs[p], s->x[p], s->H[p], s->n[p]);
                KR_CK_LAUNCH();
                s->launches++;
            }
        }
    }
    s->k7seq = false;
    s->seqMode = 0;
}


// Player p's step over hands [hoff, hoff + hcnt) (all hands: hcnt < 0); g
// is the gradient of those hands' rows.
void launch_step(kr_solver* s, int p, int mode, const double* g, int negate, double pos, double neg, double shrink,
                 cudaStream_t st, bool dev = false, int64_t hoff = 0, int64_t hcnt = -1) {
    const int64_t H = hcnt < 0 ? s->H[p] : hcnt;
    const int64_t o = hoff * s->n[p];
    double *regret = s->regret[p] + o, *x = s->x[p] + o, *avg = s->avg[p] + o;
    if (mode == 1 && s->jit[p].kern && s->jitRule[p] == s->rule) {
        jit_step_launch(s->jit[p], s->device, H, g, negate, regret, x, avg, pos, neg, shrink,
                        dev ? s->d_fac : nullptr, dev ? s->d_cnt : nullptr, 0, nullptr, nullptr, st, nullptr, 0,
                        hcnt < 0 ? jit_stagger_ns() : 0);
        s->launches++;
        return;
    }
    if (s->levelled[p]) {
        const int team = s->team[p], threads = s->teamThreads;
        const int hpb = threads / team;
        const unsigned grid = unsigned((H + hpb - 1) / hpb);
        if (grid == 0) return;
        const size_t smem = team_smem(s->n[p], s->nnodes[p], hpb, s->treeLen[p]);
        auto kern = team == 2 ? k_player_team<2> : team == 4 ? k_player_team<4> : k_player_team<8>;
        krb::launch_pdl(true, kern, grid, threads, smem, st, mode, s->d_tree[p], s->nnodes[p], s->n[p], s->na[p],
                        s->treeLen[p], H, hpb, g, negate, regret, x, avg, pos, neg, shrink, s->rule,
                        dev ? s->d_fac : nullptr, dev ? s->d_cnt : nullptr, 0, nullptr, nullptr);
        KR_CK_LAUNCH();
        s->launches++;
        return;
    }
    if (s->rule != 0) throw Fail{KR_INVALID_INPUT, "update rule needs a reference-ordered treeplex"};
    if (dev) throw Fail{KR_CUDA, "internal: graph replay needs the team step kernel"};
    const int nt = s->nt[p];
    const unsigned grid = unsigned((H + nt - 1) / nt);
    if (grid == 0) return;
    const int na = s->na[p];
    const size_t smem = step_smem(s->n[p], nt, s->nnodes[p], na);
    krb::launch(k_player_step, grid, nt, smem, st, mode, s->d_tree[p], s->nnodes[p], s->n[p], H, nt, g, negate,
                regret, x, avg, pos, neg, shrink);
    KR_CK_LAUNCH();
    s->launches++;
}

// One DCFR iteration's products and steps (solver.hpp:365-388); dev: the
// scalars from the device tables (graph replay).
void iteration_body(kr_solver* s, cudaStream_t st, double pos, double neg, double shrink, bool dev) {
    kr_engine* e = s->eng;
    if (s->k7seq) {
        for (int p = 0; p < 2; ++p) {
            if (s->seqMode == 1) kron_product_seq(e, p, s->xs[1 - p], s->g, st);   // g1 = A x2, A^T x1
            else kf_product_staged(e, p, s->xs[1 - p], s->g, st);
            engine_account(e, p);
            jit_step_launch(s->jitSeq[p], s->device, s->H[p], s->g, p, s->regret[p], s->xs[p], s->avg[p], pos, neg,
                            shrink, dev ? s->d_fac : nullptr, dev ? s->d_cnt : nullptr, 0, nullptr, nullptr, st,
                            s->d_bstart[p], s->nboards, jit_stagger_ns());
            s->launches++;
        }
        return;
    }
    engine_ax(e, s->x[1], s->g, st);                               // g1 = A x2
    if (!dev) engine_selfcheck(e, 0, s->x[1], s->g, st);
    launch_step(s, 0, 1, s->g, 0, pos, neg, shrink, st, dev);      // P1 sweep/seqform/discount/avg
    engine_atx(e, s->x[0], s->g, st);                              // A^T x1
    if (!dev) engine_selfcheck(e, 1, s->x[0], s->g, st);
    launch_step(s, 1, 1, s->g, 1, pos, neg, shrink, st, dev);      // P2 with g2 = -A^T x1
}

// Best-response totals of `player` against device strategy `opp`; fills
// per-board values (host) and returns their sum.
// Per-board best-response totals of `player` against device strategy `opp`,
// written to device memory `dst` (nboards values), nothing synchronised.
void best_response_to(kr_solver* s, int player, const double* opp, double* dst, cudaStream_t st,
                      const int* slot = nullptr, int64_t slotStride = 0, double* g = nullptr,
                      double* handval = nullptr) {
    kr_engine* e = s->eng;
    if (!g) g = s->g;
    if (!handval) handval = s->handval;
    if (player == 0) engine_ax(e, opp, g, st);
    else engine_atx(e, opp, g, st);
    engine_selfcheck(e, player, opp, g, st);  // bestResponseValue calls eng.Ax / eng.ATx (solver.hpp:299)
    const int nn = s->nnodes[player], n = s->n[player];
    const int bt = 128;
    const int na = s->na[player];
    const size_t smem = size_t((2 * nn + 1 + na + 2) * 4) + size_t(n + 1) * bt * 8 + 16;
    const unsigned grid = unsigned((s->H[player] + bt - 1) / bt);
    if (grid) {
        krb::launch(k_best_response, grid, bt, smem, st, s->d_tree[player], nn, n, s->H[player], g, player == 1, handval,
                                                nullptr);
        KR_CK_LAUNCH();
        s->launches++;
    }
    krb::launch(k_board_sums, unsigned(s->nboards), 256, 0, st, handval, s->d_bstart[player], s->nboards, dst, slot,
                                                        slotStride);
    KR_CK_LAUNCH();
    s->launches++;
}

// Both checkpoint best responses (br1 vs avg2 into dst0, br2 vs avg1 into
// dst1): player 2's forks onto the solver's side stream and joins back, so
// the two products and walks overlap (inside a graph capture they become
// parallel branches).  Each has its own scratch, so the values are the bits
// of the serial order.
void best_responses(kr_solver* s, double* dst0, double* dst1, cudaStream_t st, const int* slot = nullptr,
                    int64_t slotStride = 0) {
    if (s->brSerial || !s->side) {
        best_response_to(s, 0, s->a[1], dst0, st, slot, slotStride);
        best_response_to(s, 1, s->a[0], dst1, st, slot, slotStride);
        return;
    }
    KR_CK(cudaEventRecord(s->evFork, st));
    KR_CK(cudaStreamWaitEvent(s->side, s->evFork, 0));
    best_response_to(s, 1, s->a[0], dst1, s->side, slot, slotStride, s->g2, s->handval2);
    best_response_to(s, 0, s->a[1], dst0, st, slot, slotStride);
    KR_CK(cudaEventRecord(s->evJoin, s->side));
    KR_CK(cudaStreamWaitEvent(st, s->evJoin, 0));
}

// One checkpoint's per-board best-response values in global board order,
// dst[0 .. nbT) = br1 (vs avg2), dst[nbT .. 2 nbT) = br2 (vs avg1), at slot
// *slot of stride slotStride when given.  With a communicator this rank's
// values are all-gathered in-stream and scattered into place on every rank.
void checkpoint_values(kr_solver* s, double* dst, cudaStream_t st, const int* slot = nullptr,
                       int64_t slotStride = 0) {
    if (!s->comm) {
        best_responses(s, dst, dst + s->nboards, st, slot, slotStride);
        return;
    }
    best_responses(s, s->ckSend, s->ckSend + s->nbMax, st);
    comm_allgather(s->comm, s->ckSend, s->ckRecv, size_t(2) * s->nbMax, st);
    const int n = s->world * 2 * s->nbMax;
    krb::launch(k_ck_scatter, unsigned((n + 255) / 256), 256, 0, st, s->ckRecv, s->world, s->nbMax, s->d_bpre, dst,
                slot, slotStride);
    KR_CK_LAUNCH();
    s->launches++;
}

// The same, copied to the host (synchronises the stream).
void best_response_dev(kr_solver* s, int player, const double* opp, std::vector<double>& boards, cudaStream_t st) {
    best_response_to(s, player, opp, s->boardval, st);
    boards.assign(size_t(s->nboards), 0.0);
    KR_CK(cudaMemcpyAsync(boards.data(), s->boardval, 8 * size_t(s->nboards), cudaMemcpyDeviceToHost, st));
    KR_CK(cudaStreamSynchronize(st));
}

void destroy_solver(kr_solver* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    if (s->ovSide) cudaStreamDestroy(s->ovSide);
    krb::dev_free(s->xs[0]);
    krb::dev_free(s->xs[1]);
    for (cudaEvent_t ev : s->ovEv)
        if (ev) cudaEventDestroy(ev);
    krb::dev_free(s->gB);
    for (int p = 0; p < 2; ++p) {
        krb::dev_free(s->d_tree[p]);
        krb::dev_free(s->d_bstart[p]);
        krb::dev_free(s->regret[p]);
        krb::dev_free(s->avg[p]);
        krb::dev_free(s->x[p]);
        krb::dev_free(s->a[p]);
    }
    krb::dev_free(s->d_fac);
    krb::dev_free(s->d_ws);
    krb::dev_free(s->d_cnt);
    krb::dev_free(s->g);
    krb::dev_free(s->handval);
    krb::dev_free(s->boardval);
    krb::dev_free(s->g2);
    krb::dev_free(s->handval2);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->evFork) cudaEventDestroy(s->evFork);
    if (s->evJoin) cudaEventDestroy(s->evJoin);
    krb::dev_free(s->d_flag);
    krb::dev_free(s->ckSend);
    krb::dev_free(s->ckRecv);
    krb::dev_free(s->d_bpre);
    delete s;
}

}  // namespace
}  // namespace krb

using krb::Fail;
using krb::guarded;

extern "C" {

int kr_solver_create(kr_engine* e, const kr_treeplex* p1, const kr_treeplex* p2, int nboards, const int32_t* hands1,
                     const int32_t* hands2, double pot, kr_solver** out) {
    return guarded([&] {
        if (!e || !p1 || !p2 || !hands1 || !hands2 || !out || nboards < 1)
            throw Fail{KR_INVALID_INPUT, "null argument to kr_solver_create"};
        if (!(pot > 0)) throw Fail{KR_INVALID_INPUT, "pot must be positive"};
        KR_CK(cudaSetDevice(e->device));
        auto* s = new kr_solver();
        try {
            s->eng = e;
            s->device = e->device;
            s->nboards = nboards;
            s->pot = pot;
            const kr_treeplex* tp[2] = {p1, p2};
            const int32_t* hands[2] = {hands1, hands2};
            // single-board engines: eight lanes per hand (their grids are a
            // few dozen blocks; config 2 measured 19,000 -> 22,500 K7 DCFR
            // it/s and 6,410 -> 6,850 factored, tools/config2_team_probe.py);
            // multi-board grids keep four (config 3: 2/4/8 within +-1.2%).
            // Read once, before the per-player fit below.
            int team0 = nboards == 1 ? 8 : 4;
            if (const char* env = std::getenv("KR_TEAM")) {
                const int tm = std::atoi(env);
                team0 = tm == 2 || tm == 8 ? tm : 4;
            }
            if (const char* env = std::getenv("KR_TEAM_THREADS")) {
                const int th = std::atoi(env);
                s->teamThreads = th == 64 || th == 256 ? th : 128;
            }
            for (int p = 0; p < 2; ++p) {
                const kr_treeplex& t = *tp[p];
                if (t.n_seq < 1 || t.n_nodes < 1) throw Fail{KR_INVALID_INPUT, "empty treeplex"};
                s->n[p] = t.n_seq;
                s->nnodes[p] = t.n_nodes;
                if (t.node_action_ptr[0] != 0) throw Fail{KR_INVALID_INPUT, "treeplex action_ptr[0] must be 0"};
                const int na = t.node_action_ptr[t.n_nodes];
                std::vector<char> seen(size_t(t.n_seq) + 1, 0);
                for (int v = 0; v < t.n_nodes; ++v) {
                    const int cnt = t.node_action_ptr[v + 1] - t.node_action_ptr[v];
                    if (cnt < 1 || cnt > krb::kMaxActions)
                        throw Fail{KR_INVALID_INPUT, "decision node action count out of range"};
                    if (t.node_parent_seq[v] < 0 || t.node_parent_seq[v] > t.n_seq)
                        throw Fail{KR_INVALID_INPUT, "parent sequence out of range"};
                    s->maxActs = std::max(s->maxActs, cnt);
                }
                for (int a = 0; a < na; ++a) {
                    const int sq = t.action_seq[a];
                    if (sq < 1 || sq > t.n_seq || seen[size_t(sq)]) throw Fail{KR_INVALID_INPUT, "bad action sequence id"};
                    seen[size_t(sq)] = 1;
                }
                s->tPar[p].assign(t.node_parent_seq, t.node_parent_seq + t.n_nodes);
                s->tPtr[p].assign(t.node_action_ptr, t.node_action_ptr + t.n_nodes + 1);
                s->tSeq[p].assign(t.action_seq, t.action_seq + na);
                std::vector<int32_t> buf;
                buf.insert(buf.end(), t.node_parent_seq, t.node_parent_seq + t.n_nodes);
                buf.insert(buf.end(), t.node_action_ptr, t.node_action_ptr + t.n_nodes + 1);
                buf.insert(buf.end(), t.action_seq, t.action_seq + na);
                s->na[p] = na;
                krb::append_levels(t, buf, s->levelled[p], s->nlev[p]);
                if (const char* env = std::getenv("KR_STEP"))
                    if (std::string(env) == "thread") s->levelled[p] = false;
                s->treeLen[p] = int32_t(buf.size());
                s->d_tree[p] = krb::dev_alloc<int32_t>(int64_t(buf.size()));
                KR_CK(cudaMemcpy(s->d_tree[p], buf.data(), 4 * buf.size(), cudaMemcpyHostToDevice));
                s->boardStart[p].assign(1, 0);
                for (int b = 0; b < nboards; ++b) {
                    if (hands[p][b] < 0) throw Fail{KR_INVALID_INPUT, "negative hand count"};
                    s->boardStart[p].push_back(s->boardStart[p].back() + hands[p][b]);
                }
                s->H[p] = s->boardStart[p].back();
                s->d_bstart[p] = krb::dev_alloc<int64_t>(nboards + 1);
                KR_CK(cudaMemcpy(s->d_bstart[p], s->boardStart[p].data(), 8 * size_t(nboards + 1),
                                 cudaMemcpyHostToDevice));
                // hands per block: largest multiple of 32 (<= 64) that fits
                int nt = 64;
                while (nt > 32 && krb::step_smem(t.n_seq, nt, t.n_nodes, na) > 200 * 1024) nt -= 32;
                if (krb::step_smem(t.n_seq, nt, t.n_nodes, na) > 220 * 1024)
                    throw Fail{KR_INVALID_INPUT, "treeplex too large for the on-chip solver step"};
                s->nt[p] = nt;
                // lanes per hand: the default (or KR_TEAM) raised, per player, until
                // that player's block fits the shared-memory budget; sized with the
                // launch's own hands per block (teamThreads / team)
                s->team[p] = team0;
                if (s->levelled[p]) {
                    while (s->team[p] < 8 &&
                           krb::team_smem(t.n_seq, t.n_nodes, s->teamThreads / s->team[p], s->treeLen[p]) > 200 * 1024)
                        s->team[p] *= 2;
                    const size_t tsm = krb::team_smem(t.n_seq, t.n_nodes, s->teamThreads / s->team[p], s->treeLen[p]);
                    if (tsm > 220 * 1024) s->levelled[p] = false;
                }
                const int64_t len = s->H[p] * s->n[p];
                s->regret[p] = krb::dev_alloc<double>(std::max<int64_t>(len, 1));
                s->avg[p] = krb::dev_alloc<double>(std::max<int64_t>(len, 1));
                s->x[p] = krb::dev_alloc<double>(std::max<int64_t>(len, 1));
                s->a[p] = krb::dev_alloc<double>(std::max<int64_t>(len, 1));
            }
            {
                size_t satt = 0;
                for (int p = 0; p < 2; ++p)
                    satt = std::max(satt, krb::step_smem(s->n[p], s->nt[p], s->nnodes[p], s->na[p]));
                krb::raise_smem_limit(krb::k_player_step, satt);
                // one attribute for both players (each with its own team size)
                size_t att = 48 * 1024;
                for (int p = 0; p < 2; ++p)
                    if (s->levelled[p])
                        att = std::max(att, krb::team_smem(s->n[p], s->nnodes[p], s->teamThreads / s->team[p],
                                                           s->treeLen[p]));
                krb::raise_smem_limit(krb::k_player_team<2>, att);
                krb::raise_smem_limit(krb::k_player_team<4>, att);
                krb::raise_smem_limit(krb::k_player_team<8>, att);
            }
            if (s->H[0] * s->n[0] != e->rows || s->H[1] * s->n[1] != e->cols)
                throw Fail{KR_INVALID_INPUT, "treeplex x hands does not match the engine dimensions"};
            s->g = krb::dev_alloc<double>(std::max<int64_t>(std::max(e->rows, e->cols), 1));
            s->handval = krb::dev_alloc<double>(std::max<int64_t>(std::max(s->H[0], s->H[1]), 1));
            s->boardval = krb::dev_alloc<double>(2 * int64_t(nboards));
            s->brSerial = std::getenv("KR_BR_SERIAL") != nullptr;
            if (!s->brSerial) {
                s->g2 = krb::dev_alloc<double>(std::max<int64_t>(std::max(e->rows, e->cols), 1));
                s->handval2 = krb::dev_alloc<double>(std::max<int64_t>(std::max(s->H[0], s->H[1]), 1));
                KR_CK(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
                KR_CK(cudaEventCreateWithFlags(&s->evFork, cudaEventDisableTiming));
                KR_CK(cudaEventCreateWithFlags(&s->evJoin, cudaEventDisableTiming));
            }
            s->d_flag = krb::dev_alloc<int>(1);
            const int bsm0 = int((2 * s->nnodes[0] + 1 + s->treeLen[0] + 4) * 4 + (s->n[0] + 1) * 128 * 8 + 16);
            const int bsm1 = int((2 * s->nnodes[1] + 1 + s->treeLen[1] + 4) * 4 + (s->n[1] + 1) * 128 * 8 + 16);
            krb::raise_smem_limit(krb::k_best_response, size_t(std::max(bsm0, bsm1)));
            krb::jit_prepare(s);
        } catch (...) {
            krb::destroy_solver(s);
            throw;
        }
        *out = s;
    });
}

int kr_solver_destroy(kr_solver* s) {
    return guarded([&] { krb::destroy_solver(s); });
}

int64_t kr_solver_launches(const kr_solver* s) { return s ? s->launches : 0; }

namespace {
void normalise_averages(kr_solver* s, cudaStream_t st, bool dev = false) {
    const int64_t n0 = s->H[0] * s->n[0], n1 = s->H[1] * s->n[1];
    if (n0 > 0 && n1 > 0) {
        krb::launch(krb::k_normalise2, unsigned((n0 + n1 + 255) / 256), 256, 0, st, s->avg[0], n0, s->a[0], s->avg[1],
                    n1, s->a[1], s->weightSum, dev ? s->d_ws : nullptr, dev ? s->d_cnt : nullptr);
        s->launches++;
        return;
    }
    for (int p = 0; p < 2; ++p) {
        const int64_t len = s->H[p] * s->n[p];
        if (len == 0) continue;
        krb::launch(krb::k_normalise, unsigned((len + 255) / 256), 256, 0, st, s->avg[p], len, s->weightSum, s->a[p],
                                                                      dev ? s->d_ws : nullptr,
                                                                      dev ? s->d_cnt : nullptr);
        KR_CK_LAUNCH();
        s->launches++;
    }
}
}  // namespace

namespace {
// Iterations t = s->t+1 .. maxIters by replaying two captured CUDA graphs:
// one DCFR iteration (tick, A x2, step 1, A^T x1, step 2) and the same plus
// a checkpoint (normalise, two best responses into checkpoint slot d_cnt[1],
// tick).  The per-iteration scalars come from device tables built here with
// the host loop's exact expressions (kr_solver_iterate), so a replayed
// iteration is bitwise the iteration kr_solver_iterate would launch.  The
// engine's and solver's flop / launch counters advance per replay.
// Counter deltas of one captured graph (added per replay).
struct GraphDelta {
    int64_t flops = 0, elaunch = 0, slaunch = 0;
};

// Capture one DCFR iteration (counter tick, A x2, step 1, A^T x1, step 2),
// plus a checkpoint when withCk (normalise, the two best responses into
// checkpoint slot d_cnt[1] of dck, tick): the scalars come from the device
// tables d_fac / d_ws indexed by the device counters.
// Board-half pipelining: every board is an independent block of A (the
// products and both players' steps are board-local), so the iteration runs
// as A x2 [half 0], A x2 [half 1] beside P1 [half 0], A^T x1 [half 0] beside
// P1 [half 1], ... : each step overlaps the other half's product (the
// products are shared-memory bound, the steps latency-bound).  Every board
// computes exactly what it computes in the serial order.  Multi-board
// implicit and Kronecker-factored engines, opt-in (KR_OVERLAP=1): measured
// slower at config 3 (K7 DCFR 5,055 -> 4,147 it/s, Kronecker-factored
// 1,323 -> 1,178): half-size product grids lose more to their tails than the
// steps gain beside them (profiles/r02/jit_step_probe_r02z.log).
bool overlap_ok(const kr_solver* s) {
    const char* env = std::getenv("KR_OVERLAP");
    if (!(env && std::atoi(env) == 1)) return false;
    return !s->k7seq && s->nboards >= 2 && (s->eng->kron || s->eng->kf) && krb::engine_boards(s->eng) == s->nboards;
}

void ensure_overlap(kr_solver* s) {
    if (s->ovSide) return;
    KR_CK(cudaStreamCreateWithFlags(&s->ovSide, cudaStreamNonBlocking));
    for (auto& ev : s->ovEv) KR_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    s->gB = krb::dev_alloc<double>(std::max<int64_t>(s->eng->cols, 1));
}

// One iteration's products and steps, board halves pipelined (graph capture).
void overlapped_iteration(kr_solver* s, cudaStream_t st) {
    kr_engine* e = s->eng;
    cudaStream_t T = s->ovSide;
    const int nb = s->nboards, bm = nb / 2;
    const int b[3] = {0, bm, nb};
    cudaEvent_t* ev = s->ovEv;
    KR_CK(cudaEventRecord(ev[0], st));
    KR_CK(cudaStreamWaitEvent(T, ev[0], 0));
    for (int p = 0; p < 2; ++p) {
        const double* in = s->x[1 - p];
        double* g = p == 0 ? s->g : s->gB;
        for (int h = 0; h < 2; ++h) {
            if (p == 1) KR_CK(cudaStreamWaitEvent(st, ev[2 + h], 0));   // x1 of this half is final
            if (!krb::engine_product_boards(e, p, in, g, st, b[h], b[h + 1]))
                throw Fail{KR_CUDA, "internal: board-range product on a factored engine"};
            KR_CK(cudaEventRecord(ev[4 + h], st));
            KR_CK(cudaStreamWaitEvent(T, ev[4 + h], 0));
            const int64_t h0 = s->boardStart[p][size_t(b[h])], h1 = s->boardStart[p][size_t(b[h + 1])];
            krb::launch_step(s, p, 1, g + h0 * s->n[p], p, 0.0, 0.0, 0.0, T, true, h0, h1 - h0);
            if (p == 0) KR_CK(cudaEventRecord(ev[2 + h], T));
        }
        krb::engine_account(e, p);
    }
    KR_CK(cudaEventRecord(ev[6], T));
    KR_CK(cudaStreamWaitEvent(st, ev[6], 0));
}

void capture_iteration(kr_solver* s, bool withCk, double* dck, cudaStream_t st, cudaGraphExec_t& exec,
                       GraphDelta& d) {
    kr_engine* e = s->eng;
    const bool ov = overlap_ok(s);
    if (ov) ensure_overlap(s);
    const int64_t f0 = e->flops_total, el0 = e->launches, sl0 = s->launches;
    cudaGraph_t g;
    KR_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
        krb::launch(krb::k_tick, 1, 1, 0, st, s->d_cnt, 0);
        KR_CK_LAUNCH();
        s->launches++;
        if (ov) {
            overlapped_iteration(s, st);
        } else {
            krb::iteration_body(s, st, 0.0, 0.0, 0.0, true);
        }
        if (withCk) {
            normalise_averages(s, st, true);                                     // solver.hpp:390-391
            krb::checkpoint_values(s, dck, st, s->d_cnt + 1, 2 * int64_t(s->totalBoards()));
            krb::launch(krb::k_tick, 1, 1, 0, st, s->d_cnt, 1);
            KR_CK_LAUNCH();
            s->launches++;
        }
    } catch (...) {
        cudaStreamEndCapture(st, &g);
        throw;
    }
    KR_CK(cudaStreamEndCapture(st, &g));
    const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    KR_CK(ie);
    d.flops = e->flops_total - f0;
    d.elaunch = e->launches - el0;
    d.slaunch = s->launches - sl0;
    e->flops_total = f0;
    e->launches = el0;
    s->launches = sl0;
}

// The device tables of iterations t = s->t + 1 .. maxIters, filled with the
// host loop's exact expressions (kr_solver_iterate), and the counters
// {d_cnt[0], d_cnt[1]} = {s->t, 0}.  Returns weightSum after each iteration.
std::vector<double> iteration_tables(kr_solver* s, int maxIters, cudaStream_t st) {
    const int t0 = s->t;
    std::vector<double> fac(size_t(3) * (maxIters + 1), 0.0), ws(size_t(maxIters) + 1, 0.0);
    double w = s->weightSum;
    ws[size_t(t0)] = w;
    for (int t = t0 + 1; t <= maxIters; ++t) {
        fac[3 * size_t(t)] = krb::discount_factor(t, s->alpha);
        fac[3 * size_t(t) + 1] = krb::discount_factor(t, s->beta);
        const double shrink = std::pow(double(t) / (t + 1), s->gamma);
        fac[3 * size_t(t) + 2] = shrink;
        w += 1;  // solver.hpp:384-387, as kr_solver_iterate
        w *= shrink;
        ws[size_t(t)] = w;
    }
    krb::dev_free(s->d_fac);
    krb::dev_free(s->d_ws);
    s->d_fac = s->d_ws = nullptr;
    s->d_fac = krb::dev_alloc<double>(int64_t(fac.size()));
    s->d_ws = krb::dev_alloc<double>(int64_t(ws.size()));
    if (!s->d_cnt) s->d_cnt = krb::dev_alloc<int>(2);
    KR_CK(cudaMemcpyAsync(s->d_fac, fac.data(), 8 * fac.size(), cudaMemcpyHostToDevice, st));
    KR_CK(cudaMemcpyAsync(s->d_ws, ws.data(), 8 * ws.size(), cudaMemcpyHostToDevice, st));
    const int cnt0[2] = {t0, 0};
    KR_CK(cudaMemcpyAsync(s->d_cnt, cnt0, sizeof(cnt0), cudaMemcpyHostToDevice, st));
    KR_CK(cudaStreamSynchronize(st));
    return ws;
}

bool graphs_ok(const kr_solver* s) {
    return s->graphs && s->levelled[0] && s->levelled[1] && !std::getenv("KR_NO_GRAPH") && !s->eng->scRef;
}

// Iterations t = s->t+1 .. maxIters by replaying two captured CUDA graphs:
// one DCFR iteration and the same plus a checkpoint into dck.  A replayed
// iteration is bitwise the iteration kr_solver_iterate would launch.  The
// engine's and solver's flop / launch counters advance per replay.
void run_graphs(kr_solver* s, int maxIters, int every, double* dck, std::vector<int>& at, cudaStream_t st) {
    kr_engine* e = s->eng;
    const int t0 = s->t;
    const std::vector<double> ws = iteration_tables(s, maxIters, st);
    const bool timing = e->timing;
    e->timing = false;
    cudaGraphExec_t gIt = nullptr, gCk = nullptr;
    GraphDelta dIt, dCk;
    try {
        capture_iteration(s, false, dck, st, gIt, dIt);
        capture_iteration(s, true, dck, st, gCk, dCk);
        for (int t = t0 + 1; t <= maxIters; ++t) {
            const bool isCk = t % every == 0 || t == maxIters;
            KR_CK(cudaGraphLaunch(isCk ? gCk : gIt, st));
            const GraphDelta& d = isCk ? dCk : dIt;
            e->flops_total += d.flops;
            e->launches += d.elaunch;
            s->launches += d.slaunch;
            if (isCk) at.push_back(t);
        }
        e->flops_last = e->kron ? krb::kron_flops(e, 1) : e->flops_per_product;
    } catch (...) {
        if (gIt) cudaGraphExecDestroy(gIt);
        if (gCk) cudaGraphExecDestroy(gCk);
        e->timing = timing;
        throw;
    }
    cudaGraphExecDestroy(gIt);
    cudaGraphExecDestroy(gCk);
    e->timing = timing;
    s->t = maxIters;
    s->weightSum = ws[size_t(maxIters)];
}

// kr_solver_iterate's n iterations as replays of one captured iteration graph.
void iterate_graph(kr_solver* s, int n, cudaStream_t st) {
    kr_engine* e = s->eng;
    const int t1 = s->t + n;
    const std::vector<double> ws = iteration_tables(s, t1, st);
    const bool timing = e->timing;
    e->timing = false;
    cudaGraphExec_t g = nullptr;
    GraphDelta d;
    try {
        capture_iteration(s, false, nullptr, st, g, d);
        for (int q = 0; q < n; ++q) {
            KR_CK(cudaGraphLaunch(g, st));
            e->flops_total += d.flops;
            e->launches += d.elaunch;
            s->launches += d.slaunch;
        }
        e->flops_last = e->kron ? krb::kron_flops(e, 1) : e->flops_per_product;
    } catch (...) {
        if (g) cudaGraphExecDestroy(g);
        e->timing = timing;
        throw;
    }
    cudaGraphExecDestroy(g);
    e->timing = timing;
    s->t = t1;
    s->weightSum = ws[size_t(t1)];
}
}  // namespace

int kr_solver_set_comm(kr_solver* s, kr_comm* c, const int32_t* boards_per_rank) {
    return guarded([&] {
        if (!s) throw Fail{KR_INVALID_INPUT, "null solver"};
        KR_CK(cudaSetDevice(s->device));
        krb::dev_free(s->ckSend);
        krb::dev_free(s->ckRecv);
        krb::dev_free(s->d_bpre);
        s->ckSend = s->ckRecv = nullptr;
        s->d_bpre = nullptr;
        s->comm = nullptr;
        s->world = 1;
        s->rank = 0;
        if (!c) return;
        if (!boards_per_rank) throw Fail{KR_INVALID_INPUT, "a communicator needs the boards of every rank"};
        const int world = krb::comm_size(c), rank = krb::comm_rank(c);
        if (krb::comm_device(c) != s->device) throw Fail{KR_INVALID_INPUT, "communicator and solver on different devices"};
        if (boards_per_rank[rank] != s->nboards) throw Fail{KR_INVALID_INPUT, "this rank's board count differs"};
        std::vector<int32_t> pre(size_t(world) + 1, 0);
        int nbMax = 0;
        for (int r = 0; r < world; ++r) {
            if (boards_per_rank[r] < 0) throw Fail{KR_INVALID_INPUT, "negative board count"};
            pre[size_t(r) + 1] = pre[size_t(r)] + boards_per_rank[r];
            nbMax = std::max(nbMax, int(boards_per_rank[r]));
        }
        s->world = world;
        s->rank = rank;
        s->nbTotal = pre[size_t(world)];
        s->nbMax = nbMax;
        s->ckSend = krb::dev_alloc<double>(2 * int64_t(nbMax));
        s->ckRecv = krb::dev_alloc<double>(2 * int64_t(nbMax) * world);
        s->d_bpre = krb::dev_alloc<int32_t>(world + 1);
        KR_CK(cudaMemcpy(s->d_bpre, pre.data(), 4 * pre.size(), cudaMemcpyHostToDevice));
        krb::dev_free(s->boardval);  // checkpoint values in global order: 2 x nbTotal
        s->boardval = nullptr;
        s->boardval = krb::dev_alloc<double>(2 * int64_t(std::max(s->nbTotal, s->nboards)));
        s->comm = c;
    });
}

int kr_solver_set_rule(kr_solver* s, int rule) {
    return guarded([&] {
        if (!s) throw Fail{KR_INVALID_INPUT, "null solver"};
        if (rule < 0 || rule > 2) throw Fail{KR_INVALID_INPUT, "unknown update rule"};
        if (rule != 0 && !(s->levelled[0] && s->levelled[1]))
            throw Fail{KR_INVALID_INPUT, "update rule needs a reference-ordered treeplex"};
        s->rule = rule;
        KR_CK(cudaSetDevice(s->device));
        krb::jit_prepare(s);
    });
}

int64_t kr_jit_step_source(const kr_treeplex* t, int rule, char* buf, int64_t cap) {
    if (!t) return -1;
    const char* ge = std::getenv("KR_JIT_SOURCE_GROUPS");   // inspect the warp-group form
    const std::string src = krb::jit_step_source(*t, rule, 0, ge ? std::atoi(ge) : 1);
    if (src.empty()) return -1;
    if (buf && cap > 0) {
        const size_t n = std::min(src.size(), size_t(cap - 1));
        std::memcpy(buf, src.data(), n);
        buf[n] = 0;
    }
    return int64_t(src.size());
}

int kr_solver_step_kind(const kr_solver* s, int player, const char** why) {
    if (!s || player < 0 || player > 1) return -1;
    if (why) *why = s->jitWhy[player].c_str();
    if (s->jit[player].kern && s->jitRule[player] == s->rule) return 2;
    return s->levelled[player] ? 1 : 0;
}

int kr_solver_begin(kr_solver* s, double alpha, double beta, double gamma) {
    return guarded([&] {
        if (!s) throw Fail{KR_INVALID_INPUT, "null solver"};
        KR_CK(cudaSetDevice(s->device));
        cudaStream_t st = s->eng->stream;
        for (int p = 0; p < 2; ++p) {
            const int64_t len = s->H[p] * s->n[p];
            KR_CK(cudaMemsetAsync(s->regret[p], 0, 8 * size_t(len), st));
            KR_CK(cudaMemsetAsync(s->avg[p], 0, 8 * size_t(len), st));
        }
        // x1, x2 = sequenceForm of zero regrets (solver.hpp:363-364)
        krb::launch_step(s, 0, 0, nullptr, 0, 0, 0, 0, st);
        krb::launch_step(s, 1, 0, nullptr, 0, 0, 0, 0, st);
        s->k7seq = false;
        if (krb::k7seq_ok(s)) krb::enter_seq(s, st);
        s->alpha = alpha;
        s->beta = beta;
        s->gamma = gamma;
        s->t = 0;
        s->weightSum = 0;
        s->begun = true;
    });
}

int kr_solver_iterate(kr_solver* s, int n) {
    return guarded([&] {
        if (!s || !s->begun) throw Fail{KR_INVALID_INPUT, "kr_solver_begin must precede kr_solver_iterate"};
        if (n < 0) throw Fail{KR_INVALID_INPUT, "negative iteration count"};
        KR_CK(cudaSetDevice(s->device));
        kr_engine* e = s->eng;
        cudaStream_t st = e->stream;
        if (s->k7seq && !krb::k7seq_ok(s)) krb::leave_seq(s, st);
        if (n >= 2 && graphs_ok(s)) {  // one captured iteration, replayed n times
            iterate_graph(s, n, st);
            return;
        }
        for (int q = 0; q < n; ++q) {
            const int t = ++s->t;  // solver.hpp:365-388
            const double pos = krb::discount_factor(t, s->alpha), neg = krb::discount_factor(t, s->beta);
            const double shrink = std::pow(double(t) / (t + 1), s->gamma);
            krb::iteration_body(s, st, pos, neg, shrink, false);
            s->weightSum += 1;
            s->weightSum *= shrink;
        }
    });
}

int kr_solver_checkpoint(kr_solver* s, double* board_br1, double* board_br2) {
    return guarded([&] {
        if (!s || !s->begun || s->t < 1) throw Fail{KR_INVALID_INPUT, "no iterations to checkpoint"};
        if (!board_br1 || !board_br2) throw Fail{KR_INVALID_INPUT, "null output arrays"};
        KR_CK(cudaSetDevice(s->device));
        cudaStream_t st = s->eng->stream;
        normalise_averages(s, st);                            // solver.hpp:390-391
        const size_t nb = size_t(s->totalBoards());
        // br1 vs avg2, br2 vs avg1 (solver.hpp:327-328), side by side
        krb::checkpoint_values(s, s->boardval, st);
        std::vector<double> b(2 * nb);
        KR_CK(cudaMemcpyAsync(b.data(), s->boardval, 8 * b.size(), cudaMemcpyDeviceToHost, st));
        KR_CK(cudaStreamSynchronize(st));
        std::memcpy(board_br1, b.data(), 8 * nb);
        std::memcpy(board_br2, b.data() + nb, 8 * nb);
    });
}

int kr_solver_averages(kr_solver* s, double* avg1, double* avg2) {
    return guarded([&] {
        if (!s || !s->begun || s->t < 1) throw Fail{KR_INVALID_INPUT, "no iterations to average"};
        KR_CK(cudaSetDevice(s->device));
        cudaStream_t st = s->eng->stream;
        normalise_averages(s, st);                            // solver.hpp:400-401
        for (int p = 0; p < 2; ++p) {
            double* dst = p == 0 ? avg1 : avg2;
            const int64_t len = s->H[p] * s->n[p];
            if (dst && len) KR_CK(cudaMemcpyAsync(dst, s->a[p], 8 * size_t(len), cudaMemcpyDeviceToHost, st));
        }
        KR_CK(cudaStreamSynchronize(st));
    });
}

int kr_solver_iteration(const kr_solver* s) { return s ? s->t : -1; }

int kr_solver_run(kr_solver* s, const kr_dcfr_params* prm, kr_dcfr_result* r) {
    return guarded([&] {
        if (!s || !prm || !r) throw Fail{KR_INVALID_INPUT, "null argument to kr_solver_run"};
        if (prm->max_iters < 1) throw Fail{KR_INVALID_INPUT, "iteration budget must be positive"};
        if (prm->checkpoint_every < 1) throw Fail{KR_INVALID_INPUT, "checkpoint period must be positive"};
        kr_engine* e = s->eng;
        KR_CK(cudaSetDevice(s->device));
        cudaStream_t st = e->stream;
        cudaEvent_t ev0, ev1;
        KR_CK(cudaEventCreate(&ev0));
        KR_CK(cudaEventCreate(&ev1));
        KR_CK(cudaEventRecord(ev0, st));
        const int64_t flops0 = e->flops_total;
        auto ck = [](int rc) {
            if (rc != KR_OK) {
                int code = 0;
                throw Fail{rc, kr_last_error(&code)};
            }
        };
        ck(kr_solver_set_rule(s, prm->rule));
        ck(kr_solver_begin(s, prm->alpha, prm->beta, prm->gamma));
        r->trace_len = 0;
        const int nb = s->totalBoards();
        std::vector<double> b1(static_cast<size_t>(nb)), b2(static_cast<size_t>(nb));
        // Record one checkpoint's per-board values (solver.hpp:389-392; the
        // board-order sums are the chance-root average of SURVEY.md 8(d)).
        auto record = [&](const double* v1, const double* v2) {
            double br1 = 0, br2 = 0, expl;
            for (int b = 0; b < nb; ++b) {
                br1 += v1[b];
                br2 += v2[b];
            }
            if (nb == 1) {
                expl = (v1[0] + v2[0]) / 2 / s->pot;  // solver.hpp:329-330
            } else {
                expl = 0;
                for (int b = 0; b < nb; ++b) expl += (v1[b] + v2[b]) / 2 / s->pot;
                expl /= nb;
            }
            const int i = r->trace_len;
            if (i < r->trace_cap) {
                if (r->trace_iter) r->trace_iter[i] = s->t;
                if (r->trace_expl) r->trace_expl[i] = expl;
                if (r->trace_br1) r->trace_br1[i] = br1;
                if (r->trace_br2) r->trace_br2[i] = br2;
                for (int b = 0; b < nb; ++b) {
                    if (r->trace_board_br1) r->trace_board_br1[size_t(i) * nb + b] = v1[b];
                    if (r->trace_board_br2) r->trace_board_br2[size_t(i) * nb + b] = v2[b];
                }
            }
            r->trace_len = i + 1;
            r->iterations = s->t;
            r->exploitability = expl;
            return expl;
        };
        if (prm->target_exploitability > 0) {
            // early stop: every checkpoint's value is needed on the host at once
            while (s->t < prm->max_iters) {
                // run to the next checkpoint (t % every == 0 or t == maxIters)
                const int next =
                    std::min(prm->max_iters, (s->t / prm->checkpoint_every + 1) * prm->checkpoint_every);
                ck(kr_solver_iterate(s, next - s->t));
                ck(kr_solver_checkpoint(s, b1.data(), b2.data()));
                if (record(b1.data(), b2.data()) <= prm->target_exploitability) break;
            }
        } else {
            // no early stop: checkpoints write to a device buffer, read back once
            const int nck = (prm->max_iters + prm->checkpoint_every - 1) / prm->checkpoint_every + 1;
            double* dck = krb::dev_alloc<double>(int64_t(nck) * 2 * nb);
            std::vector<int> at;
            try {
                if (graphs_ok(s)) {
                    run_graphs(s, prm->max_iters, prm->checkpoint_every, dck, at, st);
                } else {
                    while (s->t < prm->max_iters) {
                        const int next =
                            std::min(prm->max_iters, (s->t / prm->checkpoint_every + 1) * prm->checkpoint_every);
                        ck(kr_solver_iterate(s, next - s->t));
                        double* slot = dck + size_t(at.size()) * 2 * nb;
                        normalise_averages(s, st);                             // solver.hpp:390-391
                        krb::checkpoint_values(s, slot, st);           // br1 vs avg2, br2 vs avg1
                        at.push_back(s->t);
                    }
                }
                std::vector<double> host(at.size() * 2 * size_t(nb));
                KR_CK(cudaMemcpyAsync(host.data(), dck, 8 * host.size(), cudaMemcpyDeviceToHost, st));
                KR_CK(cudaStreamSynchronize(st));
                const int tEnd = s->t;
                for (size_t c = 0; c < at.size(); ++c) {
                    s->t = at[c];  // record() stamps the checkpoint's iteration
                    record(host.data() + c * 2 * nb, host.data() + c * 2 * nb + nb);
                }
                s->t = tEnd;
            } catch (...) {
                krb::dev_free(dck);
                throw;
            }
            krb::dev_free(dck);
        }
        KR_CK(cudaEventRecord(ev1, st));
        KR_CK(cudaEventSynchronize(ev1));
        float ms = 0;
        KR_CK(cudaEventElapsedTime(&ms, ev0, ev1));
        r->seconds = ms / 1e3;
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        if (r->avg1 || r->avg2) ck(kr_solver_averages(s, r->avg1, r->avg2));
        r->gradient_flops = e->flops_total - flops0;
        krb::engine_selfcheck_raise(e);
    });
}

int kr_solver_best_response(kr_solver* s, int player, const double* opp, int64_t n, double* value,
                            double* board_values) {
    return guarded([&] {
        if (!s || !opp || !value) throw Fail{KR_INVALID_INPUT, "null argument"};
        if (player != 0 && player != 1) throw Fail{KR_INVALID_INPUT, "player must be 0 or 1"};
        const int opp_p = 1 - player;
        const int64_t len = s->H[opp_p] * s->n[opp_p];
        if (n != len)
            throw Fail{KR_INVALID_INPUT,
                       "strategy vector has size " + std::to_string(n) + ", expected " + std::to_string(len)};
        KR_CK(cudaSetDevice(s->device));
        cudaStream_t st = s->eng->stream;
        KR_CK(cudaMemcpyAsync(s->a[opp_p], opp, 8 * size_t(len), cudaMemcpyHostToDevice, st));
        KR_CK(cudaMemsetAsync(s->d_flag, 0, 4, st));
        if (s->H[opp_p]) {
            krb::launch(krb::k_validate, unsigned((s->H[opp_p] + 127) / 128), 128, 0, st, s->d_tree[opp_p], s->nnodes[opp_p], s->n[opp_p], s->H[opp_p], s->a[opp_p], 1e-9, s->d_flag);
            KR_CK_LAUNCH();
            s->launches++;
        }
        int flag = 0;
        KR_CK(cudaMemcpyAsync(&flag, s->d_flag, 4, cudaMemcpyDeviceToHost, st));
        KR_CK(cudaStreamSynchronize(st));
        if (flag & 1) throw Fail{KR_INVALID_INPUT, "strategy vector has negative entries"};
        if (flag & 2) throw Fail{KR_INVALID_INPUT, "strategy violates flow conservation at a node"};
        std::vector<double> b;
        krb::best_response_dev(s, player, s->a[opp_p], b, st);
        double total = 0;
        for (int i = 0; i < s->nboards; ++i) {
            total += b[size_t(i)];
            if (board_values) board_values[i] = b[size_t(i)];
        }
        *value = total;
    });
}

}  // extern "C"

// ===================================================================== turn
// Turn endgames (beyond the reference): a
// turn betting tree whose continuations t lead into river subgames, one per
// river card b.  The payoff is block diagonal (the turn fold block and, per
// continuation, the river boards), so the gradient is one engine product per
// block; turn and river couple only through the treeplex: river roots hang
// under sigma_p(t).  One player's half-iteration (the CPU restatement is
// oracle/turn_oracle.py):
//   1. river team steps per continuation (regrets, mass-1 strategies, each
//      river hand's root value; no averaging yet);
//   2. root values summed over the boards in ascending order per turn hand,
//      added to the turn sequence sigma_p(t) (k_turn_contrib, k_turn_fold);
//   3. the turn team step, whose sweep adds those sums after the children;
//   4. river strategies scaled by the turn reach of sigma_p(t), then
//      averaged (k_river_scale).
// With the boards sharded over GPUs, step 2's per-turn-hand sums are the
// place of the per-iteration allreduce of the north star.
struct kr_turn_solver {
    int device = 0;
    kr_engine* turnEng = nullptr;
    std::vector<kr_engine*> riverEng;
    int T = 0, m = 0, nb = 0;
    int64_t Hr = 0;                                // river hands over all boards
    struct TreeDev {
        int32_t* d = nullptr;
        int len = 0, na = 0, nn = 0, n = 0;
        // the step compiled for this tree (kr_jit.cu) and its host copy
        krb::JitStep jit;
        int jitRule = -1;
        std::vector<int32_t> par, ptr, seq;
    };
    TreeDev turnTree[2];
    std::vector<TreeDev> riverTree[2];             // [p][t]
    std::vector<int> sigma[2];                     // [p][t]
    int64_t* d_boff = nullptr;                     // [nb+1] river-hand offsets per board
    int32_t* d_r2t = nullptr;                      // [Hr] turn hand of each river hand
    int32_t* d_t2r = nullptr;                      // [nb*m] river index of a turn hand, -1 = holds b
    std::vector<int64_t> off[2];                   // vector offsets: [turn | t0 | t1 | ...]
    double *regret[2] = {nullptr, nullptr}, *avg[2] = {nullptr, nullptr}, *x[2] = {nullptr, nullptr};
    double *a[2] = {nullptr, nullptr};
    double *g = nullptr, *root = nullptr, *extra = nullptr, *handval = nullptr, *bval = nullptr;
    int64_t* d_one = nullptr;                      // {0, m}: one "board" of turn hands for k_board_sums
    double pot = 0;
    int64_t launches = 0;
    int rule = 0;  // KR_RULE_*
    // The river values reach the turn hands board by board: contrib holds
    // this rank's [T][m][nbMax] values (a marker where a board holds the
    // hand), gathered every rank's (world x that, rank-major = global board
    // order), and k_turn_fold adds them per turn hand in board order: the
    // same fold on one GPU and on any number of ranks.  Transport: comm (NCCL,
    // in-stream) or xfn (host callback, stream synchronised), else none.
    kr_comm* comm = nullptr;
    void (*xfn)(void*) = nullptr;
    void* xuser = nullptr;
    int world = 1, rank = 0, nbMax = 0;
    int32_t* d_bpre = nullptr;                     // [world + 1] board prefix over the ranks
    double* contrib = nullptr;
    double* gathered = nullptr;                    // == contrib with one rank
    bool ownBufs = true;                           // false: the caller's (set_exchange)
    // graph replay (one GPU, no exchange): per-iteration pos/neg/shrink from
    // a device table indexed by the device iteration counter
    double* d_fac = nullptr;
    int* d_cnt = nullptr;
    int32_t* d_sigma = nullptr;                    // [2][T] sigma_p(t), for k_turn_fold
    int64_t* d_roff = nullptr;                     // [2][T+1] river block offsets (from off[p][1])
    int32_t* d_nr = nullptr;                       // [2][T] river sequences per continuation
    // the continuations' independent river products and player steps run
    // side by side: continuation t on side[t], forked from / joined into the
    // solver stream (KR_TURN_SERIAL=1: all on the solver stream)
    std::vector<cudaStream_t> side;
    cudaEvent_t evFork = nullptr;
    std::vector<cudaEvent_t> evJoin;
};

namespace krb {
namespace {

constexpr uint64_t kSkipBits = 0x7ff8000000000001ULL;  // NaN marker: the board holds the hand

// This rank's river root values per (continuation t, turn hand h, local
// board b): contrib[(t m + h) nbMax + b], the marker where board b holds h
// (or past this rank's boards).
__global__ void k_turn_contrib(const double* __restrict__ root, int64_t Hr, const int32_t* __restrict__ t2r,
                               const int64_t* __restrict__ boff, int nb, int m, int T, int nbMax,
                               double* __restrict__ contrib) {
    krb::pdl_entry();
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= int64_t(T) * m * nbMax) return;
    const int b = int(q % nbMax);
    const int64_t th = q / nbMax;
    const int h = int(th % m), t = int(th / m);
    double v = __longlong_as_double((long long)kSkipBits);
    if (b < nb) {
        const int r = t2r[int64_t(b) * m + h];
        if (r >= 0) v = root[int64_t(t) * Hr + boff[b] + r];
    }
    contrib[q] = v;
}

// Per turn hand h and continuation t in order: extra[h, sigma(t)] += the sum
// over all boards in global order (rank-major, each rank's boards ascending;
// boards holding h skipped) -- one left fold, the same on one GPU and on any
// number of ranks.  One warp per turn hand: the lanes stage a continuation's
// per-board values in shared memory (coalesced), lane 0 folds them in board
// order (one thread per hand, 9 CTAs, took ~20 us per half-iteration).
constexpr int kFoldWarps = 4;
__global__ void __launch_bounds__(32 * kFoldWarps) k_turn_fold(const double* __restrict__ gathered, int world,
                                                               int nbMax, const int32_t* __restrict__ bpre, int T,
                                                               int m, int nt, const int32_t* __restrict__ sigma,
                                                               double* __restrict__ extra) {
    krb::pdl_entry();
    extern __shared__ double fs[];   // [kFoldWarps][world * nbMax]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int h = blockIdx.x * kFoldWarps + w;
    if (h >= m) return;
    const int64_t per = int64_t(T) * m * nbMax;
    double* v = fs + size_t(w) * size_t(world) * nbMax;
    for (int t = 0; t < T; ++t) {
        int n = 0;
        for (int r = 0; r < world; ++r) {
            const double* g = gathered + r * per + (int64_t(t) * m + h) * nbMax;
            const int nbr = bpre[r + 1] - bpre[r];
            for (int b = lane; b < nbr; b += 32) v[n + b] = g[b];
            n += nbr;
        }
        __syncwarp();
        if (lane == 0) {
            double acc = 0.0;
            for (int q = 0; q < n; ++q) {
                const double x = v[q];
                if (uint64_t(__double_as_longlong(x)) != kSkipBits) acc += x;
            }
            extra[int64_t(h) * nt + sigma[t] - 1] += acc;
        }
        __syncwarp();
    }
}

// One rank, no exchange: the same fold straight from the river root values
// (k_turn_contrib + k_turn_fold without the staging array): board b's value
// for turn hand h is root[t Hr + boff[b] + t2r[b m + h]], boards holding h
// skipped, added in board order.
__global__ void __launch_bounds__(32 * kFoldWarps) k_turn_fold_direct(const double* __restrict__ root, int64_t Hr,
                                                                      const int32_t* __restrict__ t2r,
                                                                      const int64_t* __restrict__ boff, int nb, int T,
                                                                      int m, int nt, const int32_t* __restrict__ sigma,
                                                                      double* __restrict__ extra) {
    krb::pdl_entry();
    extern __shared__ double fs[];   // [kFoldWarps][T][nb]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int h = blockIdx.x * kFoldWarps + w;
    if (h >= m) return;
    double* v = fs + size_t(w) * size_t(T) * nb;
    // every continuation's values staged at once (one load latency), then
    // folded continuation by continuation in order
    for (int b = lane; b < nb; b += 32) {
        const int r = t2r[int64_t(b) * m + h];
        for (int t = 0; t < T; ++t)
            v[t * nb + b] = r >= 0 ? root[int64_t(t) * Hr + boff[b] + r] : __longlong_as_double((long long)kSkipBits);
    }
    __syncwarp();
    if (lane == 0)
        for (int t = 0; t < T; ++t) {
            double acc = 0.0;
            for (int b = 0; b < nb; ++b) {
                const double x = v[t * nb + b];
                if (uint64_t(__double_as_longlong(x)) != kSkipBits) acc += x;
            }
            extra[int64_t(h) * nt + sigma[t] - 1] += acc;
        }
}

__global__ void k_river_scale(double* __restrict__ x, double* __restrict__ avg, const double* __restrict__ xturn,
                              const int32_t* __restrict__ r2t, int64_t Hr, int nr, int nt, int sigma,
                              double shrink, int doAvg, const double* __restrict__ fac = nullptr,
                              const int* __restrict__ dt = nullptr) {
    krb::pdl_entry();
    if (fac) shrink = fac[3 * *dt + 2];  // graph replay
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= Hr * nr) return;
    const int64_t r = q < (int64_t(1) << 32) ? int64_t(uint32_t(q) / uint32_t(nr)) : q / nr;
    const double xv = xturn[int64_t(r2t[r]) * nt + sigma - 1] * x[q];
    x[q] = xv;
    if (doAvg) avg[q] = (avg[q] + xv) * shrink;  // solver.hpp:382-386
}

// Every continuation's river blocks of player p in one launch (the bits of T
// k_river_scale launches): block t holds Hr x nr[t] entries at roff[t].
__global__ void k_river_scale_all(double* __restrict__ x, double* __restrict__ avg,
                                  const double* __restrict__ xturn, const int32_t* __restrict__ r2t, int64_t Hr,
                                  int nt, int T, const int64_t* __restrict__ roff, const int32_t* __restrict__ nrs,
                                  const int32_t* __restrict__ sigma, double shrink, int doAvg,
                                  const double* __restrict__ fac, const int* __restrict__ dt) {
    krb::pdl_entry();
    if (fac) shrink = fac[3 * *dt + 2];  // graph replay
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= roff[T]) return;
    int t = 0;
    while (q >= roff[t + 1]) ++t;
    const int nr = nrs[t];
    const int64_t off = q - roff[t];
    // a continuation block holds Hr x nr < 2^32 values: 32-bit division (the
    // 64-bit one is a long software sequence per element)
    const int64_t r = off < (int64_t(1) << 32) ? int64_t(uint32_t(off) / uint32_t(nr)) : off / nr;
    const double xv = xturn[int64_t(r2t[r]) * nt + sigma[t] - 1] * x[q];
    x[q] = xv;
    if (doAvg) avg[q] = (avg[q] + xv) * shrink;  // solver.hpp:382-386
}

kr_turn_solver::TreeDev make_tree(const kr_treeplex& t) {
    if (t.n_seq < 1 || t.n_nodes < 1 || !t.node_parent_seq || !t.node_action_ptr || !t.action_seq)
        throw Fail{KR_INVALID_INPUT, "empty treeplex"};
    const int na = t.node_action_ptr[t.n_nodes];
    std::vector<int32_t> buf;
    buf.insert(buf.end(), t.node_parent_seq, t.node_parent_seq + t.n_nodes);
    buf.insert(buf.end(), t.node_action_ptr, t.node_action_ptr + t.n_nodes + 1);
    buf.insert(buf.end(), t.action_seq, t.action_seq + na);
    bool ok = false;
    int nlev = 0;
    append_levels(t, buf, ok, nlev);
    if (!ok) throw Fail{KR_INVALID_INPUT, "turn solver needs reference-ordered treeplexes"};
    kr_turn_solver::TreeDev d;
    d.par.assign(t.node_parent_seq, t.node_parent_seq + t.n_nodes);
    d.ptr.assign(t.node_action_ptr, t.node_action_ptr + t.n_nodes + 1);
    d.seq.assign(t.action_seq, t.action_seq + na);
    d.len = int(buf.size());
    d.na = na;
    d.nn = t.n_nodes;
    d.n = t.n_seq;
    d.d = dev_alloc<int32_t>(d.len);
    KR_CK(cudaMemcpy(d.d, buf.data(), 4 * buf.size(), cudaMemcpyHostToDevice));
    return d;
}

constexpr int kTurnTeam = 4;

// Compile the river trees' steps (and the turn tree's when its hands fill
// the GPU) for the current rule, as jit_prepare does for kr_solver.
void turn_jit_prepare(kr_turn_solver* s) {
    const char* env = std::getenv("KR_STEP");
    const bool force = env && std::string(env) == "jit";
    auto prep = [&](kr_turn_solver::TreeDev& T, int64_t H) {
        if (T.jitRule == s->rule) return;
        T.jit = JitStep{};
        T.jitRule = -1;
        if (!force && H < int64_t(2) * 148 * kJitHands) return;   // (the 1,128-hand turn tree: no gain compiled)
        kr_treeplex t{};
        t.n_nodes = T.nn;
        t.n_seq = T.n;
        t.node_parent_seq = T.par.data();
        t.node_action_ptr = T.ptr.data();
        t.action_seq = T.seq.data();
        std::string why;
        if (jit_step_compile(t, s->rule, T.jit, why)) T.jitRule = s->rule;
    };
    for (int p = 0; p < 2; ++p) {
        prep(s->turnTree[p], s->m);
        for (auto& T : s->riverTree[p]) prep(T, s->Hr);
    }
}

void team_step(kr_turn_solver* s, const kr_turn_solver::TreeDev& T, int64_t H, int mode, const double* g, int negate,
               double* regret, double* x, double* avg, double pos, double neg, double shrink, int noAvg,
               double* rootOut, const double* extra, cudaStream_t st, const double* fac, const int* dt) {
    if (mode == 1 && T.jit.kern && T.jitRule == s->rule) {
        jit_step_launch(T.jit, s->device, H, g, negate, regret, x, avg, pos, neg, shrink, fac, dt, noAvg, rootOut,
                        extra, st);
        s->launches++;
        return;
    }
    const int hpb = 256 / kTurnTeam;
    const unsigned grid = unsigned((H + hpb - 1) / hpb);
    if (!grid) return;
    const size_t smem = team_smem(T.n, T.nn, hpb, T.len);
    krb::launch(k_player_team<kTurnTeam>, grid, 256, smem, st, mode, T.d, T.nn, T.n, T.na, T.len, H, hpb, g, negate, regret, x,
                                                      avg, pos, neg, shrink, s->rule, fac, dt, noAvg, rootOut,
                                                      extra);
    KR_CK_LAUNCH();
    s->launches++;
}

// Continuation t's stream: side[t] between fork() and join(), else st.
cudaStream_t cont_stream(kr_turn_solver* s, int t, cudaStream_t st) {
    return s->side.empty() ? st : s->side[size_t(t)];
}
void fork(kr_turn_solver* s, cudaStream_t st) {
    if (s->side.empty()) return;
    KR_CK(cudaEventRecord(s->evFork, st));
    for (cudaStream_t q : s->side) KR_CK(cudaStreamWaitEvent(q, s->evFork, 0));
}
void join(kr_turn_solver* s, cudaStream_t st) {
    for (size_t t = 0; t < s->side.size(); ++t) {
        KR_CK(cudaEventRecord(s->evJoin[t], s->side[t]));
        KR_CK(cudaStreamWaitEvent(st, s->evJoin[t], 0));
    }
}

// KR_TURN_FUSE=0: one river-scale launch per continuation instead of one for
// all of them (the same bits).
bool turn_fuse() {
    const char* env = std::getenv("KR_TURN_FUSE");
    return !(env && std::atoi(env) == 0);
}

// The river root values of every continuation into `extra`: this rank's
// per-board values, exchanged over the ranks (all-gather), folded in global
// board order.
void gather_all(kr_turn_solver* s, int p, int nt, cudaStream_t st) {
    if (!s->comm && !s->xfn) {   // one rank: fold straight from the root values
        krb::launch(k_turn_fold_direct, unsigned((s->m + kFoldWarps - 1) / kFoldWarps), 32 * kFoldWarps,
                    size_t(kFoldWarps) * size_t(s->T) * size_t(s->nb) * sizeof(double), st, s->root, s->Hr, s->d_t2r,
                    s->d_boff,
                    s->nb, s->T, s->m, nt, s->d_sigma + p * s->T, s->extra);
        KR_CK_LAUNCH();
        s->launches++;
        return;
    }
    const int64_t count = int64_t(s->T) * s->m * s->nbMax;
    krb::launch(k_turn_contrib, unsigned((count + 255) / 256), 256, 0, st, s->root, s->Hr, s->d_t2r, s->d_boff, s->nb,
                s->m, s->T, s->nbMax, s->contrib);
    KR_CK_LAUNCH();
    s->launches++;
    if (s->comm) {
        comm_allgather(s->comm, s->contrib, s->gathered, size_t(count), st);
    } else if (s->xfn) {
        KR_CK(cudaStreamSynchronize(st));
        s->xfn(s->xuser);  // all-gathers contrib into gathered (the caller's buffers)
    }
    krb::launch(k_turn_fold, unsigned((s->m + kFoldWarps - 1) / kFoldWarps), 32 * kFoldWarps,
                size_t(kFoldWarps) * size_t(s->world) * size_t(s->nbMax) * sizeof(double), st, s->gathered, s->world,
                s->nbMax, s->d_bpre,
                s->T, s->m, nt, s->d_sigma + p * s->T, s->extra);
    KR_CK_LAUNCH();
    s->launches++;
}

// Player p's half-iteration (mode 1) or initial strategy (mode 0).
// fac / dt: graph replay (the factors from the device table, else the scalars).
void turn_player(kr_turn_solver* s, int p, int mode, double pos, double neg, double shrink, cudaStream_t st,
                 const double* fac = nullptr, const int* dt = nullptr) {
    const int nt = s->turnTree[p].n;
    KR_CK(cudaMemsetAsync(s->extra, 0, 8 * size_t(s->m) * nt, st));
    fork(s, st);
    for (int t = 0; t < s->T; ++t) {
        const int64_t o = s->off[p][size_t(t) + 1];
        team_step(s, s->riverTree[p][size_t(t)], s->Hr, mode, s->g + o, p == 1, s->regret[p] + o, s->x[p] + o,
                  s->avg[p] + o, pos, neg, shrink, 1, mode == 1 ? s->root + int64_t(t) * s->Hr : nullptr, nullptr,
                  cont_stream(s, t, st), fac, dt);
    }
    join(s, st);
    if (mode == 1) gather_all(s, p, nt, st);
    team_step(s, s->turnTree[p], s->m, mode, s->g, p == 1, s->regret[p], s->x[p], s->avg[p], pos, neg, shrink, 0,
              nullptr, mode == 1 ? s->extra : nullptr, st, fac, dt);
    if (turn_fuse()) {
        const int64_t o = s->off[p][1], n = s->off[p].back() - o;
        krb::launch(k_river_scale_all, unsigned((n + 255) / 256), 256, 0, st, s->x[p] + o, s->avg[p] + o, s->x[p], s->d_r2t, s->Hr, nt, s->T, s->d_roff + p * (s->T + 1),
            s->d_nr + p * s->T, s->d_sigma + p * s->T, shrink, mode == 1, fac, dt);
        KR_CK_LAUNCH();
        s->launches++;
        return;
    }
    for (int t = 0; t < s->T; ++t) {
        const int64_t o = s->off[p][size_t(t) + 1];
        const int nr = s->riverTree[p][size_t(t)].n;
        const int64_t n = s->Hr * nr;
        krb::launch(k_river_scale, unsigned((n + 255) / 256), 256, 0, st, s->x[p] + o, s->avg[p] + o, s->x[p], s->d_r2t, s->Hr,
                                                                  nr, nt, s->sigma[p][size_t(t)], shrink, mode == 1,
                                                                  fac, dt);
        KR_CK_LAUNCH();
        s->launches++;
    }
}

void turn_gradient(kr_turn_solver* s, int p, const double* opp, double* g, cudaStream_t st) {
    const int q = 1 - p;  // opponent's blocks are the inputs
    fork(s, st);
    if (p == 0) engine_ax(s->turnEng, opp, g, st);
    else engine_atx(s->turnEng, opp, g, st);
    for (int t = 0; t < s->T; ++t) {
        const double* in = opp + s->off[q][size_t(t) + 1];
        double* out = g + s->off[p][size_t(t) + 1];
        if (p == 0) engine_ax(s->riverEng[size_t(t)], in, out, cont_stream(s, t, st));
        else engine_atx(s->riverEng[size_t(t)], in, out, cont_stream(s, t, st));
    }
    join(s, st);
}

// bestResponseValue of player p against the device strategy opp.
double turn_br(kr_turn_solver* s, int p, const double* opp, cudaStream_t st) {
    turn_gradient(s, p, opp, s->g, st);
    const int nt = s->turnTree[p].n;
    KR_CK(cudaMemsetAsync(s->extra, 0, 8 * size_t(s->m) * nt, st));
    const int bt = 128;
    auto br = [&](const kr_turn_solver::TreeDev& T, int64_t H, const double* g, double* out, const double* extra) {
        const size_t smem = size_t((2 * T.nn + 1 + T.na + 2) * 4) + size_t(T.n + 1) * bt * 8 + 16;
        krb::launch(k_best_response, unsigned((H + bt - 1) / bt), bt, smem, st, T.d, T.nn, T.n, H, g, p == 1, out, extra);
        KR_CK_LAUNCH();
        s->launches++;
    };
    for (int t = 0; t < s->T; ++t)
        br(s->riverTree[p][size_t(t)], s->Hr, s->g + s->off[p][size_t(t) + 1], s->root + int64_t(t) * s->Hr,
           nullptr);
    gather_all(s, p, nt, st);
    br(s->turnTree[p], s->m, s->g, s->handval, s->extra);
    krb::launch(k_board_sums, 1, 256, 0, st, s->handval, s->d_one, 1, s->bval, nullptr, 0);
    KR_CK_LAUNCH();
    s->launches++;
    double v = 0;
    KR_CK(cudaMemcpyAsync(&v, s->bval, 8, cudaMemcpyDeviceToHost, st));
    KR_CK(cudaStreamSynchronize(st));
    return v;
}

void destroy_turn(kr_turn_solver* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    for (int p = 0; p < 2; ++p) {
        krb::dev_free(s->turnTree[p].d);
        for (auto& t : s->riverTree[p]) krb::dev_free(t.d);
        krb::dev_free(s->regret[p]);
        krb::dev_free(s->avg[p]);
        krb::dev_free(s->x[p]);
        krb::dev_free(s->a[p]);
    }
    if (s->ownBufs) {
        if (s->gathered != s->contrib) krb::dev_free(s->gathered);
        krb::dev_free(s->contrib);
    }
    void* ps[] = {s->d_boff, s->d_r2t, s->d_t2r, s->g,     s->root,  s->handval, s->bval,
                  s->d_one,  s->d_fac, s->d_cnt, s->d_sigma, s->d_roff, s->d_nr, s->d_bpre, s->extra};
    for (void* q : ps) krb::dev_free(q);
    for (cudaStream_t q : s->side) cudaStreamDestroy(q);
    for (cudaEvent_t ev : s->evJoin) cudaEventDestroy(ev);
    if (s->evFork) cudaEventDestroy(s->evFork);
    delete s;
}

}  // namespace
}  // namespace krb

extern "C" {

int kr_turn_solver_create(kr_engine* turnEng, int T, kr_engine* const* riverEngs, const kr_treeplex* turnTrees,
                          const kr_treeplex* riverTrees, int m, int nb, const int32_t* mb, const int32_t* riverToTurn,
                          const int32_t* sigma, double pot, kr_turn_solver** out) {
    return guarded([&] {
        if (!turnEng || T < 1 || !riverEngs || !turnTrees || !riverTrees || m < 1 || nb < 1 || !mb || !riverToTurn ||
            !sigma || !out)
            throw Fail{KR_INVALID_INPUT, "bad arguments to kr_turn_solver_create"};
        if (!(pot > 0)) throw Fail{KR_INVALID_INPUT, "pot must be positive"};
        KR_CK(cudaSetDevice(turnEng->device));
        auto* s = new kr_turn_solver();
        try {
            s->device = turnEng->device;
            s->turnEng = turnEng;
            s->T = T;
            s->m = m;
            s->nb = nb;
            s->pot = pot;
            std::vector<int64_t> boff{0};
            for (int b = 0; b < nb; ++b) boff.push_back(boff.back() + mb[b]);
            s->Hr = boff.back();
            std::vector<int32_t> t2r(size_t(nb) * m, -1);
            for (int b = 0; b < nb; ++b)
                for (int64_t r = boff[size_t(b)]; r < boff[size_t(b) + 1]; ++r) {
                    const int h = riverToTurn[r];
                    if (h < 0 || h >= m) throw Fail{KR_INVALID_INPUT, "river hand maps outside the turn hands"};
                    t2r[size_t(b) * m + size_t(h)] = int32_t(r - boff[size_t(b)]);
                }
            for (int p = 0; p < 2; ++p) {
                s->turnTree[p] = krb::make_tree(turnTrees[p]);
                s->off[p].assign(1, 0);
                s->off[p].push_back(int64_t(m) * turnTrees[p].n_seq);
                for (int t = 0; t < T; ++t) {
                    const kr_treeplex& rt = riverTrees[2 * t + p];
                    s->riverTree[p].push_back(krb::make_tree(rt));
                    s->sigma[p].push_back(sigma[2 * t + p]);
                    if (sigma[2 * t + p] < 1 || sigma[2 * t + p] > turnTrees[p].n_seq)
                        throw Fail{KR_INVALID_INPUT, "continuation sequence out of range"};
                    s->off[p].push_back(s->off[p].back() + s->Hr * rt.n_seq);
                }
            }
            // the engines must cover exactly these blocks
            if (turnEng->rows != s->off[0][1] || turnEng->cols != s->off[1][1])
                throw Fail{KR_INVALID_INPUT, "turn engine does not match m x n_turn"};
            for (int t = 0; t < T; ++t) {
                kr_engine* e = riverEngs[t];
                if (!e || e->device != s->device || e->rows != s->off[0][size_t(t) + 2] - s->off[0][size_t(t) + 1] ||
                    e->cols != s->off[1][size_t(t) + 2] - s->off[1][size_t(t) + 1])
                    throw Fail{KR_INVALID_INPUT, "river engine does not match its continuation block"};
                s->riverEng.push_back(e);
            }
            // the team kernel's shared memory for the largest tree
            size_t att = 48 * 1024;
            for (int p = 0; p < 2; ++p) {
                att = std::max(att, krb::team_smem(s->turnTree[p].n, s->turnTree[p].nn, 256 / krb::kTurnTeam,
                                                   s->turnTree[p].len));
                for (auto& rt : s->riverTree[p])
                    att = std::max(att, krb::team_smem(rt.n, rt.nn, 256 / krb::kTurnTeam, rt.len));
            }
            if (att > 220 * 1024) throw Fail{KR_INVALID_INPUT, "treeplex too large for the on-chip solver step"};
            krb::raise_smem_limit(krb::k_player_team<krb::kTurnTeam>, att);
            s->d_boff = krb::dev_alloc<int64_t>(int64_t(boff.size()));
            KR_CK(cudaMemcpy(s->d_boff, boff.data(), 8 * boff.size(), cudaMemcpyHostToDevice));
            s->d_r2t = krb::dev_alloc<int32_t>(s->Hr);
            KR_CK(cudaMemcpy(s->d_r2t, riverToTurn, 4 * size_t(s->Hr), cudaMemcpyHostToDevice));
            s->d_t2r = krb::dev_alloc<int32_t>(int64_t(t2r.size()));
            KR_CK(cudaMemcpy(s->d_t2r, t2r.data(), 4 * t2r.size(), cudaMemcpyHostToDevice));
            for (int p = 0; p < 2; ++p) {
                const int64_t len = s->off[p].back();
                s->regret[p] = krb::dev_alloc<double>(len);
                s->avg[p] = krb::dev_alloc<double>(len);
                s->x[p] = krb::dev_alloc<double>(len);
                s->a[p] = krb::dev_alloc<double>(len);
            }
            s->g = krb::dev_alloc<double>(std::max(s->off[0].back(), s->off[1].back()));
            s->root = krb::dev_alloc<double>(s->Hr * T);  // one block of river hands per continuation
            {
                std::vector<int32_t> sg;
                for (int p = 0; p < 2; ++p) sg.insert(sg.end(), s->sigma[p].begin(), s->sigma[p].end());
                s->d_sigma = krb::dev_alloc<int32_t>(int64_t(sg.size()));
                KR_CK(cudaMemcpy(s->d_sigma, sg.data(), 4 * sg.size(), cudaMemcpyHostToDevice));
                std::vector<int64_t> ro;
                std::vector<int32_t> nr;
                for (int p = 0; p < 2; ++p) {
                    for (int t = 0; t <= T; ++t) ro.push_back(s->off[p][size_t(t) + 1] - s->off[p][1]);
                    for (int t = 0; t < T; ++t) nr.push_back(s->riverTree[p][size_t(t)].n);
                }
                s->d_roff = krb::dev_alloc<int64_t>(int64_t(ro.size()));
                s->d_nr = krb::dev_alloc<int32_t>(int64_t(nr.size()));
                KR_CK(cudaMemcpy(s->d_roff, ro.data(), 8 * ro.size(), cudaMemcpyHostToDevice));
                KR_CK(cudaMemcpy(s->d_nr, nr.data(), 4 * nr.size(), cudaMemcpyHostToDevice));
            }
            if (T > 1 && !std::getenv("KR_TURN_SERIAL")) {
                s->side.resize(size_t(T));
                s->evJoin.resize(size_t(T));
                for (int t = 0; t < T; ++t) {
                    KR_CK(cudaStreamCreateWithFlags(&s->side[size_t(t)], cudaStreamNonBlocking));
                    KR_CK(cudaEventCreateWithFlags(&s->evJoin[size_t(t)], cudaEventDisableTiming));
                }
                KR_CK(cudaEventCreateWithFlags(&s->evFork, cudaEventDisableTiming));
            }
            s->extra = krb::dev_alloc<double>(int64_t(m) * std::max(turnTrees[0].n_seq, turnTrees[1].n_seq));
            {   // one rank until kr_turn_solver_set_comm / _set_exchange
                s->nbMax = std::max(nb, 1);
                s->contrib = krb::dev_alloc<double>(std::max<int64_t>(int64_t(T) * m * s->nbMax, 1));
                s->gathered = s->contrib;
                const int32_t pre[2] = {0, nb};
                s->d_bpre = krb::dev_alloc<int32_t>(2);
                KR_CK(cudaMemcpy(s->d_bpre, pre, 8, cudaMemcpyHostToDevice));
            }
            s->handval = krb::dev_alloc<double>(std::max<int64_t>(m, s->Hr));
            s->bval = krb::dev_alloc<double>(1);
            const int64_t one[2] = {0, m};
            s->d_one = krb::dev_alloc<int64_t>(2);
            KR_CK(cudaMemcpy(s->d_one, one, 16, cudaMemcpyHostToDevice));
            KR_CK(cudaDeviceSynchronize());
        } catch (...) {
            krb::destroy_turn(s);
            throw;
        }
        *out = s;
    });
}

int kr_turn_solver_destroy(kr_turn_solver* s) {
    return guarded([&] { krb::destroy_turn(s); });
}

int kr_turn_solver_run(kr_turn_solver* s, const kr_dcfr_params* prm, kr_dcfr_result* r) {
    return guarded([&] {
        if (!s || !prm || !r) throw Fail{KR_INVALID_INPUT, "null argument to kr_turn_solver_run"};
        if (prm->max_iters < 1 || prm->checkpoint_every < 1)
            throw Fail{KR_INVALID_INPUT, "iteration budget and checkpoint period must be positive"};
        if (prm->rule < KR_RULE_DCFR || prm->rule > KR_RULE_PRMP) throw Fail{KR_INVALID_INPUT, "unknown update rule"};
        s->rule = prm->rule;
        KR_CK(cudaSetDevice(s->device));
        krb::turn_jit_prepare(s);
        cudaStream_t st = s->turnEng->stream;
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
        cudaGraphExec_t exec = nullptr;
        struct ExecGuard {  // the graph (and the events) go on every exit path
            cudaGraphExec_t& x;
            cudaEvent_t &a, &b;
            ~ExecGuard() {
                if (x) cudaGraphExecDestroy(x);
                if (a) cudaEventDestroy(a);
                if (b) cudaEventDestroy(b);
            }
        } guard{exec, ev0, ev1};
        KR_CK(cudaEventCreate(&ev0));
        KR_CK(cudaEventCreate(&ev1));
        KR_CK(cudaEventRecord(ev0, st));
        for (int p = 0; p < 2; ++p) {
            KR_CK(cudaMemsetAsync(s->regret[p], 0, 8 * size_t(s->off[p].back()), st));
            KR_CK(cudaMemsetAsync(s->avg[p], 0, 8 * size_t(s->off[p].back()), st));
        }
        krb::turn_player(s, 0, 0, 0, 0, 0, st);  // sequenceForm of zero regrets (solver.hpp:363-364)
        krb::turn_player(s, 1, 0, 0, 0, 0, st);
        double ws = 0;
        r->trace_len = 0;
        // Without a host exchange (one GPU, or NCCL ranks: the all-gathers are
        // captured in-stream) every iteration replays one captured graph
        // (tick, both gradients and player steps), its factors read
        // from a device table filled with the loop's own expressions, so a
        // replay is bitwise the launched iteration.  Checkpoints stay on the
        // host path (their values are read back).  KR_NO_GRAPH: launch by launch.
        int64_t launchDelta = 0;
        if (!s->xfn && !std::getenv("KR_NO_GRAPH")) {
            std::vector<double> fac(size_t(3) * (prm->max_iters + 1), 0.0);
            for (int t = 1; t <= prm->max_iters; ++t) {
                fac[3 * size_t(t)] = krb::discount_factor(t, prm->alpha);
                fac[3 * size_t(t) + 1] = krb::discount_factor(t, prm->beta);
                fac[3 * size_t(t) + 2] = std::pow(double(t) / (t + 1), prm->gamma);
            }
            krb::dev_free(s->d_fac);
            s->d_fac = nullptr;
            s->d_fac = krb::dev_alloc<double>(int64_t(fac.size()));
            if (!s->d_cnt) s->d_cnt = krb::dev_alloc<int>(2);
            KR_CK(cudaMemcpyAsync(s->d_fac, fac.data(), 8 * fac.size(), cudaMemcpyHostToDevice, st));
            KR_CK(cudaMemsetAsync(s->d_cnt, 0, 2 * sizeof(int), st));
            KR_CK(cudaStreamSynchronize(st));
            const int64_t l0 = s->launches;
            cudaGraph_t gr;
            KR_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            try {
                krb::launch(krb::k_tick, 1, 1, 0, st, s->d_cnt, 0);
                KR_CK_LAUNCH();
                s->launches++;
                krb::turn_gradient(s, 0, s->x[1], s->g, st);
                krb::turn_player(s, 0, 1, 0, 0, 0, st, s->d_fac, s->d_cnt);
                krb::turn_gradient(s, 1, s->x[0], s->g, st);
                krb::turn_player(s, 1, 1, 0, 0, 0, st, s->d_fac, s->d_cnt);
            } catch (...) {
                cudaStreamEndCapture(st, &gr);
                throw;
            }
            KR_CK(cudaStreamEndCapture(st, &gr));
            const cudaError_t ie = cudaGraphInstantiate(&exec, gr, 0);
            cudaGraphDestroy(gr);
            KR_CK(ie);
            launchDelta = s->launches - l0;
            s->launches = l0;
        }
        for (int t = 1; t <= prm->max_iters; ++t) {
            const double pos = krb::discount_factor(t, prm->alpha), neg = krb::discount_factor(t, prm->beta);
            const double shrink = std::pow(double(t) / (t + 1), prm->gamma);
            if (exec) {
                KR_CK(cudaGraphLaunch(exec, st));
                s->launches += launchDelta;
            } else {
                krb::turn_gradient(s, 0, s->x[1], s->g, st);    // g1 = A x2
                krb::turn_player(s, 0, 1, pos, neg, shrink, st);
                krb::turn_gradient(s, 1, s->x[0], s->g, st);    // A^T x1 (negated in the steps)
                krb::turn_player(s, 1, 1, pos, neg, shrink, st);
            }
            ws += 1;
            ws *= shrink;
            if (t % prm->checkpoint_every == 0 || t == prm->max_iters) {
                for (int p = 0; p < 2; ++p) {
                    const int64_t len = s->off[p].back();
                    krb::launch(krb::k_normalise, unsigned((len + 255) / 256), 256, 0, st, s->avg[p], len, ws, s->a[p],
                                                                                  nullptr, nullptr);
                    KR_CK_LAUNCH();
                }
                const double br1 = krb::turn_br(s, 0, s->a[1], st), br2 = krb::turn_br(s, 1, s->a[0], st);
                const double expl = (br1 + br2) / 2 / s->pot;
                const int i = r->trace_len;
                if (i < r->trace_cap) {
                    if (r->trace_iter) r->trace_iter[i] = t;
                    if (r->trace_expl) r->trace_expl[i] = expl;
                    if (r->trace_br1) r->trace_br1[i] = br1;
                    if (r->trace_br2) r->trace_br2[i] = br2;
                }
                r->trace_len = i + 1;
                r->iterations = t;
                r->exploitability = expl;
                if (prm->target_exploitability > 0 && expl <= prm->target_exploitability) break;
            }
        }
        KR_CK(cudaEventRecord(ev1, st));
        KR_CK(cudaEventSynchronize(ev1));
        float ms = 0;
        KR_CK(cudaEventElapsedTime(&ms, ev0, ev1));
        r->seconds = ms / 1e3;
        for (int p = 0; p < 2; ++p) {
            double* dst = p == 0 ? r->avg1 : r->avg2;
            if (dst) KR_CK(cudaMemcpy(dst, s->a[p], 8 * size_t(s->off[p].back()), cudaMemcpyDeviceToHost));
        }
        r->gradient_flops = 0;
    });
}

int64_t kr_turn_solver_launches(const kr_turn_solver* s) { return s ? s->launches : 0; }

namespace {
// Shard layout of a turn solver: world ranks, boards_per_rank, the
// contribution / gathered buffers sized for the largest shard.
void turn_shards(kr_turn_solver* s, int world, int rank, const int32_t* bpr, double* send = nullptr,
                 double* recv = nullptr) {
    if (world < 1 || rank < 0 || rank >= world) throw Fail{KR_INVALID_INPUT, "bad rank / size"};
    std::vector<int32_t> pre(size_t(world) + 1, 0);
    int nbMax = 0;
    for (int r = 0; r < world; ++r) {
        const int n = bpr ? bpr[r] : s->nb;
        if (n < 0) throw Fail{KR_INVALID_INPUT, "negative board count"};
        pre[size_t(r) + 1] = pre[size_t(r)] + n;
        nbMax = std::max(nbMax, n);
    }
    if ((bpr ? bpr[rank] : s->nb) != s->nb) throw Fail{KR_INVALID_INPUT, "this rank's board count differs"};
    KR_CK(cudaSetDevice(s->device));
    KR_CK(cudaDeviceSynchronize());
    if (s->ownBufs) {
        if (s->gathered != s->contrib) krb::dev_free(s->gathered);
        krb::dev_free(s->contrib);
    }
    krb::dev_free(s->d_bpre);
    s->contrib = s->gathered = nullptr;
    s->d_bpre = nullptr;
    s->world = world;
    s->rank = rank;
    s->nbMax = std::max(nbMax, 1);
    const int64_t count = int64_t(s->T) * s->m * s->nbMax;
    if (send) {
        s->contrib = send;
        s->gathered = recv;
        s->ownBufs = false;
    } else {
        s->contrib = krb::dev_alloc<double>(std::max<int64_t>(count, 1));
        s->gathered = world == 1 ? s->contrib : krb::dev_alloc<double>(std::max<int64_t>(count * world, 1));
        s->ownBufs = true;
    }
    s->d_bpre = krb::dev_alloc<int32_t>(world + 1);
    KR_CK(cudaMemcpy(s->d_bpre, pre.data(), 4 * pre.size(), cudaMemcpyHostToDevice));
}
}  // namespace

int kr_turn_solver_set_exchange(kr_turn_solver* s, void (*fn)(void*), void* user, int world, int rank,
                                const int32_t* boards_per_rank, double* send, double* recv) {
    return guarded([&] {
        if (!s) throw Fail{KR_INVALID_INPUT, "null solver"};
        if (fn && (!boards_per_rank || !send || !recv))
            throw Fail{KR_INVALID_INPUT, "an exchange needs the boards of every rank and its two buffers"};
        s->comm = nullptr;
        s->xfn = nullptr;
        s->xuser = nullptr;
        if (!fn) {
            turn_shards(s, 1, 0, nullptr);
            return;
        }
        turn_shards(s, world, rank, boards_per_rank, send, recv);
        s->xfn = fn;
        s->xuser = user;
    });
}

int kr_turn_solver_set_comm(kr_turn_solver* s, kr_comm* c, const int32_t* boards_per_rank) {
    return guarded([&] {
        if (!s) throw Fail{KR_INVALID_INPUT, "null solver"};
        s->comm = nullptr;
        s->xfn = nullptr;
        if (!c) {
            turn_shards(s, 1, 0, nullptr);
            return;
        }
        if (!boards_per_rank) throw Fail{KR_INVALID_INPUT, "a communicator needs the boards of every rank"};
        if (krb::comm_device(c) != s->device) throw Fail{KR_INVALID_INPUT, "communicator and solver on different devices"};
        turn_shards(s, krb::comm_size(c), krb::comm_rank(c), boards_per_rank);
        s->comm = c;
    });
}

int kr_turn_solver_sizes(const kr_turn_solver* s, int64_t out[4]) {
    return guarded([&] {
        if (!s || !out) throw Fail{KR_INVALID_INPUT, "null argument"};
        out[0] = s->off[0].back();
        out[1] = s->off[1].back();
        out[2] = int64_t(s->T) * s->m;  // exchanged values per board (kr_turn_solver_set_exchange)
        out[3] = s->Hr;
    });
}

}  // extern "C"
