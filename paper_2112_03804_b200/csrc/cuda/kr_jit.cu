// kr_jit.cu — the DCFR player step compiled for the instance's own treeplex.
//
// The player step (cfrSweep -> sequenceForm -> discount -> average,
// solver.hpp:222-264, 374-387) walks the same small tree (15 decision nodes,
// 43 sequences per player at configs 2 / 3) for every hand.  The generic
// kernels (k_player_team) read that tree from shared-memory tables, split a
// hand's nodes over 4 lanes that synchronise level by level, and stage every
// per-hand array (regrets, values, node values: 816 B per hand) in shared
// memory, which caps residency at ~256 hands per SM and spends ~17,000
// thread-instructions per hand on table walks and index arithmetic.
//
// Here the tree is compiled in.  At solver creation the host emits CUDA C for
// the tree — straight-line code, one thread per hand, the hand's regrets and
// node values in registers, every index a constant — and compiles it with
// NVRTC for sm_100a (-fmad=false, as the library).  Each node performs the
// reference's operations in the reference's order (the same expressions as
// k_player_team, which is bitwise the oracle), so results are bit-identical.
// A CTA is one warp of 32 hands: the 32 x n tile of each hand-major array is
// contiguous in HBM, so whole tiles move with TMA bulk copies through one
// tile buffer (32 n doubles, 344 B per hand at n = 43): regrets in (to
// registers), gradients in, x out while the lanes stream the averages with
// coalesced loads, regrets out.  Lane h reads row h of the tile with stride n
// (conflict-free for odd n).  With ~12 CTAs per SM (168 registers) config 3's
// 51,888 hands run in one round and the kernel is bound by its HBM traffic
// (6 x 8 n bytes per hand).
//
// NVRTC is bound at run time (dlopen, like NCCL in kr_comm.cu).  When it is
// missing, or the tree is too large for registers, the solver keeps the
// generic kernels (kr_solver_step_kind reports which one runs).
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "kr_common.cuh"
#include "kr_jit.cuh"

namespace krb {
namespace {

struct NvrtcApi {
    decltype(&::nvrtcCreateProgram) create = nullptr;
    decltype(&::nvrtcCompileProgram) compile = nullptr;
    decltype(&::nvrtcGetCUBINSize) cubinSize = nullptr;
    decltype(&::nvrtcGetCUBIN) cubin = nullptr;
    decltype(&::nvrtcGetProgramLogSize) logSize = nullptr;
    decltype(&::nvrtcGetProgramLog) log = nullptr;
    decltype(&::nvrtcDestroyProgram) destroy = nullptr;
    bool ok = false;
};

const NvrtcApi& nvrtc() {
    static NvrtcApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"})
            if (!h) h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
        if (const char* p = std::getenv("KR_NVRTC_LIB"))
            if (!h) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.create = reinterpret_cast<decltype(api.create)>(sym("nvrtcCreateProgram"));
        api.compile = reinterpret_cast<decltype(api.compile)>(sym("nvrtcCompileProgram"));
        api.cubinSize = reinterpret_cast<decltype(api.cubinSize)>(sym("nvrtcGetCUBINSize"));
        api.cubin = reinterpret_cast<decltype(api.cubin)>(sym("nvrtcGetCUBIN"));
        api.logSize = reinterpret_cast<decltype(api.logSize)>(sym("nvrtcGetProgramLogSize"));
        api.log = reinterpret_cast<decltype(api.log)>(sym("nvrtcGetProgramLog"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(sym("nvrtcDestroyProgram"));
        api.ok = api.create && api.compile && api.cubinSize && api.cubin && api.logSize && api.log && api.destroy;
    });
    return api;
}

// The device helpers every generated kernel starts with: mbarrier-tracked
// bulk copies global -> shared, bulk stores shared -> global, proxy fences.
const char* kPreamble = R"(
typedef unsigned long long u64;
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(u64* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(u64* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(u64* b, unsigned parity) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W_%=;\n\t}" :: "r"(sa(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, unsigned bytes, u64* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst), "r"(sa(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
)";

// Level structure of a levelled treeplex (append_levels in kr_solver.cu).
struct Levels {
    int n = 0, nn = 0, nlev = 0;
    std::vector<int> aptr, aseq, parentSeq, lev;
    std::vector<std::vector<int>> levNodes;       // per level, ascending node id
    std::vector<std::vector<int>> children;       // per sequence 0..n: child nodes, descending
};

bool levels_of(const kr_treeplex& t, Levels& L) {
    L.n = t.n_seq;
    L.nn = t.n_nodes;
    L.aptr.assign(t.node_action_ptr, t.node_action_ptr + t.n_nodes + 1);
    L.aseq.assign(t.action_seq, t.action_seq + t.node_action_ptr[t.n_nodes]);
    L.parentSeq.assign(t.node_parent_seq, t.node_parent_seq + t.n_nodes);
    std::vector<int> owner(size_t(L.n) + 1, -1);
    for (int v = 0; v < L.nn; ++v)
        for (int a = L.aptr[size_t(v)]; a < L.aptr[size_t(v) + 1]; ++a) owner[size_t(L.aseq[size_t(a)])] = v;
    L.lev.assign(size_t(L.nn), 0);
    for (int v = 0; v < L.nn; ++v) {
        const int ps = L.parentSeq[size_t(v)];
        if (ps == 0) L.lev[size_t(v)] = 0;
        else if (owner[size_t(ps)] >= 0 && owner[size_t(ps)] < v) L.lev[size_t(v)] = L.lev[size_t(owner[size_t(ps)])] + 1;
        else return false;
        L.nlev = std::max(L.nlev, L.lev[size_t(v)] + 1);
    }
    L.levNodes.assign(size_t(L.nlev), {});
    for (int v = 0; v < L.nn; ++v) L.levNodes[size_t(L.lev[size_t(v)])].push_back(v);
    L.children.assign(size_t(L.n) + 1, {});
    for (int v = L.nn - 1; v >= 0; --v) L.children[size_t(L.parentSeq[size_t(v)])].push_back(v);
    return true;
}

// rm_stats of kr_solver.cu (regretMatch, solver.hpp:166-194) over the values
// vals[0..cnt) into locals <p>pos / <p>sum / <p>cut / <p>uni.
void emit_stats(std::ostringstream& o, const std::string& p, const std::vector<std::string>& vals) {
    o << "  double " << p << "best = " << vals[0] << ";\n";
    o << "  double " << p << "mab = fabs(" << p << "best);\n";
    o << "  double " << p << "sum = " << p << "best > 0 ? 0.0 + " << p << "best : 0.0;\n";
    for (size_t a = 1; a < vals.size(); ++a) {
        o << "  { const double r_ = " << vals[a] << "; " << p << "best = (" << p << "best < r_) ? r_ : " << p
          << "best; const double ar_ = fabs(r_); " << p << "mab = (" << p << "mab < ar_) ? ar_ : " << p
          << "mab; if (r_ > 0) " << p << "sum += r_; }\n";
    }
    o << "  const double " << p << "tol = 1e-9 * (1 + " << p << "mab);\n";
    o << "  const bool " << p << "pos = " << p << "best > " << p << "tol;\n";
    o << "  const double " << p << "cut = " << p << "best - " << p << "tol;\n";
    o << "  double " << p << "uni = 0;\n";
    // 1.0 / ties for ties in 1..cnt: the correctly rounded constants the
    // division produces (the compiler folds 1.0 / k exactly), no runtime divide
    o << "  if (!" << p << "pos) { int ties_ = 0;";
    for (const auto& v : vals) o << " if (" << v << " >= " << p << "cut) ++ties_;";
    o << " " << p << "uni = ties_ == 0 ? __longlong_as_double(0x7ff0000000000000ll) : ";   // 1.0 / 0
    for (size_t k = 1; k < vals.size(); ++k) o << "ties_ == " << k << " ? 1.0 / " << k << ".0 : ";
    o << "1.0 / " << vals.size() << ".0; }\n";
}

std::string prob(const std::string& p, const std::string& v) {
    return "(" + p + "pos ? (" + v + " > 0 ? " + v + " / " + p + "sum : 0.0) : (" + v + " >= " + p + "cut ? " + p +
           "uni : 0.0))";
}

std::string reg(int sq) { return "r" + std::to_string(sq - 1); }       // regret of sequence sq
std::string val(int sq) { return "Gh[" + std::to_string(sq - 1) + "]"; }  // value / probability / reach of sq

// One decision node of the sweep (k_player_team mode 1, per node): regret
// matching on the pre-update regrets, the node value, the regret update, the
// rule's discount, the post-update strategy into the value slots.  child(c)
// is the expression holding child node c's value.
template <class Child>
void emit_node(std::ostringstream& o, const Levels& L, int v, int rule, Child&& child) {
    const int a0 = L.aptr[size_t(v)], cnt = L.aptr[size_t(v) + 1] - a0;
    std::vector<int> seqs(L.aseq.begin() + a0, L.aseq.begin() + a0 + cnt);
    const std::string p = "s" + std::to_string(v) + "_";
    o << "  {\n";
    std::vector<std::string> rv;
    for (int sq : seqs) rv.push_back(reg(sq));
    emit_stats(o, p, rv);
    o << "  double nodeVal = 0;\n";
    for (int a = 0; a < cnt; ++a) {
        const int sq = seqs[size_t(a)];
        o << "  double ev" << a << ";\n  { double cs = 0.0;";
        for (int c : L.children[size_t(sq)]) o << " cs += " << child(c) << ";";
        o << " if (ex) cs += ex[" << sq - 1 << "];";
        o << " const double gr = " << val(sq) << "; const double gv = negate ? -gr : gr; ev" << a
          << " = gv + cs; nodeVal += " << prob(p, reg(sq)) << " * ev" << a << "; }\n";
    }
    for (int a = 0; a < cnt; ++a) {
        const int sq = seqs[size_t(a)];
        o << "  const double d" << a << " = ev" << a << " - nodeVal; " << reg(sq) << " += d" << a << ";\n";
    }
    o << "  nv" << v << " = nodeVal;\n";
    if (rule != 0)
        for (int sq : seqs) o << "  " << reg(sq) << " = " << reg(sq) << " * (" << reg(sq) << " > 0 ? pos : neg);\n";
    const std::string q = "t" + std::to_string(v) + "_";
    if (rule == 2) {  // PRM+: match R + d
        std::vector<std::string> w;
        for (int a = 0; a < cnt; ++a) {
            o << "  const double w" << a << " = " << reg(seqs[size_t(a)]) << " + d" << a << ";\n";
            w.push_back("w" + std::to_string(a));
        }
        emit_stats(o, q, w);
        for (int a = 0; a < cnt; ++a) o << "  " << val(seqs[size_t(a)]) << " = " << prob(q, w[size_t(a)]) << ";\n";
    } else {
        emit_stats(o, q, rv);
        for (int sq : seqs) o << "  " << val(sq) << " = " << prob(q, reg(sq)) << ";\n";
    }
    o << "  }\n";
}

// sequenceForm for node v's actions: reach = mass * prob (V[0] = 1.0)
void emit_reach(std::ostringstream& o, const Levels& L, int v) {
    const int ps = L.parentSeq[size_t(v)];
    for (int a = L.aptr[size_t(v)]; a < L.aptr[size_t(v) + 1]; ++a) {
        const int sq = L.aseq[size_t(a)];
        o << "  " << val(sq) << " = " << (ps == 0 ? std::string("1.0") : val(ps)) << " * " << val(sq) << ";\n";
    }
}

// The kernel source for one player's tree and update rule (mode 1 of
// k_player_team: sweep, sequence form, discount, average).
// layout: 0 hand-major; 1 gradients and strategies sequence-major per board
// (implicit engine); 2 strategies sequence-major over all hands (Kronecker-
// factored engine), gradients hand-major.
std::string generate(const Levels& L, int rule, int minBlocks, int hands, int layout) {
    std::ostringstream o;
    const int N = L.n;
    o << kPreamble;
    o << "#define N " << N << "\n#define HB " << hands << "\n";
    o << "#define MINB " << minBlocks << "\n#define GSEQ " << (layout == 1 ? 1 : 0) << "\n#define XSEQ " << layout
      << "\n";
    {
        const char* k = std::getenv("KR_JIT_STAGGER_K");   // CTAs start at K staggered times
        o << "#define STAGGER_K " << (k ? std::max(2, std::atoi(k)) : 3) << "\n";
    }
    o << R"(extern "C" __global__ void __launch_bounds__(HB, MINB) kr_step(const double* __restrict__ g, int negate,
    double* __restrict__ regret, double* __restrict__ xout, double* __restrict__ avg, double pos, double neg,
    double shrink, const double* __restrict__ fac, const int* __restrict__ dt, int noAvg,
    double* __restrict__ rootOut, const double* __restrict__ extra, long long H,
    const long long* __restrict__ bstart, int nb, int stagger) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) double G[];  // tile: regrets in, then gradients -> values -> probabilities -> x
  __shared__ __align__(8) u64 bar;
  if (fac) { const int t = *dt; pos = fac[3 * t]; neg = fac[3 * t + 1]; shrink = fac[3 * t + 2]; }
  // stagger (ns): a full-GPU grid runs as one round whose CTAs would all
  // move their tiles, then all compute; starting two thirds of them stagger /
  // 2 x stagger late lets the others' transfers overlap their compute (+2% at
  // config 3; the bits are the same whatever the order, every hand being
  // independent).  0 where other kernels share the GPU (turn continuations).
  if (stagger > 0 && gridDim.x >= 2 * 148 && blockIdx.x % STAGGER_K)
    __nanosleep(unsigned(stagger) * (blockIdx.x % STAGGER_K));
  const int lane = threadIdx.x;
  const long long h0 = (long long)blockIdx.x * HB;
  const int nh = (int)(H - h0 < HB ? H - h0 : HB);
  const long long e0 = h0 * N;
  const int ne = nh * N;
  const unsigned bytes = HB * N * 8;
  // whole tiles move by TMA when every tile address is 16-byte aligned (the
  // turn solver's per-continuation blocks start at arbitrary offsets)
  const bool full = nh == HB && (((unsigned long long)(regret + e0) | (GSEQ ? 0ull : (unsigned long long)(g + e0)) |
                                   (XSEQ ? 0ull : (unsigned long long)(xout + e0)) |
                                   (noAvg ? 0ull : (unsigned long long)(avg + e0))) & 15ull) == 0;
  if (full) {
    if (lane == 0) {
      bar_init(&bar);
      bar_expect(&bar, bytes);
      g2s(G, regret + e0, bytes, &bar);
      if (!GSEQ) l2_prefetch(g + e0, bytes);      // the next tile in, and the averages
      if (!noAvg) l2_prefetch(avg + e0, bytes);   // streamed at the end, wait in L2
    }
    __syncthreads();
    bar_wait(&bar, 0);
  } else {
    for (int q = lane; q < ne; q += HB) G[q] = regret[e0 + q];
    __syncthreads();
  }
  double* Gh = G + lane * N;
)";
    for (int i = 0; i < N; ++i) o << "  double r" << i << " = Gh[" << i << "];\n";
    o << R"(  __syncthreads();
  // GSEQ / XSEQ == 1: gradients / strategies sequence-major per board (the
  // implicit engine's coalesced layout, [seq][hand] from the board's first
  // hand times N): lane h reads / writes its own hand's N values, m apart.
  // XSEQ == 2: strategies sequence-major over all hands, [seq][hand] (the
  // Kronecker-factored engine's staging layout), H apart.
  long long gb = 0, gm = 1;
  if ((GSEQ || XSEQ == 1) && lane < nh) {
    const long long hg = h0 + lane;
    int lo = 0, hi = nb;
    while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (bstart[mid] <= hg) lo = mid; else hi = mid; }
    gb = bstart[lo] * N + (hg - bstart[lo]);
    gm = bstart[lo + 1] - bstart[lo];
  }
  if (XSEQ == 2) { gb = h0 + lane; gm = H; }
  if (GSEQ) {
    if (lane < nh) {
#pragma unroll
      for (int q = 0; q < N; ++q) Gh[q] = g[gb + q * gm];
    }
    __syncthreads();
  } else if (full) {
    if (lane == 0) { fence_async(); bar_expect(&bar, bytes); g2s(G, g + e0, bytes, &bar); }
    __syncthreads();
    bar_wait(&bar, 1);
  } else {
    for (int q = lane; q < ne; q += HB) G[q] = g[e0 + q];
    __syncthreads();
  }
  if (lane < nh) {
    const double* ex = extra ? extra + (h0 + lane) * N : nullptr;
)";
    for (int v = 0; v < L.nn; ++v) o << "  double nv" << v << ";\n";
    // cfrSweep, deepest level first (k_player_team mode 1)
    for (int l = L.nlev - 1; l >= 0; --l)
        for (int v : L.levNodes[size_t(l)]) emit_node(o, L, v, rule, [](int c) { return "nv" + std::to_string(c); });
    // seqVal[0]: root nodes, descending
    o << "  if (rootOut) { double acc = 0.0;";
    for (auto it = L.levNodes[0].rbegin(); it != L.levNodes[0].rend(); ++it) o << " acc += nv" << *it << ";";
    o << " rootOut[h0 + lane] = acc; }\n";
    // sequenceForm: reach = mass * prob, root level first
    for (int l = 0; l < L.nlev; ++l)
        for (int v : L.levNodes[size_t(l)]) emit_reach(o, L, v);
    if (rule == 0)  // discount (solver.hpp:262-264)
        for (int sq = 1; sq <= N; ++sq)
            o << "  " << reg(sq) << " = " << reg(sq) << " * (" << reg(sq) << " > 0 ? pos : neg);\n";
    o << R"(  }
  __syncthreads();
  if (XSEQ) {
    if (lane < nh) {
#pragma unroll
      for (int q = 0; q < N; ++q) xout[gb + q * gm] = Gh[q];
    }
  } else if (full) {  // x out by TMA while the lanes stream the averages (solver.hpp:382-386)
    fence_async();
    __syncthreads();
    if (lane == 0) { s2g(xout + e0, G, bytes); bulk_commit(); }
  } else {
    for (int q = lane; q < ne; q += HB) xout[e0 + q] = G[q];
  }
  if (!noAvg) {
#pragma unroll 8
    for (int q = lane; q < ne; q += HB) avg[e0 + q] = (avg[e0 + q] + G[q]) * shrink;
  }
  if (full && lane == 0) bulk_wait_read();
  __syncthreads();
)";
    for (int i = 0; i < N; ++i) o << "  Gh[" << i << "] = r" << i << ";\n";
    o << R"(  if (full) {
    fence_async();
    __syncthreads();
    if (lane == 0) { s2g(regret + e0, G, bytes); bulk_commit(); bulk_wait_all(); }
  } else {
    __syncthreads();
    for (int q = lane; q < ne; q += HB) regret[e0 + q] = G[q];
  }
}
)";
    return o.str();
}

// Minimum resident CTAs per SM the step is compiled for (__launch_bounds__):
// 12 caps it at 168 registers (a few hundred bytes of spills at n = 43) so
// that 384 hands fit an SM (config 3's 51,888 hands in one round); 1 lets
// ptxas use ~228 (KR_JIT_MINB overrides).
// Hands (threads) per CTA: 128 (four warps that wait on the same tile
// barriers and run the same code together, so they share instruction fetch;
// KR_JIT_HANDS overrides: 32, 64, 128 or 256).
int jit_hands() {
    if (const char* e = std::getenv("KR_JIT_HANDS")) {
        const int h = std::atoi(e);
        if (h == 32 || h == 64 || h == 128 || h == 256) return h;
    }
    return 128;
}

// Two-group kernels: resident 64-thread units per SM they are compiled for
// (KR_JIT_PAIR_MINB overrides; 11 caps registers at ~93).
int jit_pair_min_blocks() {
    if (const char* e = std::getenv("KR_JIT_PAIR_MINB")) return std::max(1, std::atoi(e));
    return 11;
}

int jit_min_blocks() {
    if (const char* e = std::getenv("KR_JIT_MINB")) return std::max(1, std::atoi(e));
    return 12;
}

// Two warp groups per hand set: group 0 owns the level-0 (root) nodes and
// part of the subtrees below them, group 1 the other subtrees, balanced by
// action count.  Each thread holds only its group's regrets (about half), so
// twice the warps fit an SM.  Group 1 hands its subtree roots' node values to
// group 0 through shared memory; group 0 hands the root sequences' reach back.
// Returns false when the tree has no level-1 node to give group 1.
struct Split {
    int groups = 1;
    std::vector<int> grp;     // per node: its group
    std::vector<int> slot;    // per node: exchange slot (level-1 nodes of groups > 0), else -1
    int nx = 0;
};

// Up to `want` groups: the level-1 subtrees dealt greedily (heaviest first,
// by action count) to the lightest group, group 0 also holding the roots.
bool split_tree(const Levels& L, Split& S, int want = 2) {
    if (L.nlev < 2 || want < 2) return false;
    std::vector<int> owner(size_t(L.n) + 1, -1);
    for (int v = 0; v < L.nn; ++v)
        for (int a = L.aptr[size_t(v)]; a < L.aptr[size_t(v) + 1]; ++a) owner[size_t(L.aseq[size_t(a)])] = v;
    std::vector<int> sub(size_t(L.nn), -1), weight(size_t(L.nn), 0);
    std::vector<int> w(size_t(want), 0);
    for (int v = 0; v < L.nn; ++v) {
        const int acts = L.aptr[size_t(v) + 1] - L.aptr[size_t(v)];
        if (L.lev[size_t(v)] == 0) {
            w[0] += acts;
            continue;
        }
        int u = v;
        while (L.lev[size_t(u)] > 1) u = owner[size_t(L.parentSeq[size_t(u)])];
        sub[size_t(v)] = u;
        weight[size_t(u)] += acts;
    }
    std::vector<int> roots(L.levNodes[1]);
    std::sort(roots.begin(), roots.end(), [&](int x, int y) {
        return weight[size_t(x)] != weight[size_t(y)] ? weight[size_t(x)] > weight[size_t(y)] : x < y;
    });
    std::vector<int> rootGrp(size_t(L.nn), 0);
    for (int u : roots) {
        int best = 0;   // the lightest group, preferring groups other than 0 on ties
        for (int q = 1; q < want; ++q)
            if (w[size_t(q)] <= w[size_t(best)]) best = q;
        rootGrp[size_t(u)] = best;
        w[size_t(best)] += weight[size_t(u)];
    }
    int used = 1;
    for (int q = 1; q < want; ++q)
        if (w[size_t(q)] > 0) used = q + 1;
    if (used < 2) return false;
    for (int q = 1; q < used; ++q)
        if (w[size_t(q)] == 0) return false;   // keep the groups contiguous
    S.groups = used;
    S.grp.assign(size_t(L.nn), 0);
    S.slot.assign(size_t(L.nn), -1);
    for (int v = 0; v < L.nn; ++v)
        if (L.lev[size_t(v)] > 0) S.grp[size_t(v)] = rootGrp[size_t(sub[size_t(v)])];
    for (int v : L.levNodes[1])
        if (S.grp[size_t(v)] > 0) S.slot[size_t(v)] = S.nx++;
    return true;
}

std::string generate_pair(const Levels& L, const Split& S, int rule, int minBlocks, int hands, int layout = 0) {
    std::ostringstream o;
    const int N = L.n;
    o << kPreamble;
    o << "#define N " << N << "\n#define HB " << hands << "\n#define NT (" << S.groups << " * HB)\n#define NX "
      << std::max(S.nx, 1) << "\n";
    o << "#define MINB " << minBlocks << "\n#define GSEQ " << (layout == 1 ? 1 : 0) << "\n#define XSEQ " << layout
      << "\n";
    o << R"(__device__ __forceinline__ void bar_all() { asm volatile("barrier.sync 1, %0;" :: "n"(NT) : "memory"); }
extern "C" __global__ void __launch_bounds__(NT, MINB) kr_step(const double* __restrict__ g, int negate,
    double* __restrict__ regret, double* __restrict__ xout, double* __restrict__ avg, double pos, double neg,
    double shrink, const double* __restrict__ fac, const int* __restrict__ dt, int noAvg,
    double* __restrict__ rootOut, const double* __restrict__ extra, long long H,
    const long long* __restrict__ bstart, int nb, int stagger) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) double G[];  // tile: regrets in, then gradients -> values -> probabilities -> x
  double* X = G + HB * N;                        // group 1 -> group 0: subtree roots' node values
  __shared__ __align__(8) u64 bar;
  if (fac) { const int t = *dt; pos = fac[3 * t]; neg = fac[3 * t + 1]; shrink = fac[3 * t + 2]; }
  const int tid = threadIdx.x, grp = tid / HB, hand = tid - grp * HB;
  const long long h0 = (long long)blockIdx.x * HB;
  const int nh = (int)(H - h0 < HB ? H - h0 : HB);
  const long long e0 = h0 * N;
  const int ne = nh * N;
  const unsigned bytes = HB * N * 8;
  const bool full = nh == HB && (((unsigned long long)(regret + e0) | (GSEQ ? 0ull : (unsigned long long)(g + e0)) |
                                   (XSEQ ? 0ull : (unsigned long long)(xout + e0)) |
                                   (noAvg ? 0ull : (unsigned long long)(avg + e0))) & 15ull) == 0;
  if (full) {
    if (tid == 0) {
      bar_init(&bar);
      bar_expect(&bar, bytes);
      g2s(G, regret + e0, bytes, &bar);
      if (!GSEQ) l2_prefetch(g + e0, bytes);
      if (!noAvg) l2_prefetch(avg + e0, bytes);
    }
    bar_all();
    bar_wait(&bar, 0);
  } else {
    for (int q = tid; q < ne; q += NT) G[q] = regret[e0 + q];
    bar_all();
  }
  double* Gh = G + hand * N;
  double* Xh = X + hand * NX;
  const bool valid = hand < nh;
  const double* ex = (extra && valid) ? extra + (h0 + hand) * N : nullptr;
  // sequence-major layouts (as the one-thread kernel): this hand's N values
  // m apart from gb (per board, XSEQ / GSEQ 1) or H apart (XSEQ 2)
  long long gb = 0, gm = 1;
  if ((GSEQ || XSEQ == 1) && valid) {
    const long long hg = h0 + hand;
    int lo = 0, hi = nb;
    while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (bstart[mid] <= hg) lo = mid; else hi = mid; }
    gb = bstart[lo] * N + (hg - bstart[lo]);
    gm = bstart[lo + 1] - bstart[lo];
  }
  if (XSEQ == 2) { gb = h0 + hand; gm = H; }
)";
    // the part both groups run between their own sections (same barrier sequence)
    const std::string loadTile = R"(  bar_all();
  if (full) {
    if (tid == 0) { fence_async(); bar_expect(&bar, bytes); g2s(G, g + e0, bytes, &bar); }
    bar_wait(&bar, 1);
  } else {
    for (int q = tid; q < ne; q += NT) G[q] = g[e0 + q];
  }
  bar_all();
)";
    const std::string outTile = R"(  bar_all();
  if (full) {
    fence_async();
    bar_all();
    if (tid == 0) { s2g(xout + e0, G, bytes); bulk_commit(); }
  } else {
    for (int q = tid; q < ne; q += NT) xout[e0 + q] = G[q];
  }
)";
    const std::string outAvg = R"(  if (!noAvg) {
#pragma unroll 8
    for (int q = tid; q < ne; q += NT) avg[e0 + q] = (avg[e0 + q] + G[q]) * shrink;
  }
  if (full && tid == 0) bulk_wait_read();
  bar_all();
)";
    const std::string outR = R"(  if (full) {
    fence_async();
    bar_all();
    if (tid == 0) { s2g(regret + e0, G, bytes); bulk_commit(); bulk_wait_all(); }
  } else {
    bar_all();
    for (int q = tid; q < ne; q += NT) regret[e0 + q] = G[q];
  }
)";
    for (int gi = 0; gi < S.groups; ++gi) {
        std::vector<int> mine;   // sequences of this group's nodes
        for (int v = 0; v < L.nn; ++v)
            if (S.grp[size_t(v)] == gi)
                for (int a = L.aptr[size_t(v)]; a < L.aptr[size_t(v) + 1]; ++a) mine.push_back(L.aseq[size_t(a)]);
        std::sort(mine.begin(), mine.end());
        o << (gi == 0 ? "  if (grp == 0) {\n" : "  } else if (grp == " + std::to_string(gi) + ") {\n");
        for (int sq : mine) o << "  double " << reg(sq) << " = " << val(sq) << ";\n";
        for (int v = 0; v < L.nn; ++v)
            if (S.grp[size_t(v)] == gi) o << "  double nv" << v << " = 0.0;\n";
        if (layout == 1) {   // each group gathers its own sequences' gradients
            o << "  bar_all();\n  if (valid) {\n";
            for (int sq : mine) o << "    " << val(sq) << " = g[gb + " << sq - 1 << " * gm];\n";
            o << "  }\n  bar_all();\n";
        } else {
            o << loadTile;
        }
        // the group's nodes below level 0, deepest level first
        o << "  if (valid) {\n";
        for (int l = L.nlev - 1; l >= 1; --l)
            for (int v : L.levNodes[size_t(l)])
                if (S.grp[size_t(v)] == gi) emit_node(o, L, v, rule, [](int c) { return "nv" + std::to_string(c); });
        if (gi > 0)
            for (int v : L.levNodes[1])
                if (S.grp[size_t(v)] == gi) o << "  Xh[" << S.slot[size_t(v)] << "] = nv" << v << ";\n";
        o << "  }\n  bar_all();\n";   // B: the other groups' subtree values are in X
        if (gi == 0) {
            o << "  if (valid) {\n";
            for (int v : L.levNodes[0])
                emit_node(o, L, v, rule, [&](int c) {
                    return S.grp[size_t(c)] > 0 ? "Xh[" + std::to_string(S.slot[size_t(c)]) + "]"
                                                : "nv" + std::to_string(c);
                });
            o << "  if (rootOut) { double acc = 0.0;";
            for (auto it = L.levNodes[0].rbegin(); it != L.levNodes[0].rend(); ++it) o << " acc += nv" << *it << ";";
            o << " rootOut[h0 + hand] = acc; }\n";
            for (int v : L.levNodes[0]) emit_reach(o, L, v);
            o << "  }\n";
        }
        o << "  bar_all();\n";   // C: the root sequences' reach is in G
        o << "  if (valid) {\n";
        for (int l = 1; l < L.nlev; ++l)
            for (int v : L.levNodes[size_t(l)])
                if (S.grp[size_t(v)] == gi) emit_reach(o, L, v);
        if (rule == 0)
            for (int sq : mine) o << "  " << reg(sq) << " = " << reg(sq) << " * (" << reg(sq) << " > 0 ? pos : neg);\n";
        o << "  }\n";
        if (layout) {   // each group writes its own sequences' strategies
            o << "  bar_all();\n  if (valid) {\n";
            for (int sq : mine) o << "    xout[gb + " << sq - 1 << " * gm] = " << val(sq) << ";\n";
            o << "  }\n";
        } else {
            o << outTile;
        }
        o << outAvg;
        for (int sq : mine) o << "  " << val(sq) << " = " << reg(sq) << ";\n";
        o << outR;
    }
    o << "  }\n}\n";
    return o.str();
}

struct Gen {
    std::string src;
    int hands = 0, threads = 0;   // hands and threads per CTA
    size_t smem = 0;              // dynamic shared memory per CTA
};

// The source for the tree.  groups > 1: the hand set's tree split over that
// many warp groups (small grids: single boards, where one thread per hand
// leaves most SMs idle), 32 hands per CTA; empty when the tree does not split
// that way.  Otherwise one thread per hand, compiled for the resident CTAs
// per SM that one round of config 3's hands needs; KR_JIT_SPLIT=1: two warp
// groups per hand set (80 registers, twice the warps, but the groups wait on
// each other: within 1-2% of the one-thread kernel at config 3,
// profiles/r02/jit_step_probe_r02z.log).
Gen jit_source(const Levels& L, int rule, int hands, int layout, int groups) {
    Gen r;
    Split S;
    const char* e = std::getenv("KR_JIT_SPLIT");
    if (groups > 1) {
        if (!split_tree(L, S, groups)) return r;
        r.src = generate_pair(L, S, rule, 1, 32, layout);
        r.hands = 32;
        r.threads = 32 * S.groups;
        r.smem = size_t(32) * size_t(L.n + std::max(S.nx, 1)) * sizeof(double);
        return r;
    }
    if (!layout && e && std::atoi(e) == 1 && split_tree(L, S)) {
        const int hb = std::max(32, hands / 2);   // hands per CTA; 2 x hb threads
        r.src = generate_pair(L, S, rule, std::max(1, jit_pair_min_blocks() * 64 / (2 * hb)), hb);
        r.hands = hb;
        r.threads = 2 * hb;
        r.smem = size_t(hb) * size_t(L.n + S.nx) * sizeof(double);
        return r;
    }
    r.src = generate(L, rule, std::max(1, jit_min_blocks() * 32 / hands), hands, layout);
    r.hands = r.threads = hands;
    r.smem = size_t(hands) * size_t(L.n) * sizeof(double);
    return r;
}

struct Compiled {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kern = nullptr;
    std::string log;
};

std::mutex g_jit_mu;
std::map<std::string, Compiled>& jit_cache() {
    static std::map<std::string, Compiled> m;
    return m;
}

}  // namespace

bool jit_step_compile(const kr_treeplex& t, int rule, JitStep& out, std::string& why, int layout, int groups) {
    out = JitStep{};
    if (const char* env = std::getenv("KR_STEP"))
        if (std::string(env) != "jit") {
            why = "KR_STEP=" + std::string(env);
            return false;
        }
    if (t.n_seq < 1 || t.n_seq > kJitMaxSeq) {
        why = "treeplex has " + std::to_string(t.n_seq) + " sequences (compiled step: 1.." +
              std::to_string(kJitMaxSeq) + ")";
        return false;
    }
    Levels L;
    if (!levels_of(t, L)) {
        why = "treeplex is not level-ordered";
        return false;
    }
    const NvrtcApi& api = nvrtc();
    if (!api.ok) {
        why = "NVRTC not available";
        return false;
    }
    const Gen gen = jit_source(L, rule, jit_hands(), layout, groups);
    const std::string& src = gen.src;
    if (src.empty()) {
        why = "treeplex does not split into " + std::to_string(groups) + " warp groups";
        return false;
    }
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = jit_cache().find(src);
    if (it == jit_cache().end()) {
        Compiled c;
        nvrtcProgram prog = nullptr;
        if (api.create(&prog, src.c_str(), "kr_step.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
            why = "nvrtcCreateProgram failed";
            return false;
        }
        const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17", "-lineinfo",
                              "--ptxas-options=-v"};
        const nvrtcResult r = api.compile(prog, 5, opts);
        size_t ls = 0;
        api.logSize(prog, &ls);
        c.log.resize(ls);
        if (ls) api.log(prog, &c.log[0]);
        if (r != NVRTC_SUCCESS) {
            api.destroy(&prog);
            why = "NVRTC compile failed: " + c.log;
            return false;
        }
        size_t cs = 0;
        api.cubinSize(prog, &cs);
        std::vector<char> cubin(cs);
        api.cubin(prog, cubin.data());
        api.destroy(&prog);
        if (cudaLibraryLoadData(&c.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
            cudaLibraryGetKernel(&c.kern, c.lib, "kr_step") != cudaSuccess) {
            cudaGetLastError();
            why = "loading the compiled step failed";
            return false;
        }
        it = jit_cache().emplace(src, std::move(c)).first;
    }
    // ptxas' spills of the compiled step (its -v report): a tree whose
    // regrets overflow the register budget runs slower than the generic team
    // kernel (the 91-sequence tree: 1,265 against 1,804 it/s), so heavy
    // spilling keeps the generic kernel
    {
        const std::string& lg = it->second.log;
        const size_t at = lg.find(" bytes spill stores");
        if (at != std::string::npos) {
            size_t b = lg.rfind(' ', at - 1);
            const long spills = std::strtol(lg.c_str() + (b == std::string::npos ? 0 : b + 1), nullptr, 10);
            const char* lim = std::getenv("KR_JIT_MAX_SPILL");
            if (spills > (lim ? std::atol(lim) : 1024)) {
                why = "compiled step spills " + std::to_string(spills) + " bytes per thread";
                return false;
            }
        }
    }
    out.kern = it->second.kern;
    out.layout = layout;
    out.n = t.n_seq;
    out.hands = gen.hands;
    out.threads = gen.threads;
    out.smem = gen.smem;
    out.log = it->second.log;
    return true;
}

int jit_stagger_ns() {
    if (const char* e = std::getenv("KR_JIT_STAGGER")) return std::max(0, std::atoi(e));
    return 4000;
}

void jit_step_launch(const JitStep& j, int device, int64_t H, const double* g, int negate, double* regret,
                     double* xout, double* avg, double pos, double neg, double shrink, const double* fac,
                     const int* dt, int noAvg, double* rootOut, const double* extra, cudaStream_t st,
                     const int64_t* bstart, int nb, int stagger) {
    const unsigned grid = unsigned((H + j.hands - 1) / j.hands);
    if (grid == 0) return;
    if (j.smem > 48 * 1024) {   // once per kernel and device
        static std::mutex mu;
        static std::map<std::pair<cudaKernel_t, int>, size_t> done;
        std::lock_guard<std::mutex> lk(mu);
        size_t& have = done[{j.kern, device}];
        if (have < j.smem) {
            KR_CK(cudaKernelSetAttributeForDevice(j.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(j.smem),
                                                  device));
            have = j.smem;
        }
    }
    long long Hl = H;
    void* args[] = {&g,   &negate, &regret,  &xout,  &avg, &pos,    &neg, &shrink, &fac,
                    &dt,  &noAvg,  &rootOut, &extra, &Hl,  &bstart, &nb,  &stagger};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(unsigned(j.threads));
    cfg.dynamicSmemBytes = j.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    unsigned& prev = last_grid(st);
    cfg.numAttrs = pdl_enabled(grid, prev, true) ? 1 : 0;
    prev = grid;
    KR_CK(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(j.kern), args));
}

std::string jit_step_source(const kr_treeplex& t, int rule, int layout, int groups) {
    Levels L;
    if (!levels_of(t, L)) return "";
    return jit_source(L, rule, jit_hands(), layout, groups).src;
}

}  // namespace krb
