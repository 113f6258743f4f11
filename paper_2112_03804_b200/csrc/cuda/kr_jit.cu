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
    o << "  if (!" << p << "pos) { int ties_ = 0;";
    for (const auto& v : vals) o << " if (" << v << " >= " << p << "cut) ++ties_;";
    o << " " << p << "uni = 1.0 / ties_; }\n";
}

std::string prob(const std::string& p, const std::string& v) {
    return "(" + p + "pos ? (" + v + " > 0 ? " + v + " / " + p + "sum : 0.0) : (" + v + " >= " + p + "cut ? " + p +
           "uni : 0.0))";
}

std::string reg(int sq) { return "r" + std::to_string(sq - 1); }       // regret of sequence sq
std::string val(int sq) { return "Gh[" + std::to_string(sq - 1) + "]"; }  // value / probability / reach of sq

// The kernel source for one player's tree and update rule (mode 1 of
// k_player_team: sweep, sequence form, discount, average).
std::string generate(const Levels& L, int rule, int minBlocks, int hands) {
    std::ostringstream o;
    const int N = L.n;
    o << kPreamble;
    o << "#define N " << N << "\n#define HB " << hands << "\n";
    o << "#define MINB " << minBlocks << "\n";
    o << R"(extern "C" __global__ void __launch_bounds__(HB, MINB) kr_step(const double* __restrict__ g, int negate,
    double* __restrict__ regret, double* __restrict__ xout, double* __restrict__ avg, double pos, double neg,
    double shrink, const double* __restrict__ fac, const int* __restrict__ dt, int noAvg,
    double* __restrict__ rootOut, const double* __restrict__ extra, long long H) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) double G[];  // tile: regrets in, then gradients -> values -> probabilities -> x
  __shared__ __align__(8) u64 bar;
  if (fac) { const int t = *dt; pos = fac[3 * t]; neg = fac[3 * t + 1]; shrink = fac[3 * t + 2]; }
  const int lane = threadIdx.x;
  const long long h0 = (long long)blockIdx.x * HB;
  const int nh = (int)(H - h0 < HB ? H - h0 : HB);
  const long long e0 = h0 * N;
  const int ne = nh * N;
  const unsigned bytes = HB * N * 8;
  // whole tiles move by TMA when every tile address is 16-byte aligned (the
  // turn solver's per-continuation blocks start at arbitrary offsets)
  const bool full = nh == HB && (((unsigned long long)(regret + e0) | (unsigned long long)(g + e0) |
                                   (unsigned long long)(xout + e0) | (noAvg ? 0ull : (unsigned long long)(avg + e0))) &
                                  15ull) == 0;
  if (full) {
    if (lane == 0) {
      bar_init(&bar);
      bar_expect(&bar, bytes);
      g2s(G, regret + e0, bytes, &bar);
      l2_prefetch(g + e0, bytes);                 // the next tile in, and the averages
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
  if (full) {
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
    // cfrSweep, deepest level first (k_player_team mode 1)
    for (int l = L.nlev - 1; l >= 0; --l)
        for (int v : L.levNodes[size_t(l)]) {
            const int a0 = L.aptr[size_t(v)], cnt = L.aptr[size_t(v) + 1] - a0;
            std::vector<int> seqs(L.aseq.begin() + a0, L.aseq.begin() + a0 + cnt);
            const std::string p = "s" + std::to_string(v) + "_";
            o << "  double nv" << v << ";\n  {\n";
            std::vector<std::string> rv;
            for (int sq : seqs) rv.push_back(reg(sq));
            emit_stats(o, p, rv);
            o << "  double nodeVal = 0;\n";
            for (int a = 0; a < cnt; ++a) {
                const int sq = seqs[size_t(a)];
                o << "  double ev" << a << ";\n  { double cs = 0.0;";
                for (int c : L.children[size_t(sq)]) o << " cs += nv" << c << ";";
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
                for (int sq : seqs)
                    o << "  " << reg(sq) << " = " << reg(sq) << " * (" << reg(sq) << " > 0 ? pos : neg);\n";
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
    // seqVal[0]: root nodes, descending
    o << "  if (rootOut) { double acc = 0.0;";
    for (auto it = L.levNodes[0].rbegin(); it != L.levNodes[0].rend(); ++it) o << " acc += nv" << *it << ";";
    o << " rootOut[h0 + lane] = acc; }\n";
    // sequenceForm: reach = mass * prob, root level first
    for (int l = 0; l < L.nlev; ++l)
        for (int v : L.levNodes[size_t(l)]) {
            const int ps = L.parentSeq[size_t(v)];
            for (int a = L.aptr[size_t(v)]; a < L.aptr[size_t(v) + 1]; ++a) {
                const int sq = L.aseq[size_t(a)];
                o << "  " << val(sq) << " = " << (ps == 0 ? std::string("1.0") : val(ps)) << " * " << val(sq) << ";\n";
            }
        }
    if (rule == 0)  // discount (solver.hpp:262-264)
        for (int sq = 1; sq <= N; ++sq)
            o << "  " << reg(sq) << " = " << reg(sq) << " * (" << reg(sq) << " > 0 ? pos : neg);\n";
    o << R"(  }
  __syncthreads();
  if (full) {  // x out by TMA while the lanes stream the averages (solver.hpp:382-386)
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

int jit_min_blocks() {
    if (const char* e = std::getenv("KR_JIT_MINB")) return std::max(1, std::atoi(e));
    return 12;
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

bool jit_step_compile(const kr_treeplex& t, int rule, JitStep& out, std::string& why) {
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
    const int hands = jit_hands();
    const std::string src = generate(L, rule, jit_min_blocks() * 32 / hands, hands);
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
    out.kern = it->second.kern;
    out.n = t.n_seq;
    out.hands = hands;
    out.smem = size_t(hands) * size_t(t.n_seq) * sizeof(double);
    out.log = it->second.log;
    return true;
}

void jit_step_launch(const JitStep& j, int device, int64_t H, const double* g, int negate, double* regret,
                     double* xout, double* avg, double pos, double neg, double shrink, const double* fac,
                     const int* dt, int noAvg, double* rootOut, const double* extra, cudaStream_t st) {
    const unsigned grid = unsigned((H + j.hands - 1) / j.hands);
    if (grid == 0) return;
    if (j.smem > 48 * 1024) {
        static std::mutex mu;
        std::lock_guard<std::mutex> lk(mu);
        KR_CK(cudaKernelSetAttributeForDevice(j.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(j.smem),
                                              device));
    }
    long long Hl = H;
    void* args[] = {&g, &negate, &regret, &xout, &avg, &pos, &neg, &shrink, &fac, &dt, &noAvg, &rootOut, &extra, &Hl};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(unsigned(j.hands));
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

std::string jit_step_source(const kr_treeplex& t, int rule) {
    Levels L;
    if (!levels_of(t, L)) return "";
    return generate(L, rule, jit_min_blocks() * 32 / jit_hands(), jit_hands());
}

}  // namespace krb
