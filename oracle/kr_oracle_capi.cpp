// kr_oracle_capi.cpp — C ABI over the CPU ORACLE (test infrastructure only).
// Loaded by tests/ (via oracle/pyoracle.py), __graft_entry__.smoke() and the
// cpu_baseline leg of bench.py.  Never by the product.
#include <chrono>
#include <cstring>
#include <memory>
#include <random>
#include <thread>

#include "kr_oracle.hpp"

using namespace kro;

namespace {
thread_local std::string g_err;
thread_local std::string g_code;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        g_code = e.code;
        if (e.code == "INVALID_INPUT") return 1;
        if (e.code == "PARSE") return 2;
        if (e.code == "GUARD_EXCEEDED") return 4;
        if (e.code == "DEGENERATE_BELIEFS") return 5;
        if (e.code == "CONTRACT") return 6;
        return 7;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_code = "INTERNAL";
        return 7;
    }
}

struct Inst {
    RiverInstance inst;
    KronPayoff kp;
};
struct Sp {
    Sparsification s;
};

SpMat fromArrays(bool rowMajor, int64_t rows, int64_t cols, const int64_t* outer, const int32_t* inner,
                 const double* val) {
    SpMat m;
    m.rowMajor = rowMajor;
    m.rows = rows;
    m.cols = cols;
    int64_t no = rowMajor ? rows : cols;
    m.outer.assign(outer, outer + no + 1);
    int64_t nnz = outer[no];
    m.inner.assign(inner, inner + nnz);
    m.val.assign(val, val + nnz);
    return m;
}
}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }
const char* or_last_code() { return g_code.c_str(); }

// name: golden | twenty_card | bluffing | all_tie | random_small | bench |
//       river_full (board code in `board`, deck "standard52" or "26" ranks x {c,d})
int or_builtin(const char* name, uint64_t seed, int hands, int shared, const char* board, int deckKind, int tree,
               void** out) {
    return guarded([&] {
        std::string n(name);
        auto h = std::make_unique<Inst>();
        if (n == "golden") h->inst = goldenInstance();
        else if (n == "twenty_card") h->inst = twentyCardInstance();
        else if (n == "bluffing") h->inst = bluffingInstance();
        else if (n == "all_tie") h->inst = allTieInstance();
        else if (n == "random_small") {
            std::mt19937_64 rng(seed);
            for (int skip = 0; skip < shared; ++skip) (void)randomSmallInstance(rng, hands);  // n-th draw of a stream
            h->inst = randomSmallInstance(rng, hands);
        } else if (n == "bench") h->inst = benchInstance(seed, hands, shared);
        else if (n == "river_full") {
            Deck deck = Deck::standard52();
            if (deckKind == 26) {
                deck.cards.clear();
                for (int r = 2; r <= 14; ++r)
                    for (int s = 0; s < 2; ++s) deck.cards.emplace_back(r, s);
            }
            BettingConfig cfg = tree == 3 ? threeBetConfig() : referenceBettingConfig();
            if (tree == 91) {  // menus {0.33, 0.75, 1.5}, raise cap 3
                cfg = threeBetConfig();
                for (int x = 0; x < kBetContexts; ++x) cfg.menu1[x] = cfg.menu2[x] = {0.33, 0.75, 1.5};
            }
            h->inst = fullRangeRiver(Board::fromCode(board), deck, seed, cfg);
        } else throw InvalidInputError("unknown builtin '" + n + "'");
        h->kp = assemble(h->inst);
        *out = h.release();
    });
}

// Instance from parsed JSON fields (tests parse JSON in Python, mirroring
// instance_io.hpp:103-229).  hands: 4-char codes concatenated; menus:
// counts[2*5] then values; raiseCap < 0 means none; deck NULL = standard52.
int or_instance(const char* board, const char* deck, int nHands1, const char* hands1, const double* w1,
                int nHands2, const char* hands2, const double* w2, double stack1, double stack2, double pot,
                const int* menuCounts, const double* menuValues, int allIn, int raiseCap, void** out) {
    return guarded([&] {
        BettingConfig cfg;
        cfg.stack1 = stack1;
        cfg.stack2 = stack2;
        cfg.potContribution = pot;
        int k = 0;
        for (int p = 0; p < 2; ++p)
            for (int c = 0; c < kBetContexts; ++c) {
                auto& m = p == 0 ? cfg.menu1[c] : cfg.menu2[c];
                for (int q = 0; q < menuCounts[p * kBetContexts + c]; ++q) m.push_back(menuValues[k++]);
            }
        cfg.allIn = allIn != 0;
        if (raiseCap >= 0) cfg.raiseCap = raiseCap;
        Deck d = Deck::standard52();
        if (deck) {
            d.cards.clear();
            size_t L = std::strlen(deck);
            for (size_t i = 0; i + 1 < L; i += 2) d.cards.push_back(Card::fromCode(std::string_view(deck + i, 2)));
        }
        std::vector<Hand> h1, h2;
        for (int i = 0; i < nHands1; ++i) h1.push_back(Hand::fromCode(std::string_view(hands1 + 4 * i, 4)));
        for (int i = 0; i < nHands2; ++i) h2.push_back(Hand::fromCode(std::string_view(hands2 + 4 * i, 4)));
        auto h = std::make_unique<Inst>();
        h->inst = makeRiverInstance(Board::fromCode(board), h1, std::vector<double>(w1, w1 + nHands1), h2,
                                    std::vector<double>(w2, w2 + nHands2), cfg, d);
        h->kp = assemble(h->inst);
        *out = h.release();
    });
}

void or_instance_free(void* h) { delete static_cast<Inst*>(h); }

// out: m1 m2 n1 n2 rows cols nodes dec0 dec1 terminals folds showdowns nnzF nnzS
void or_inst_dims(void* h, int64_t* out) {
    const auto& kp = static_cast<Inst*>(h)->kp;
    const Skeleton& sk = kp.skeleton;
    int folds = 0;
    for (const auto& t : sk.terminals) folds += t.fold ? 1 : 0;
    int64_t v[] = {kp.m1(), kp.m2(), kp.n1, kp.n2, kp.rows(), kp.cols(), int64_t(sk.nodes.size()),
                   sk.decisionNodes(0), sk.decisionNodes(1), int64_t(sk.terminals.size()), folds,
                   int64_t(sk.terminals.size()) - folds, kp.F.nnz(), kp.S.nnz()};
    std::memcpy(out, v, sizeof(v));
}
double or_inst_beta(void* h) { return static_cast<Inst*>(h)->kp.beta; }
void or_inst_hands(void* h, int player, char* out) {
    const auto& hs = static_cast<Inst*>(h)->inst.hands[player];
    for (size_t i = 0; i < hs.size(); ++i) std::memcpy(out + 4 * i, hs[i].code().data(), 4);
}
void or_inst_vectors(void* h, double* mu1, double* mu2, double* lam1, double* lam2) {
    const auto& kp = static_cast<Inst*>(h)->kp;
    std::memcpy(mu1, kp.mu1.data(), kp.mu1.size() * 8);
    std::memcpy(mu2, kp.mu2.data(), kp.mu2.size() * 8);
    std::memcpy(lam1, kp.lambda1.data(), kp.lambda1.size() * 8);
    std::memcpy(lam2, kp.lambda2.data(), kp.lambda2.size() * 8);
}
void or_inst_W(void* h, double* W, double* Hx) {
    const auto& kp = static_cast<Inst*>(h)->kp;
    std::memcpy(W, kp.W.data(), kp.W.size() * 8);
    std::memcpy(Hx, kp.Hcross.data(), kp.Hcross.size() * 8);
}
// terminals: per terminal [fold, folder, seq1, seq2] ints and [q1, q2] doubles
void or_inst_terminals(void* h, int32_t* ints, double* qs, char* paths, int pathStride) {
    const auto& sk = static_cast<Inst*>(h)->kp.skeleton;
    for (size_t t = 0; t < sk.terminals.size(); ++t) {
        const auto& T = sk.terminals[t];
        ints[4 * t] = T.fold;
        ints[4 * t + 1] = T.folder;
        ints[4 * t + 2] = T.seq1;
        ints[4 * t + 3] = T.seq2;
        qs[2 * t] = T.q1;
        qs[2 * t + 1] = T.q2;
        std::memset(paths + t * pathStride, 0, pathStride);
        std::memcpy(paths + t * pathStride, T.path.data(), std::min<size_t>(T.path.size(), pathStride - 1));
    }
}
// treeplex: for each player node (preorder) : parentSeq, nActions, then action seqs
// returns number of ints written (call with out=NULL to size)
int or_inst_treeplex(void* h, int player, int32_t* out) {
    const auto& sk = static_cast<Inst*>(h)->kp.skeleton;
    int k = 0;
    for (int idx : sk.playerNodes[player]) {
        const auto& v = sk.nodes[idx];
        if (out) out[k] = v.parentSeq(player);
        ++k;
        if (out) out[k] = int(v.actions.size());
        ++k;
        for (const auto& a : v.actions) {
            if (out) out[k] = a.seq;
            ++k;
        }
    }
    return k;
}
// F and S (CSR n1 x n2)
void or_inst_FS(void* h, int which, int64_t* outer, int32_t* inner, double* val) {
    const auto& kp = static_cast<Inst*>(h)->kp;
    const SpMat& m = which == 0 ? kp.F : kp.S;
    std::memcpy(outer, m.outer.data(), m.outer.size() * 8);
    std::memcpy(inner, m.inner.data(), m.inner.size() * 4);
    std::memcpy(val, m.val.data(), m.val.size() * 8);
}

// sparsifyW (sparsify.hpp:68-103) on a dense row-major W: rank and the
// nnz of What, U, V.
int or_peel(const double* W, int rows, int cols, int maxIters, int64_t* out) {
    return guarded([&] {
        WFactorization wf = sparsifyW(std::vector<double>(W, W + size_t(rows) * cols), rows, cols, maxIters);
        out[0] = wf.rank();
        out[1] = wf.What.nnz();
        out[2] = wf.U.nnz();
        out[3] = wf.V.nnz();
    });
}

int64_t or_dense_nnz(void* h) { return densePayoffNonzeros(static_cast<Inst*>(h)->kp); }
int or_dense_expand(void* h, double guard, double* out) {
    return guarded([&] {
        auto A = denseExpand(static_cast<Inst*>(h)->kp, guard);
        std::memcpy(out, A.data(), A.size() * 8);
    });
}

// technique 0 = A (peel with peelIters), 1 = B
int or_sparsify(void* h, int technique, int post, int peelIters, void** out) {
    return guarded([&] {
        const auto& kp = static_cast<Inst*>(h)->kp;
        auto s = std::make_unique<Sp>();
        if (technique == 0) s->s = techniqueA(kp, sparsifyW(kp.W, kp.m1(), kp.m2(), peelIters));
        else s->s = techniqueB(kp);
        if (post) s->s = postprocess(s->s);
        *out = s.release();
    });
}
// Technique B with postprocessing (sparsify.hpp:246-406) from raw KronPayoff
// pieces instead of an instance: strength keys and cards per hand (W_ij =
// sign(key1_i - key2_j) for disjoint hands, H× = 1 for overlapping ones, as
// assemble builds them, kron.hpp:134-166), lambda1 / lambda2 as given, F and S
// as CSR.  The turn checker (turn_oracle.py) uses it to apply each block of a
// turn game with the reference's factored matvec.
int or_sparsify_pieces(int m1, int m2, int n1, int n2, const uint32_t* key1, const uint32_t* key2,
                       const uint8_t* cards1, const uint8_t* cards2, const double* l1, const double* l2,
                       const int64_t* fptr, const int32_t* fcol, const double* fval, const int64_t* sptr,
                       const int32_t* scol, const double* sval, void** out) {
    return guarded([&] {
        KronPayoff kp;
        kp.n1 = n1;
        kp.n2 = n2;
        kp.hands[0].resize(size_t(m1));
        kp.hands[1].resize(size_t(m2));
        kp.lambda1.assign(l1, l1 + m1);
        kp.lambda2.assign(l2, l2 + m2);
        kp.W.assign(size_t(m1) * m2, 0.0);
        kp.Hcross.assign(size_t(m1) * m2, 0.0);
        for (int i = 0; i < m1; ++i)
            for (int j = 0; j < m2; ++j) {
                const int a0 = cards1[2 * i], a1 = cards1[2 * i + 1], b0 = cards2[2 * j], b1 = cards2[2 * j + 1];
                const bool ok = a0 != b0 && a0 != b1 && a1 != b0 && a1 != b1;
                kp.Hcross[size_t(i) * m2 + j] = ok ? 0.0 : 1.0;
                kp.W[size_t(i) * m2 + j] = ok ? (key1[i] > key2[j] ? 1.0 : (key1[i] < key2[j] ? -1.0 : 0.0)) : 0.0;
            }
        kp.F = fromArrays(true, n1, n2, fptr, fcol, fval);
        kp.S = fromArrays(true, n1, n2, sptr, scol, sval);
        auto sp = std::make_unique<Sp>();
        sp->s = postprocess(techniqueB(kp));
        *out = sp.release();
    });
}

int or_postprocess(void* sp, void** out) {
    return guarded([&] {
        auto s = std::make_unique<Sp>();
        s->s = postprocess(static_cast<Sp*>(sp)->s);
        *out = s.release();
    });
}
void or_sp_free(void* h) { delete static_cast<Sp*>(h); }
// out: rows cols k nnzA nnzU nnzM nnzV technique postprocessed
void or_sp_sizes(void* h, int64_t* out) {
    const auto& s = static_cast<Sp*>(h)->s;
    int64_t v[] = {s.rows(), s.cols(), s.k(), s.Ahat.nnz(), s.U.nnz(), s.M.nnz(), s.V.nnz(),
                   s.technique == Technique::A ? 0 : 1, s.postprocessed ? 1 : 0};
    std::memcpy(out, v, sizeof(v));
}
// which: 0 Ahat (CSR) 1 U (CSR) 2 M (CSC) 3 V (CSC)
void or_sp_export(void* h, int which, int64_t* outer, int32_t* inner, double* val) {
    const auto& s = static_cast<Sp*>(h)->s;
    const SpMat& m = which == 0 ? s.Ahat : which == 1 ? s.U : which == 2 ? s.M : s.V;
    std::memcpy(outer, m.outer.data(), m.outer.size() * 8);
    std::memcpy(inner, m.inner.data(), m.inner.size() * 4);
    std::memcpy(val, m.val.data(), m.val.size() * 8);
}
int or_sp_from_arrays(int64_t rows, int64_t cols, int64_t k, const int64_t* aO, const int32_t* aI, const double* aV,
                      const int64_t* uO, const int32_t* uI, const double* uV, const int64_t* mO, const int32_t* mI,
                      const double* mV, const int64_t* vO, const int32_t* vI, const double* vV, int technique,
                      int post, int validate, void** out) {
    return guarded([&] {
        auto s = std::make_unique<Sp>();
        s->s.Ahat = fromArrays(true, rows, cols, aO, aI, aV);
        s->s.U = fromArrays(true, rows, k, uO, uI, uV);
        s->s.M = fromArrays(false, k, k, mO, mI, mV);
        s->s.V = fromArrays(false, cols, k, vO, vI, vV);
        s->s.technique = technique == 0 ? Technique::A : Technique::B;
        s->s.postprocessed = post != 0;
        if (validate) validateSparsification(s->s);
        *out = s.release();
    });
}

int or_matvec(void* sp, const double* x, int64_t n, double* y, int64_t* flops) {
    return guarded([&] {
        GradientWorkspace ws;
        Vec xv(x, x + n);
        Vec out = matvec(static_cast<Sp*>(sp)->s, xv, ws);
        std::memcpy(y, out.data(), out.size() * 8);
        if (flops) *flops = ws.flops;
    });
}
int or_matvec_t(void* sp, const double* y, int64_t n, double* x, int64_t* flops) {
    return guarded([&] {
        GradientWorkspace ws;
        Vec yv(y, y + n);
        Vec out = matvecTranspose(static_cast<Sp*>(sp)->s, yv, ws);
        std::memcpy(x, out.data(), out.size() * 8);
        if (flops) *flops = ws.flops;
    });
}
// Repeated single-thread matvec pairs for the CPU baseline: returns seconds.
double or_time_pairs(void* sp, const double* x, const double* y, int reps, double* sink) {
    const auto& s = static_cast<Sp*>(sp)->s;
    GradientWorkspace ws;
    Vec xv(x, x + s.cols()), yv(y, y + s.rows());
    double acc = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
        Vec a = matvec(s, xv, ws);
        Vec b = matvecTranspose(s, yv, ws);
        acc += a[0] + b[0];
    }
    double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (sink) *sink = acc;
    return sec;
}
// Same, with `threads` independent sparsifications processed concurrently
// (one per thread: the multi-board CPU baseline; the reference engine itself
// is sequential per call).  Inputs are dense Gaussians from
// std::mt19937_64(seed + board) as the reference's bench draws them
// (tools/main.cpp:313-317): the reference skips exact zeros
// (engine.hpp:38, 105-106, 119-120, 127), so sparse inputs would flatter it.
// The inputs are drawn before the clock starts.
double or_time_pairs_multi(void** sps, int count, int threads, int reps, double* sink) {
    std::vector<std::thread> pool;
    std::vector<double> sinks(size_t(threads), 0.0);
    std::vector<Vec> xs(static_cast<size_t>(count)), ys(static_cast<size_t>(count));
    for (int b = 0; b < count; ++b) {
        const auto& s = static_cast<Sp*>(sps[b])->s;
        std::mt19937_64 rng(1 + uint64_t(b));
        std::normal_distribution<double> gauss;
        xs[size_t(b)].resize(size_t(s.cols()));
        ys[size_t(b)].resize(size_t(s.rows()));
        for (auto& v : xs[size_t(b)]) v = gauss(rng);
        for (auto& v : ys[size_t(b)]) v = gauss(rng);
    }
    auto t0 = std::chrono::steady_clock::now();
    for (int th = 0; th < threads; ++th)
        pool.emplace_back([&, th] {
            for (int b = th; b < count; b += threads) {
                const auto& s = static_cast<Sp*>(sps[b])->s;
                GradientWorkspace ws;
                const Vec& xv = xs[size_t(b)];
                const Vec& yv = ys[size_t(b)];
                for (int r = 0; r < reps; ++r) {
                    Vec a = matvec(s, xv, ws);
                    Vec c = matvecTranspose(s, yv, ws);
                    sinks[th] += a[0] + c[0];
                }
            }
        });
    for (auto& t : pool) t.join();
    double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (sink) {
        *sink = 0;
        for (double v : sinks) *sink += v;
    }
    return sec;
}
// DCFR iterations (solver.hpp:365-388, default parameters) on `count`
// independent boards, one board per host thread at a time: the CPU side of
// the solver-iterations/s baseline.  Returns wall seconds.
double or_time_dcfr_multi(void** insts, void** sps, int count, int threads, int iters, double* sink) {
    std::vector<std::thread> pool;
    std::vector<double> sinks(size_t(threads), 0.0);
    auto t0 = std::chrono::steady_clock::now();
    for (int th = 0; th < threads; ++th)
        pool.emplace_back([&, th] {
            for (int b = th; b < count; b += threads) {
                const auto& kp = static_cast<Inst*>(insts[b])->kp;
                FactoredEngine eng(static_cast<Sp*>(sps[b])->s);
                DcfrState st(kp, eng);
                st.begin(DcfrParams{});
                st.iterate(iters);
                sinks[th] += st.x1.empty() ? 0.0 : st.x1[0];
            }
        });
    for (auto& t : pool) t.join();
    double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (sink) {
        *sink = 0;
        for (double v : sinks) *sink += v;
    }
    return sec;
}

int or_reference_matvec(void* h, const double* x, int64_t n, double* y) {
    return guarded([&] {
        Vec out = referenceMatvec(static_cast<Inst*>(h)->kp, Vec(x, x + n));
        std::memcpy(y, out.data(), out.size() * 8);
    });
}
int or_reference_matvec_t(void* h, const double* y, int64_t n, double* x) {
    return guarded([&] {
        Vec out = referenceMatvecT(static_cast<Inst*>(h)->kp, Vec(y, y + n));
        std::memcpy(x, out.data(), out.size() * 8);
    });
}
int or_uniform(void* h, int player, double* out) {
    return guarded([&] {
        Vec x = uniformStrategy(static_cast<Inst*>(h)->kp, player);
        std::memcpy(out, x.data(), x.size() * 8);
    });
}
int or_best_response(void* h, void* sp, int player, const double* opp, double* out) {
    return guarded([&] {
        const auto& kp = static_cast<Inst*>(h)->kp;
        FactoredEngine eng(static_cast<Sp*>(sp)->s);
        int64_t n = player == 0 ? kp.cols() : kp.rows();
        *out = bestResponseValue(kp, eng, player, Vec(opp, opp + n));
    });
}

// Incremental DCFR over one board (test driver for the multi-rank path).
struct DcfrHandle {
    FactoredEngine eng;
    DcfrState st;
    DcfrHandle(const KronPayoff& kp, const Sparsification& s) : eng(s), st(kp, eng) {}
};
int or_dcfr_state_create(void* h, void* sp, void** out) {
    return guarded([&] {
        *out = new DcfrHandle(static_cast<Inst*>(h)->kp, static_cast<Sp*>(sp)->s);
    });
}
void or_dcfr_state_free(void* s) { delete static_cast<DcfrHandle*>(s); }
int or_dcfr_begin(void* s, double alpha, double beta, double gamma, int rule) {
    return guarded([&] {
        DcfrParams p;
        p.rule = rule;
        p.alpha = alpha;
        p.beta = beta;
        p.gamma = gamma;
        static_cast<DcfrHandle*>(s)->st.begin(p);
    });
}
int or_dcfr_iterate(void* s, int n) {
    return guarded([&] { static_cast<DcfrHandle*>(s)->st.iterate(n); });
}
int or_dcfr_checkpoint(void* s, double* br1, double* br2) {
    return guarded([&] { static_cast<DcfrHandle*>(s)->st.checkpoint(br1, br2); });
}

// engine: 0 factored (sp), 1 reference block formula, 2 dense
// trace arrays sized >= number of checkpoints.  Returns trace length in *ntrace.
int or_dcfr(void* h, void* sp, int engineKind, double alpha, double beta, double gamma, int maxIters,
            double target, int checkpointEvery, int* iterations, double* expl, int64_t* flops, int* traceIter,
            double* traceExpl, double* traceBr1, double* traceBr2, int traceCap, int* ntrace, double* avg1,
            double* avg2, double* seconds, int rule) {
    return guarded([&] {
        const auto& kp = static_cast<Inst*>(h)->kp;
        DcfrParams p;
        p.rule = rule;
        p.alpha = alpha;
        p.beta = beta;
        p.gamma = gamma;
        p.maxIters = maxIters;
        p.targetExploitability = target;
        p.checkpointEvery = checkpointEvery;
        std::unique_ptr<GradientEngine> eng;
        std::vector<double> dense;
        if (engineKind == 0) eng = std::make_unique<FactoredEngine>(static_cast<Sp*>(sp)->s);
        else if (engineKind == 1) eng = std::make_unique<ReferenceEngine>(kp);
        else eng = std::make_unique<DenseEngine>(denseExpand(kp), kp.rows(), kp.cols());
        auto t0 = std::chrono::steady_clock::now();
        DcfrResult r = dcfrSolve(kp, *eng, p);
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *iterations = r.iterations;
        *expl = r.exploitability;
        *flops = r.gradientFlops;
        int n = std::min<int>(traceCap, int(r.trace.size()));
        for (int i = 0; i < n; ++i) {
            traceIter[i] = r.trace[i].iteration;
            traceExpl[i] = r.trace[i].exploitability;
            traceBr1[i] = r.trace[i].br1;
            traceBr2[i] = r.trace[i].br2;
        }
        *ntrace = int(r.trace.size());
        if (avg1) std::memcpy(avg1, r.avg1.data(), r.avg1.size() * 8);
        if (avg2) std::memcpy(avg2, r.avg2.data(), r.avg2.size() * 8);
    });
}

}  // extern "C"
