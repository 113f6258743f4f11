// kr_host.cpp — implementation of the host side (see kr_host.hpp) and the
// krh_* C ABI (include/kr_host.h).
#include "kr_host.hpp"

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <sstream>

#include "kr_host.h"

namespace krh {

namespace {
[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }
constexpr double kMoneyTol = 1e-6;  // skeleton.hpp:19
}  // namespace

// ---------------------------------------------------------------- cards ----
int cardFromCode(const std::string& code) {
    static const std::string kR = "23456789TJQKA", kS = "cdhs";
    if (code.size() != 2) fail(INVALID_INPUT, "bad card code '" + code + "'");
    const auto r = kR.find(code[0]), s = kS.find(code[1]);
    if (r == std::string::npos || s == std::string::npos) fail(INVALID_INPUT, "bad card code '" + code + "'");
    return int(r) * 4 + int(s);
}

std::string cardCode(int id) {
    static const char* kR = "23456789TJQKA";
    static const char* kS = "cdhs";
    return {kR[id / 4], kS[id % 4]};
}

Hand Hand::of(int a, int b) {
    if (a == b) fail(INVALID_INPUT, "hand repeats card " + cardCode(a));
    Hand h;
    h.hi = uint8_t(std::max(a, b));
    h.lo = uint8_t(std::min(a, b));
    return h;
}

Hand handFromCode(const std::string& code) {
    if (code.size() != 4) fail(INVALID_INPUT, "bad hand code '" + code + "'");
    return Hand::of(cardFromCode(code.substr(0, 2)), cardFromCode(code.substr(2, 2)));
}

namespace {
uint32_t pack(int cat, int a, int b = 0, int c = 0, int d = 0, int e = 0) {
    return (uint32_t(cat) << 20) | (uint32_t(a) << 16) | (uint32_t(b) << 12) | (uint32_t(c) << 8) | (uint32_t(d) << 4) |
           uint32_t(e);
}
// highest 5-run top rank in a rank bitmask (bit r = rank r), wheel -> 5
int runTop(uint32_t m) {
    for (int top = 14; top >= 6; --top)
        if (((m >> (top - 4)) & 0x1Fu) == 0x1Fu) return top;
    const uint32_t wheel = (1u << 14) | 0x3Cu;  // A,5,4,3,2
    return (m & wheel) == wheel ? 5 : 0;
}
// the `want` highest ranks of mask skipping x1, x2 (zero-filled)
void highest(uint32_t m, int x1, int x2, int want, int* out) {
    int got = 0;
    for (int r = 14; r >= 2 && got < want; --r)
        if (r != x1 && r != x2 && (m >> r & 1u)) out[got++] = r;
    while (got < want) out[got++] = 0;
}
}  // namespace

uint32_t strengthKey(const Hand& h, const std::array<int, 5>& board) {
    int cards[7] = {h.hi, h.lo, board[0], board[1], board[2], board[3], board[4]};
    uint64_t seen = 0;
    int cnt[15] = {}, scnt[4] = {};
    uint32_t smask[4] = {}, rmask = 0;
    for (int c : cards) {
        if (seen >> c & 1ull) fail(INVALID_INPUT, "hand shares card " + cardCode(c) + " with board");
        seen |= 1ull << c;
        const int r = c / 4 + 2, s = c % 4;
        ++cnt[r];
        ++scnt[s];
        smask[s] |= 1u << r;
        rmask |= 1u << r;
    }
    int fs = -1;
    for (int s = 0; s < 4; ++s)
        if (scnt[s] >= 5) fs = s;
    if (fs >= 0)
        if (int t = runTop(smask[fs])) return pack(8, t);
    int quad = 0, t1 = 0, t2 = 0, p1 = 0, p2 = 0;
    for (int r = 14; r >= 2; --r) {
        if (cnt[r] == 4) quad = r;
        else if (cnt[r] == 3) (t1 ? (t2 ? t2 : t2 = r) : t1 = r);
        else if (cnt[r] == 2) (p1 ? (p2 ? p2 : p2 = r) : p1 = r);
    }
    int k[5];
    if (quad) {
        highest(rmask, quad, 0, 1, k);
        return pack(7, quad, k[0]);
    }
    if (t1 && (t2 || p1)) return pack(6, t1, t2 > p1 ? t2 : p1);
    if (fs >= 0) {
        highest(smask[fs], 0, 0, 5, k);
        return pack(5, k[0], k[1], k[2], k[3], k[4]);
    }
    if (int t = runTop(rmask)) return pack(4, t);
    if (t1) {
        highest(rmask, t1, 0, 2, k);
        return pack(3, t1, k[0], k[1]);
    }
    if (p1 && p2) {
        highest(rmask, p1, p2, 1, k);
        return pack(2, p1, p2, k[0]);
    }
    if (p1) {
        highest(rmask, p1, 0, 3, k);
        return pack(1, p1, k[0], k[1], k[2]);
    }
    highest(rmask, 0, 0, 5, k);
    return pack(0, k[0], k[1], k[2], k[3], k[4]);
}

// -------------------------------------------------------------- skeleton ---
const char* const kContextNames[kContexts] = {"first_action", "facing_check", "facing_bet", "after_one_raise",
                                              "after_multiple_raises"};

void BettingConfig::validate() const {
    if (!(stack1 > 0) || !(stack2 > 0)) fail(INVALID_INPUT, "stacks must be positive");
    if (!(pot > 0)) fail(INVALID_INPUT, "pot contribution must be positive");
    for (int p = 0; p < 2; ++p)
        for (const auto& m : menu[p])
            for (double f : m)
                if (!(f > 0) || !std::isfinite(f)) fail(INVALID_INPUT, "bet fractions must be positive and finite");
    if (raiseCap && *raiseCap < 0) fail(INVALID_INPUT, "raise cap must be nonnegative");
}

namespace {
std::string token(double f) {
    char b[32];
    std::snprintf(b, sizeof b, "%g", f);
    return b;
}

// Depth-first expansion (skeleton.hpp:162-310): a node's actions all take
// sequence ids before any child is expanded; children expand in action order.
struct Builder {
    const BettingConfig& cfg;
    Skeleton& out;
    double cap;
    int expand(int player, double c1, double c2, int bets, bool checked, int ps1, int ps2, const std::string& path) {
        const double own = player == 0 ? c1 : c2, other = player == 0 ? c2 : c1;
        const bool level = std::abs(c1 - c2) <= kMoneyTol;
        const int ctx = level ? (checked ? 1 : 0) : bets <= 1 ? 2 : bets == 2 ? 3 : 4;
        const int id = int(out.nodes.size());
        out.nodes.emplace_back();
        out.playerNodes[player].push_back(id);
        {
            Node& nd = out.nodes.back();
            nd.player = player;
            nd.context = ctx;
            nd.c1 = c1;
            nd.c2 = c2;
            nd.parentSeq[0] = ps1;
            nd.parentSeq[1] = ps2;
        }
        std::vector<Action> acts;
        if (level) {
            acts.push_back(Action{0, 0, own});
        } else {
            acts.push_back(Action{1, 0, own});
            acts.push_back(Action{2, 0, other});
        }
        if (!cfg.raiseCap || bets < *cfg.raiseCap) {
            struct Cand {
                double target, fraction;
                int kind;
            };
            std::vector<Cand> cand;
            const double hi = std::max(c1, c2);
            for (double f : cfg.menu[player][ctx]) {
                double t = level ? own + f * (c1 + c2) : other + f * (2.0 * other);
                if (t > cap - kMoneyTol) t = cap;
                if (t <= hi + kMoneyTol) continue;
                cand.push_back({t, f, level ? 3 : 4});
            }
            if (cfg.allIn && cap > hi + kMoneyTol) cand.push_back({cap, 0.0, 5});
            std::stable_sort(cand.begin(), cand.end(), [](const Cand& a, const Cand& b) { return a.target < b.target; });
            for (size_t i = 0; i < cand.size(); ++i) {
                if (i && std::abs(cand[i].target - cand[i - 1].target) <= kMoneyTol) continue;
                Action a;
                a.target = cand[i].target;
                a.fraction = cand[i].fraction;
                a.kind = std::abs(a.target - cap) <= kMoneyTol ? 5 : cand[i].kind;
                acts.push_back(a);
            }
        }
        const int ownParent = player == 0 ? ps1 : ps2;
        (void)ownParent;
        for (Action& a : acts) a.seq = ++out.nseq[player];
        for (Action& a : acts) {
            const int n1 = player == 0 ? a.seq : ps1, n2 = player == 1 ? a.seq : ps2;
            const double q1 = player == 0 ? a.target : c1, q2 = player == 1 ? a.target : c2;
            static const char* const kTok[] = {"k", "f", "c", "b", "r", "a"};
            std::string tk = kTok[a.kind];
            if (a.kind == 3 || a.kind == 4) tk += token(a.fraction);
            const std::string cp = path.empty() ? tk : path + "/" + tk;
            auto leaf = [&](bool fold, double t1, double t2) {
                Terminal t;
                t.fold = fold;
                t.folder = fold ? player : -1;
                t.q1 = t1;
                t.q2 = t2;
                t.seq1 = n1;
                t.seq2 = n2;
                t.path = cp;
                out.terminals.push_back(t);
                a.terminal = true;
                a.child = int(out.terminals.size()) - 1;
            };
            if (a.kind == 0) {
                if (checked) leaf(false, c1, c2);
                else a.child = expand(1 - player, c1, c2, bets, true, n1, n2, cp);
            } else if (a.kind == 1) {
                leaf(true, c1, c2);
            } else if (a.kind == 2) {
                leaf(false, q1, q2);
            } else {
                a.child = expand(1 - player, q1, q2, bets + 1, false, n1, n2, cp);
            }
        }
        out.nodes[size_t(id)].actions = std::move(acts);
        return id;
    }
};

// Compressed matrix from (outer, inner, value) triples of one storage order:
// sorted by (outer, inner), duplicates summed in input order, zeros pruned
// (makeSparse, linalg.hpp:18-25).
Compressed compress(int64_t rows, int64_t cols, bool rowMajor, std::vector<std::tuple<int64_t, int64_t, double>> t) {
    Compressed m;
    m.rowMajor = rowMajor;
    m.rows = rows;
    m.cols = cols;
    const int64_t no = rowMajor ? rows : cols;
    std::stable_sort(t.begin(), t.end(), [&](const auto& a, const auto& b) {
        const int64_t oa = rowMajor ? std::get<0>(a) : std::get<1>(a), ob = rowMajor ? std::get<0>(b) : std::get<1>(b);
        const int64_t ia = rowMajor ? std::get<1>(a) : std::get<0>(a), ib = rowMajor ? std::get<1>(b) : std::get<0>(b);
        return oa != ob ? oa < ob : ia < ib;
    });
    m.outer.assign(size_t(no) + 1, 0);
    size_t q = 0;
    for (int64_t o = 0; o < no; ++o) {
        while (q < t.size() && (rowMajor ? std::get<0>(t[q]) : std::get<1>(t[q])) == o) {
            const int64_t in = rowMajor ? std::get<1>(t[q]) : std::get<0>(t[q]);
            double v = std::get<2>(t[q]);
            ++q;
            while (q < t.size() && (rowMajor ? std::get<0>(t[q]) : std::get<1>(t[q])) == o &&
                   (rowMajor ? std::get<1>(t[q]) : std::get<0>(t[q])) == in)
                v = v + std::get<2>(t[q++]);
            if (v != 0.0) {
                m.inner.push_back(int32_t(in));
                m.val.push_back(v);
            }
        }
        m.outer[size_t(o) + 1] = int64_t(m.val.size());
    }
    return m;
}
}  // namespace

Skeleton buildSkeleton(const BettingConfig& cfg) {
    cfg.validate();
    Skeleton sk;
    sk.config = cfg;
    Builder b{cfg, sk, cfg.pot + std::min(cfg.stack1, cfg.stack2)};
    b.expand(0, cfg.pot, cfg.pot, 0, false, 0, 0, "");
    return sk;
}

// ---------------------------------------------------------------- payoff ---
Instance makeInstance(const std::array<int, 5>& board, std::vector<int> deck, std::vector<Hand> h1,
                      std::vector<double> w1, std::vector<Hand> h2, std::vector<double> w2, const BettingConfig& cfg) {
    cfg.validate();
    uint64_t deckMask = 0, boardMask = 0;
    for (int c : deck) {
        if (deckMask >> c & 1ull) fail(INVALID_INPUT, "deck repeats card " + cardCode(c));
        deckMask |= 1ull << c;
    }
    for (int i = 0; i < 5; ++i)
        for (int j = i + 1; j < 5; ++j)
            if (board[i] == board[j]) fail(INVALID_INPUT, "board repeats card " + cardCode(board[i]));
    for (int c : board) {
        if (!(deckMask >> c & 1ull)) fail(INVALID_INPUT, "board card " + cardCode(c) + " not in the deck");
        boardMask |= 1ull << c;
    }
    Instance in;
    in.board = board;
    in.deck = std::move(deck);
    in.config = cfg;
    std::vector<Hand>* hs[2] = {&h1, &h2};
    std::vector<double>* ws[2] = {&w1, &w2};
    for (int p = 0; p < 2; ++p) {
        auto& H = *hs[p];
        auto& W = *ws[p];
        if (H.empty()) fail(INVALID_INPUT, "player " + std::to_string(p + 1) + " has no hands");
        if (H.size() != W.size())
            fail(INVALID_INPUT, "player " + std::to_string(p + 1) + ": " + std::to_string(H.size()) + " hands but " +
                                    std::to_string(W.size()) + " weights");
        for (double w : W)
            if (!(w >= 0) || !std::isfinite(w)) fail(INVALID_INPUT, "belief weights must be finite and nonnegative");
        for (const Hand& h : H) {
            if ((h.mask() & deckMask) != h.mask()) fail(INVALID_INPUT, "hand " + h.code() + " uses a card outside the deck");
            if (h.mask() & boardMask) fail(INVALID_INPUT, "hand " + h.code() + " shares a card with the board");
        }
        std::vector<uint32_t> key(H.size());
        for (size_t i = 0; i < H.size(); ++i) key[i] = strengthKey(H[i], board);
        std::vector<size_t> ord(H.size());
        std::iota(ord.begin(), ord.end(), size_t(0));
        std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
            return key[a] != key[b] ? key[a] < key[b] : H[a] < H[b];
        });
        for (size_t i : ord) {
            in.hands[p].push_back(H[i]);
            in.mu[p].push_back(W[i]);
            in.key[p].push_back(key[i]);
        }
        for (size_t i = 1; i < in.hands[p].size(); ++i)
            if (in.hands[p][i] == in.hands[p][i - 1])
                fail(INVALID_INPUT, "duplicate hand " + in.hands[p][i].code() + " for player " + std::to_string(p + 1));
    }
    // assemble (kron.hpp:134-166)
    in.sk = buildSkeleton(cfg);
    std::vector<std::tuple<int64_t, int64_t, double>> ft, st;
    for (const Terminal& t : in.sk.terminals) {
        if (t.seq1 <= 0 || t.seq2 <= 0) fail(CONTRACT, "terminal missing a sequence for one player");
        if (t.fold) ft.emplace_back(t.seq1 - 1, t.seq2 - 1, t.folder == 1 ? t.q2 : -t.q1);
        else st.emplace_back(t.seq1 - 1, t.seq2 - 1, t.q1);
    }
    in.F = compress(in.sk.nseq[0], in.sk.nseq[1], true, ft);
    in.S = compress(in.sk.nseq[0], in.sk.nseq[1], true, st);
    double beta = 0;
    for (int i = 0; i < in.m(0); ++i)
        for (int j = 0; j < in.m(1); ++j)
            if (in.compatible(i, j)) beta += in.mu[0][size_t(i)] * in.mu[1][size_t(j)];
    if (!(beta > 0)) fail(DEGENERATE, "no compatible hand pair carries belief mass");
    in.beta = beta;
    const double sb = std::sqrt(beta);
    for (int p = 0; p < 2; ++p)
        for (double m : in.mu[p]) in.lambda[p].push_back(m / sb);
    return in;
}

int64_t densePayoffNonzeros(const Instance& in) {
    const int64_t nF = in.F.nnz(), nS = in.S.nnz();
    int64_t total = 0;
    for (int i = 0; i < in.m(0); ++i)
        for (int j = 0; j < in.m(1); ++j) {
            if (in.lambda[0][size_t(i)] * in.lambda[1][size_t(j)] * (in.compatible(i, j) ? 1.0 : 0.0) == 0.0) continue;
            total += nF + (in.sign(i, j) != 0 ? nS : 0);
        }
    return total;
}

// ------------------------------------------------------------- instances ---
namespace {
std::vector<int> standardDeck() {
    std::vector<int> d(52);
    std::iota(d.begin(), d.end(), 0);
    return d;
}
std::array<int, 5> boardFromCode(const std::string& s) {
    if (s.size() != 10) fail(INVALID_INPUT, "bad board code '" + s + "'");
    std::array<int, 5> b{};
    for (int i = 0; i < 5; ++i) b[i] = cardFromCode(s.substr(size_t(2 * i), 2));
    return b;
}
}  // namespace

BettingConfig referenceBettingConfig() {  // instances.hpp:19-29
    BettingConfig c;
    c.stack1 = c.stack2 = 18125;
    c.pot = 1875;
    for (int p = 0; p < 2; ++p)
        for (auto& m : c.menu[p]) m = {0.75};
    c.allIn = true;
    return c;
}

BettingConfig threeBetConfig() {
    BettingConfig c = referenceBettingConfig();
    for (int p = 0; p < 2; ++p)
        for (auto& m : c.menu[p]) m = {0.5, 1.0};
    c.raiseCap = 3;
    return c;
}

Instance goldenInstance() {  // instances.hpp:33-43
    return makeInstance(boardFromCode("2c7d9hJc3s"), standardDeck(),
                        {handFromCode("AcAd"), handFromCode("KcKd"), handFromCode("5c5d")}, {0.5, 0.3, 0.2},
                        {handFromCode("AhAs"), handFromCode("QcQd"), handFromCode("7c7h")}, {0.4, 0.4, 0.2},
                        referenceBettingConfig());
}

Instance twentyCardInstance() {  // instances.hpp:48-68
    std::vector<int> deck;
    for (int r = 0; r < 5; ++r)
        for (int s = 0; s < 4; ++s) deck.push_back(r * 4 + s);
    const auto board = boardFromCode("2c2d4h5s6c");
    std::vector<int> rest;
    for (int c : deck)
        if (std::find(board.begin(), board.end(), c) == board.end()) rest.push_back(c);
    std::vector<Hand> hands;
    for (size_t i = 0; i < rest.size(); ++i)
        for (size_t j = i + 1; j < rest.size(); ++j) hands.push_back(Hand::of(rest[i], rest[j]));
    std::vector<double> w(hands.size(), 1.0);
    return makeInstance(board, deck, hands, w, hands, w, referenceBettingConfig());
}

Instance bluffingInstance() {  // instances.hpp:73-84
    BettingConfig c;
    c.stack1 = c.stack2 = 40;
    c.pot = 10;
    c.menu[0][0] = {1.0};
    c.allIn = false;
    return makeInstance(boardFromCode("2c2d2h3c3d"), standardDeck(), {handFromCode("3h3s"), handFromCode("4c5c")},
                        {0.5, 0.5}, {handFromCode("AcAd")}, {1.0}, c);
}

Instance allTieInstance() {  // instances.hpp:88-101
    BettingConfig c;
    c.stack1 = c.stack2 = 40;
    c.pot = 10;
    c.menu[0][0] = {1.0};
    c.menu[1][1] = {1.0};
    c.allIn = false;
    return makeInstance(boardFromCode("AsKsQsJsTs"), standardDeck(), {handFromCode("2c3c"), handFromCode("4d5d")},
                        {0.5, 0.5}, {handFromCode("2h3h"), handFromCode("4h5h")}, {0.5, 0.5}, c);
}

Instance randomSmallInstance(std::mt19937_64& rng, int handsPerSide) {  // instances.hpp:105-148
    std::vector<int> full = standardDeck();
    for (int attempt = 0; attempt < 100; ++attempt) {
        std::shuffle(full.begin(), full.end(), rng);
        const int deckSize = std::uniform_int_distribution<int>(12, 20)(rng);
        std::vector<int> deck(full.begin(), full.begin() + deckSize);
        const std::array<int, 5> board{deck[0], deck[1], deck[2], deck[3], deck[4]};
        std::vector<int> rest(deck.begin() + 5, deck.end());
        std::vector<Hand> pairs;
        for (size_t i = 0; i < rest.size(); ++i)
            for (size_t j = i + 1; j < rest.size(); ++j) pairs.push_back(Hand::of(rest[i], rest[j]));
        auto draw = [&](int count) {
            std::vector<Hand> pool = pairs;
            std::shuffle(pool.begin(), pool.end(), rng);
            pool.resize(size_t(count));
            return pool;
        };
        const int maxHands = std::min<int>(12, int(pairs.size()));
        if (handsPerSide > maxHands) continue;
        auto drawCount = [&] {
            return handsPerSide > 0 ? handsPerSide : std::uniform_int_distribution<int>(2, maxHands)(rng);
        };
        std::vector<Hand> h1 = draw(drawCount());
        std::vector<Hand> h2 = draw(drawCount());
        bool any = false;
        for (const Hand& a : h1)
            for (const Hand& b : h2)
                if (!(a.mask() & b.mask())) any = true;
        if (!any) continue;
        std::uniform_real_distribution<double> weight(0.1, 1.0);
        std::vector<double> w1, w2;
        for (size_t i = 0; i < h1.size(); ++i) w1.push_back(weight(rng));
        for (size_t i = 0; i < h2.size(); ++i) w2.push_back(weight(rng));
        return makeInstance(board, deck, h1, w1, h2, w2, referenceBettingConfig());
    }
    fail(INVALID_INPUT, "failed to draw a usable random instance");
}

Instance benchInstance(uint64_t seed, int handsPerSide, int sharedCards) {  // instances.hpp:159-194
    if (handsPerSide < 1) fail(INVALID_INPUT, "handsPerSide must be positive");
    if (sharedCards < 0 || sharedCards > 40) fail(INVALID_INPUT, "sharedCards out of range");
    std::mt19937_64 rng(seed);
    std::vector<int> deck = standardDeck();
    std::shuffle(deck.begin(), deck.end(), rng);
    const std::array<int, 5> board{deck[0], deck[1], deck[2], deck[3], deck[4]};
    std::vector<int> rest(deck.begin() + 5, deck.end());
    std::vector<int> shared(rest.begin(), rest.begin() + sharedCards);
    const size_t half = (rest.size() - size_t(sharedCards)) / 2;
    std::vector<int> pool1(rest.begin() + sharedCards, rest.begin() + sharedCards + long(half));
    std::vector<int> pool2(rest.begin() + sharedCards + long(half), rest.end());
    pool1.insert(pool1.end(), shared.begin(), shared.end());
    pool2.insert(pool2.end(), shared.begin(), shared.end());
    auto drawHands = [&](const std::vector<int>& pool) {
        std::vector<Hand> pairs;
        for (size_t i = 0; i < pool.size(); ++i)
            for (size_t j = i + 1; j < pool.size(); ++j) pairs.push_back(Hand::of(pool[i], pool[j]));
        if (pairs.size() < size_t(handsPerSide)) fail(INVALID_INPUT, "pool too small for the requested hand count");
        std::shuffle(pairs.begin(), pairs.end(), rng);
        pairs.resize(size_t(handsPerSide));
        return pairs;
    };
    std::vector<Hand> h1 = drawHands(pool1), h2 = drawHands(pool2);
    std::uniform_real_distribution<double> weight(0.25, 1.0);
    std::vector<double> w1, w2;
    for (int i = 0; i < handsPerSide; ++i) w1.push_back(weight(rng));
    for (int i = 0; i < handsPerSide; ++i) w2.push_back(weight(rng));
    return makeInstance(board, standardDeck(), h1, w1, h2, w2, referenceBettingConfig());
}

// Full-range river: every deck hand disjoint from the
// board, in canonical order; beliefs uniform_real(0.25,1) from
// mt19937_64(seed), player 1's drawn before player 2's.
Instance fullRangeRiver(const std::string& boardCode, int deckKind, uint64_t seed, const BettingConfig& cfg) {
    std::vector<int> deck;
    if (deckKind == 26) {
        for (int r = 0; r < 13; ++r)
            for (int s = 0; s < 2; ++s) deck.push_back(r * 4 + s);
    } else {
        deck = standardDeck();
    }
    const auto board = boardFromCode(boardCode);
    std::vector<int> rest;
    for (int c : deck)
        if (std::find(board.begin(), board.end(), c) == board.end()) rest.push_back(c);
    std::sort(rest.begin(), rest.end());
    std::vector<Hand> hands;
    for (size_t i = 0; i < rest.size(); ++i)
        for (size_t j = i + 1; j < rest.size(); ++j) hands.push_back(Hand::of(rest[i], rest[j]));
    std::sort(hands.begin(), hands.end());
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> weight(0.25, 1.0);
    std::vector<double> w1, w2;
    for (size_t i = 0; i < hands.size(); ++i) w1.push_back(weight(rng));
    for (size_t i = 0; i < hands.size(); ++i) w2.push_back(weight(rng));
    return makeInstance(board, deck, hands, w1, hands, w2, cfg);
}

// ------------------------------------------------------------------ JSON ---
namespace {
struct Json {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0;
    bool isInt = false;
    std::string str;
    std::vector<Json> arr;
    std::vector<std::pair<std::string, Json>> obj;
    const Json* find(const std::string& k) const {
        for (auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct JsonParser {
    const std::string& s;
    size_t p = 0;
    [[noreturn]] void bad(const std::string& m) { fail(PARSE, "invalid JSON: " + m + " at offset " + std::to_string(p)); }
    void ws() {
        while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
    }
    Json value() {
        ws();
        if (p >= s.size()) bad("unexpected end");
        const char c = s[p];
        Json j;
        if (c == '{') {
            j.kind = Json::Obj;
            ++p;
            ws();
            if (p < s.size() && s[p] == '}') {
                ++p;
                return j;
            }
            while (true) {
                ws();
                Json k = value();
                if (k.kind != Json::Str) bad("object key must be a string");
                ws();
                if (p >= s.size() || s[p] != ':') bad("expected ':'");
                ++p;
                Json v = value();
                bool replaced = false;
                for (auto& kv : j.obj)
                    if (kv.first == k.str) {
                        kv.second = v;  // duplicate keys: last wins (nlohmann behaviour)
                        replaced = true;
                    }
                if (!replaced) j.obj.emplace_back(k.str, std::move(v));
                ws();
                if (p < s.size() && s[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < s.size() && s[p] == '}') {
                    ++p;
                    break;
                }
                bad("expected ',' or '}'");
            }
        } else if (c == '[') {
            j.kind = Json::Arr;
            ++p;
            ws();
            if (p < s.size() && s[p] == ']') {
                ++p;
                return j;
            }
            while (true) {
                j.arr.push_back(value());
                ws();
                if (p < s.size() && s[p] == ',') {
                    ++p;
                    continue;
                }
                if (p < s.size() && s[p] == ']') {
                    ++p;
                    break;
                }
                bad("expected ',' or ']'");
            }
        } else if (c == '"') {
            j.kind = Json::Str;
            ++p;
            while (p < s.size() && s[p] != '"') {
                if (s[p] == '\\') {
                    ++p;
                    if (p >= s.size()) bad("bad escape");
                    const char e = s[p];
                    j.str += e == 'n' ? '\n' : e == 't' ? '\t' : e;
                } else {
                    j.str += s[p];
                }
                ++p;
            }
            if (p >= s.size()) bad("unterminated string");
            ++p;
        } else if (s.compare(p, 4, "true") == 0) {
            j.kind = Json::Bool;
            j.b = true;
            p += 4;
        } else if (s.compare(p, 5, "false") == 0) {
            j.kind = Json::Bool;
            p += 5;
        } else if (s.compare(p, 4, "null") == 0) {
            p += 4;
        } else {
            const char* b = s.c_str() + p;
            char* e = nullptr;
            errno = 0;
            const double v = std::strtod(b, &e);
            if (e == b) bad("unexpected character");
            std::string tok(b, size_t(e - b));
            j.kind = Json::Num;
            j.num = v;
            j.isInt = tok.find_first_of(".eE") == std::string::npos;
            p += size_t(e - b);
        }
        return j;
    }
};

const Json& field(const Json& j, const char* name) {
    const Json* f = j.find(name);
    if (!f) fail(PARSE, std::string("missing field '") + name + "'");
    return *f;
}
int cardField(const Json& v, const char* where) {
    if (v.kind != Json::Str) fail(PARSE, std::string("card in ") + where + " must be a string code");
    try {
        return cardFromCode(v.str);
    } catch (const Error& e) {
        fail(PARSE, std::string(where) + ": " + e.msg);
    }
}
}  // namespace

// instanceFromJson (instance_io.hpp:103-229)
Instance readInstanceJson(const std::string& path) {
    std::ifstream f(path);
    if (!f) fail(IO, "cannot open '" + path + "' for reading");
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string text = ss.str();
    JsonParser jp{text};
    Json j = jp.value();
    if (j.kind != Json::Obj) fail(PARSE, "instance file must hold a JSON object");
    const Json& ver = field(j, "schema_version");
    if (ver.kind != Json::Num || !ver.isInt || ver.num != 1) fail(PARSE, "unsupported schema_version");
    std::vector<int> deck;
    const Json& ds = field(j, "deck");
    if (ds.kind == Json::Str) {
        if (ds.str != "standard52") fail(PARSE, "deck must be \"standard52\" or an explicit card list");
        deck = standardDeck();
    } else if (ds.kind == Json::Arr) {
        uint64_t seen = 0;
        for (const Json& c : ds.arr) {
            const int id = cardField(c, "deck");
            if (seen >> id & 1ull) fail(PARSE, "deck: deck repeats card " + cardCode(id));
            seen |= 1ull << id;
            deck.push_back(id);
        }
    } else {
        fail(PARSE, "deck must be \"standard52\" or an explicit card list");
    }
    const Json& bs = field(j, "board");
    if (bs.kind != Json::Arr || bs.arr.size() != 5) fail(PARSE, "board must list exactly 5 card codes");
    std::array<int, 5> board{};
    for (int i = 0; i < 5; ++i) board[i] = cardField(bs.arr[size_t(i)], "board");
    for (int i = 0; i < 5; ++i)
        for (int k = i + 1; k < 5; ++k)
            if (board[i] == board[k]) fail(INVALID_INPUT, "board repeats card " + cardCode(board[i]));
    const Json& st = field(j, "stacks");
    if (st.kind != Json::Arr || st.arr.size() != 2 || st.arr[0].kind != Json::Num || st.arr[1].kind != Json::Num)
        fail(PARSE, "stacks must be a pair of numbers");
    BettingConfig cfg;
    cfg.stack1 = st.arr[0].num;
    cfg.stack2 = st.arr[1].num;
    const Json& pc = field(j, "pot_contribution");
    if (pc.kind != Json::Num) fail(PARSE, "field 'pot_contribution' must be a number");
    cfg.pot = pc.num;
    const Json& bel = field(j, "beliefs");
    if (bel.kind != Json::Arr || bel.arr.size() != 2) fail(PARSE, "beliefs must be an array with one map per player");
    std::vector<Hand> hands[2];
    std::vector<double> weights[2];
    for (int p = 0; p < 2; ++p) {
        const Json& side = bel.arr[size_t(p)];
        if (side.kind != Json::Obj)
            fail(PARSE, "beliefs[" + std::to_string(p) + "] must map hand codes to weights");
        auto items = side.obj;  // nlohmann iterates keys in sorted order
        std::sort(items.begin(), items.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        std::set<int> seen;
        for (const auto& [code, w] : items) {
            if (code.size() != 4)
                fail(PARSE, "beliefs[" + std::to_string(p) + "] key '" + code + "' is not a two-card code");
            Hand h;
            try {
                h = handFromCode(code);
            } catch (const Error& e) {
                fail(PARSE, "beliefs[" + std::to_string(p) + "]: " + e.msg);
            }
            if (w.kind != Json::Num) fail(PARSE, "beliefs[" + std::to_string(p) + "][" + code + "] must be a number");
            if (!seen.insert(h.hi * 52 + h.lo).second)
                fail(PARSE, "beliefs[" + std::to_string(p) + "] repeats hand " + h.code());
            hands[p].push_back(h);
            weights[p].push_back(w.num);
        }
        if (hands[p].empty()) fail(PARSE, "beliefs[" + std::to_string(p) + "] must not be empty");
    }
    const Json& bet = field(j, "betting");
    const Json& ai = field(bet, "all_in");
    if (ai.kind != Json::Bool) fail(PARSE, "betting.all_in must be a boolean");
    cfg.allIn = ai.b;
    const Json& rc = field(bet, "raise_cap");
    if (rc.kind == Json::Num && rc.isInt) cfg.raiseCap = int(rc.num);
    else if (rc.kind != Json::Null) fail(PARSE, "betting.raise_cap must be an integer or null");
    const Json& menus = field(bet, "menus");
    if (menus.kind != Json::Arr || menus.arr.size() != 2) fail(PARSE, "betting.menus must hold one menu set per player");
    for (int p = 0; p < 2; ++p) {
        const Json& m = menus.arr[size_t(p)];
        if (m.kind != Json::Obj) fail(PARSE, "betting.menus entries must be objects");
        for (const auto& [key, v] : m.obj) {
            int c = -1;
            for (int q = 0; q < kContexts; ++q)
                if (key == kContextNames[q]) c = q;
            if (c < 0) fail(PARSE, "betting.menus[" + std::to_string(p) + "] has unknown context '" + key + "'");
            const std::string where = "betting.menus[" + std::to_string(p) + "]." + key;
            if (v.kind != Json::Arr) fail(PARSE, where + " must be an array of fractions");
            for (const Json& x : v.arr) {
                if (x.kind != Json::Num) fail(PARSE, where + " must contain numbers only");
                cfg.menu[p][c].push_back(x.num);
            }
        }
    }
    Instance in;
    try {
        in = makeInstance(board, deck, hands[0], weights[0], hands[1], weights[1], cfg);
    } catch (const Error& e) {
        if (e.code == PARSE) throw;
        if (e.code == DEGENERATE) fail(PARSE, "beliefs are degenerate: no compatible hand pair has positive weight");
        fail(PARSE, e.msg);
    }
    return in;
}

// --------------------------------------------------------------- factors ---
namespace {
// Column-wise builder for CSC matrices whose columns are produced in order.
struct ColBuilder {
    Compressed m;
    ColBuilder(int64_t rows, int64_t cols, bool rowMajor) {
        m.rowMajor = rowMajor;
        m.rows = rows;
        m.cols = cols;
        m.outer.assign(1, 0);
    }
    void push(int64_t inner, double v) {
        if (v != 0.0) {
            m.inner.push_back(int32_t(inner));
            m.val.push_back(v);
        }
    }
    void end() { m.outer.push_back(int64_t(m.val.size())); }
};

// Per-player-1-sequence facts about S and F (rows of the n1 x n2 CSR).
struct SeqFacts {
    std::vector<char> sAct, fAct;
};
SeqFacts seqFacts(const Instance& in) {
    SeqFacts f;
    for (int d = 0; d < in.n(0); ++d) {
        f.sAct.push_back(in.S.outer[size_t(d) + 1] > in.S.outer[size_t(d)]);
        f.fAct.push_back(in.F.outer[size_t(d) + 1] > in.F.outer[size_t(d)]);
    }
    return f;
}

// Y(i, j) = W(i,j) - W(i-1,j) (sparsify.hpp:251-254) as an int.
inline int Ydiff(const Instance& in, int i, int j) {
    return i == 0 ? in.sign(0, j) : in.sign(i, j) - in.sign(i - 1, j);
}

// Ahat = -(Lambda1 Hcross Lambda2) (x) F, rows (i, a), ascending (j, b).
Compressed buildAhatB(const Instance& in) {
    const int m1 = in.m(0), m2 = in.m(1), n1 = in.n(0), n2 = in.n(1);
    ColBuilder b(int64_t(m1) * n1, int64_t(m2) * n2, true);
    std::vector<int> blocked;
    for (int i = 0; i < m1; ++i) {
        blocked.clear();
        for (int j = 0; j < m2; ++j)
            if (!in.compatible(i, j)) blocked.push_back(j);
        for (int a = 0; a < n1; ++a) {
            for (int j : blocked) {
                const double scale = -in.lambda[0][size_t(i)] * in.lambda[1][size_t(j)];
                for (int64_t e = in.F.outer[size_t(a)]; e < in.F.outer[size_t(a) + 1]; ++e)
                    b.push(int64_t(j) * n2 + in.F.inner[size_t(e)], scale * in.F.val[size_t(e)]);
            }
            b.end();
        }
    }
    return b.m;
}

// S^T and F^T as CSR (n2 x n1) for the V builders.
Compressed transposeCsr(const Compressed& A) {
    Compressed t;
    t.rowMajor = true;
    t.rows = A.cols;
    t.cols = A.rows;
    t.outer.assign(size_t(A.cols) + 1, 0);
    for (int32_t c : A.inner) t.outer[size_t(c) + 1]++;
    for (int64_t c = 0; c < A.cols; ++c) t.outer[size_t(c) + 1] += t.outer[size_t(c)];
    std::vector<int64_t> pos(t.outer.begin(), t.outer.end() - 1);
    t.inner.resize(A.inner.size());
    t.val.resize(A.val.size());
    for (int64_t r = 0; r < A.rows; ++r)
        for (int64_t e = A.outer[size_t(r)]; e < A.outer[size_t(r) + 1]; ++e) {
            const int64_t q = pos[size_t(A.inner[size_t(e)])]++;
            t.inner[size_t(q)] = int32_t(r);
            t.val[size_t(q)] = A.val[size_t(e)];
        }
    return t;
}
}  // namespace

void validate(const Factors& s) {  // sparsify.hpp:133-145
    const int64_t k = s.M.rows;
    if (s.M.cols != k) fail(CONTRACT, "M is not square");
    if (s.U.rows != s.Ahat.rows || s.U.cols != k) fail(CONTRACT, "U dimensions do not match Ahat/M");
    if (s.V.rows != s.Ahat.cols || s.V.cols != k) fail(CONTRACT, "V dimensions do not match Ahat/M");
    for (int64_t j = 0; j < k; ++j) {
        const int64_t e = s.M.outer[size_t(j)];
        if (e == s.M.outer[size_t(j) + 1] || s.M.inner[size_t(e)] != j || s.M.val[size_t(e)] != 1.0)
            fail(CONTRACT, "M is not unit lower triangular at column " + std::to_string(j));
    }
}

Factors techniqueB(const Instance& in) {  // sparsify.hpp:246-312
    const int m1 = in.m(0), m2 = in.m(1), n1 = in.n(0), n2 = in.n(1);
    const int64_t rows = int64_t(m1) * n1, cols = int64_t(m2) * n2, k = rows + n1;
    Factors s;
    s.technique = 1;
    s.n1 = n1;
    s.n2 = n2;
    s.Ahat = buildAhatB(in);
    {  // U: [Lambda1 (x) I | lambda1 (x) I]
        ColBuilder b(rows, k, true);
        for (int i = 0; i < m1; ++i)
            for (int d = 0; d < n1; ++d) {
                const double v = in.lambda[0][size_t(i)];
                if (v != 0.0) {
                    b.push(int64_t(i) * n1 + d, v);
                    b.push(int64_t(m1) * n1 + d, v);
                }
                b.end();
            }
        s.U = b.m;
    }
    {  // M = blockdiag(D (x) I, I), D = unit lower bidiagonal with -1
        ColBuilder b(k, k, false);
        for (int64_t j = 0; j < k; ++j) {
            b.push(j, 1.0);
            if (j < int64_t(m1 - 1) * n1) b.push(j + n1, -1.0);
            b.end();
        }
        s.M = b.m;
    }
    {  // V = [(Lambda2 Y^T) (x) S^T | lambda2 (x) F^T], CSC
        const Compressed St = transposeCsr(in.S), Ft = transposeCsr(in.F);
        (void)St;
        (void)Ft;
        ColBuilder b(cols, k, false);
        for (int i = 0; i < m1; ++i)
            for (int d = 0; d < n1; ++d) {
                for (int j = 0; j < m2; ++j) {
                    const double scale = in.lambda[1][size_t(j)] * double(Ydiff(in, i, j));
                    if (scale == 0.0) continue;
                    for (int64_t e = in.S.outer[size_t(d)]; e < in.S.outer[size_t(d) + 1]; ++e)
                        b.push(int64_t(j) * n2 + in.S.inner[size_t(e)], scale * in.S.val[size_t(e)]);
                }
                b.end();
            }
        for (int d = 0; d < n1; ++d) {
            for (int j = 0; j < m2; ++j) {
                const double scale = in.lambda[1][size_t(j)];
                if (scale == 0.0) continue;
                for (int64_t e = in.F.outer[size_t(d)]; e < in.F.outer[size_t(d) + 1]; ++e)
                    b.push(int64_t(j) * n2 + in.F.inner[size_t(e)], scale * in.F.val[size_t(e)]);
            }
            b.end();
        }
        s.V = b.m;
    }
    validate(s);
    return s;
}

// postprocess(techniqueB(in)) in closed form.  With M's -1 sub-diagonal the
// elimination of zero V columns (sparsify.hpp:337-374) acts per showdown
// sequence d as follows: hand i keeps column (i, d) iff d has a showdown and
// the strength-difference row Y(i, .) carries mass; a dropped column's U entry
// folds into the last kept column at or above it in the same chain (the
// value copies exactly: 0 + -(-1) * lambda1), dropped columns above the first
// kept one vanish, and M links consecutive kept columns with -1.
Factors techniqueBPost(const Instance& in) {
    const int m1 = in.m(0), m2 = in.m(1), n1 = in.n(0), n2 = in.n(1);
    const int64_t rows = int64_t(m1) * n1, cols = int64_t(m2) * n2;
    const SeqFacts sf = seqFacts(in);
    // rowAlive(i): some j with lambda2(j) * Y(i,j) != 0
    std::vector<char> rowAlive(static_cast<size_t>(m1), 0);
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2 && !rowAlive[size_t(i)]; ++j)
            if (in.lambda[1][size_t(j)] * double(Ydiff(in, i, j)) != 0.0) rowAlive[size_t(i)] = 1;
    bool anyL2 = false;
    for (double l : in.lambda[1]) anyL2 |= l != 0.0;
    // new column numbering in original order (i-major, then the F block)
    std::vector<int64_t> colOf(static_cast<size_t>(rows), -1), fcol(size_t(n1), -1);
    int64_t k = 0;
    for (int i = 0; i < m1; ++i)
        for (int d = 0; d < n1; ++d)
            if (sf.sAct[size_t(d)] && rowAlive[size_t(i)]) colOf[size_t(i) * n1 + d] = k++;
    for (int d = 0; d < n1; ++d)
        if (sf.fAct[size_t(d)] && anyL2) fcol[size_t(d)] = k++;
    Factors s;
    s.technique = 1;
    s.postprocessed = true;
    s.n1 = n1;
    s.n2 = n2;
    s.Ahat = buildAhatB(in);
    {  // U rows (i, d): last kept column of chain d at or above i, then F col
        ColBuilder b(rows, k, true);
        std::vector<int64_t> lastKept(static_cast<size_t>(n1), -1);
        for (int i = 0; i < m1; ++i)
            for (int d = 0; d < n1; ++d) {
                const int64_t c = colOf[size_t(i) * n1 + d];
                if (c >= 0) lastKept[size_t(d)] = c;
                const double v = in.lambda[0][size_t(i)];
                if (v != 0.0) {
                    if (lastKept[size_t(d)] >= 0) b.push(lastKept[size_t(d)], v);
                    if (fcol[size_t(d)] >= 0) b.push(fcol[size_t(d)], v);
                }
                b.end();
            }
        s.U = b.m;
    }
    {  // M: CSC, column c has its diagonal and a -1 at the next kept column
        std::vector<int64_t> nextKept(static_cast<size_t>(k), -1);
        std::vector<int64_t> prev(static_cast<size_t>(n1), -1);
        for (int i = 0; i < m1; ++i)
            for (int d = 0; d < n1; ++d) {
                const int64_t c = colOf[size_t(i) * n1 + d];
                if (c < 0) continue;
                if (prev[size_t(d)] >= 0) nextKept[size_t(prev[size_t(d)])] = c;
                prev[size_t(d)] = c;
            }
        ColBuilder b(k, k, false);
        for (int64_t c = 0; c < k; ++c) {
            b.push(c, 1.0);
            if (nextKept[size_t(c)] >= 0) b.push(nextKept[size_t(c)], -1.0);
            b.end();
        }
        s.M = b.m;
    }
    {  // V: the kept columns of techniqueB's V, unchanged
        ColBuilder b(cols, k, false);
        for (int i = 0; i < m1; ++i)
            for (int d = 0; d < n1; ++d) {
                if (colOf[size_t(i) * n1 + d] < 0) continue;
                for (int j = 0; j < m2; ++j) {
                    const double scale = in.lambda[1][size_t(j)] * double(Ydiff(in, i, j));
                    if (scale == 0.0) continue;
                    for (int64_t e = in.S.outer[size_t(d)]; e < in.S.outer[size_t(d) + 1]; ++e)
                        b.push(int64_t(j) * n2 + in.S.inner[size_t(e)], scale * in.S.val[size_t(e)]);
                }
                b.end();
            }
        for (int d = 0; d < n1; ++d) {
            if (fcol[size_t(d)] < 0) continue;
            for (int j = 0; j < m2; ++j) {
                const double scale = in.lambda[1][size_t(j)];
                if (scale == 0.0) continue;
                for (int64_t e = in.F.outer[size_t(d)]; e < in.F.outer[size_t(d) + 1]; ++e)
                    b.push(int64_t(j) * n2 + in.F.inner[size_t(e)], scale * in.F.val[size_t(e)]);
            }
            b.end();
        }
        s.V = b.m;
    }
    validate(s);
    return s;
}

namespace {
struct Rect {
    int gain = 0, value = 0, r0 = 0, r1 = 0, c0 = 0, c1 = 0;
};
// Largest gain (area - height - width) rectangle of cells equal to v, by the
// histogram sweep of sparsify.hpp:34-60 (first strictly better wins).
Rect bestRect(const std::vector<int8_t>& R, int rows, int cols, int v) {
    Rect best;
    std::vector<int> hgt(static_cast<size_t>(cols), 0), stk;
    for (int i = 0; i < rows; ++i) {
        const int8_t* row = R.data() + size_t(i) * cols;
        for (int j = 0; j < cols; ++j) hgt[size_t(j)] = row[j] == v ? hgt[size_t(j)] + 1 : 0;
        stk.clear();
        for (int j = 0; j <= cols; ++j) {
            const int h = j < cols ? hgt[size_t(j)] : 0;
            while (!stk.empty() && hgt[size_t(stk.back())] >= h) {
                const int top = stk.back();
                stk.pop_back();
                const int hh = hgt[size_t(top)];
                const int left = stk.empty() ? 0 : stk.back() + 1;
                const int width = j - left;
                const int gain = hh * width - (hh + width);
                if (gain > best.gain) best = {gain, v, i - hh + 1, i, left, j - 1};
            }
            if (j < cols) stk.push_back(j);
        }
    }
    return best;
}
}  // namespace

Factors techniqueA(const Instance& in, int peelIters) {  // sparsify.hpp:68-103, 165-240
    const int m1 = in.m(0), m2 = in.m(1), n1 = in.n(0), n2 = in.n(1);
    std::vector<int8_t> R(static_cast<size_t>(m1) * m2);
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j) R[size_t(i) * m2 + j] = int8_t(in.sign(i, j));
    std::vector<Rect> rects;
    for (int it = 0; it < peelIters; ++it) {
        const Rect p = bestRect(R, m1, m2, 1), q = bestRect(R, m1, m2, -1);
        const Rect b = p.gain >= q.gain ? p : q;
        if (b.gain <= 0) break;
        for (int i = b.r0; i <= b.r1; ++i)
            for (int j = b.c0; j <= b.c1; ++j) R[size_t(i) * m2 + j] = 0;
        rects.push_back(b);
    }
    const int r = int(rects.size());
    const int64_t rows = int64_t(m1) * n1, cols = int64_t(m2) * n2, k = int64_t(r) * n1 + n1;
    Factors s;
    s.technique = 0;
    s.n1 = n1;
    s.n2 = n2;
    {  // Ahat: residual What (x) S plus blocked pairs (x) F
        ColBuilder b(rows, cols, true);
        for (int i = 0; i < m1; ++i)
            for (int a = 0; a < n1; ++a) {
                for (int j = 0; j < m2; ++j) {
                    const int w = R[size_t(i) * m2 + j];
                    if (w != 0) {
                        const double scale = in.lambda[0][size_t(i)] * in.lambda[1][size_t(j)] * double(w);
                        for (int64_t e = in.S.outer[size_t(a)]; e < in.S.outer[size_t(a) + 1]; ++e)
                            b.push(int64_t(j) * n2 + in.S.inner[size_t(e)], scale * in.S.val[size_t(e)]);
                    } else if (!in.compatible(i, j)) {
                        const double scale = -in.lambda[0][size_t(i)] * in.lambda[1][size_t(j)];
                        for (int64_t e = in.F.outer[size_t(a)]; e < in.F.outer[size_t(a) + 1]; ++e)
                            b.push(int64_t(j) * n2 + in.F.inner[size_t(e)], scale * in.F.val[size_t(e)]);
                    }
                }
                b.end();
            }
        s.Ahat = b.m;
    }
    {  // U rows (i, d): rectangle q containing i -> lambda1(i) * value, then last block
        std::vector<std::vector<int>> rowRects(static_cast<size_t>(m1));
        for (int q = 0; q < r; ++q)
            for (int i = rects[size_t(q)].r0; i <= rects[size_t(q)].r1; ++i) rowRects[size_t(i)].push_back(q);
        ColBuilder b(rows, k, true);
        for (int i = 0; i < m1; ++i)
            for (int d = 0; d < n1; ++d) {
                for (int q : rowRects[size_t(i)]) {
                    const double v = in.lambda[0][size_t(i)] * double(rects[size_t(q)].value);
                    if (v != 0.0) b.push(int64_t(q) * n1 + d, v);
                }
                if (in.lambda[0][size_t(i)] != 0.0) b.push(int64_t(r) * n1 + d, in.lambda[0][size_t(i)]);
                b.end();
            }
        s.U = b.m;
    }
    {
        ColBuilder b(k, k, false);
        for (int64_t j = 0; j < k; ++j) {
            b.push(j, 1.0);
            b.end();
        }
        s.M = b.m;
    }
    {  // V columns (q, d): lambda2(j) (x) S row d over the rectangle's columns
        ColBuilder b(cols, k, false);
        for (int q = 0; q < r; ++q)
            for (int d = 0; d < n1; ++d) {
                for (int j = rects[size_t(q)].c0; j <= rects[size_t(q)].c1; ++j) {
                    const double scale = in.lambda[1][size_t(j)] * 1.0;
                    if (scale == 0.0) continue;
                    for (int64_t e = in.S.outer[size_t(d)]; e < in.S.outer[size_t(d) + 1]; ++e)
                        b.push(int64_t(j) * n2 + in.S.inner[size_t(e)], scale * in.S.val[size_t(e)]);
                }
                b.end();
            }
        for (int d = 0; d < n1; ++d) {
            for (int j = 0; j < m2; ++j) {
                const double scale = in.lambda[1][size_t(j)];
                if (scale == 0.0) continue;
                for (int64_t e = in.F.outer[size_t(d)]; e < in.F.outer[size_t(d) + 1]; ++e)
                    b.push(int64_t(j) * n2 + in.F.inner[size_t(e)], scale * in.F.val[size_t(e)]);
            }
            b.end();
        }
        s.V = b.m;
    }
    validate(s);
    return s;
}

// postprocess (sparsify.hpp:318-406) for any factor set: eliminate every k
// coordinate whose V column is empty, folding its U column into the
// coordinates it depends on and rewriting later M rows.  Ordered maps keep
// the reference's exact accumulation order.
Factors postprocess(const Factors& s) {
    validate(s);
    const int64_t k = s.k();
    std::vector<std::map<int64_t, double>> ucol(static_cast<size_t>(k)), mrow(static_cast<size_t>(k));
    std::vector<std::set<int64_t>> users(static_cast<size_t>(k));
    for (int64_t r = 0; r < s.U.rows; ++r)
        for (int64_t e = s.U.outer[size_t(r)]; e < s.U.outer[size_t(r) + 1]; ++e)
            ucol[size_t(s.U.inner[size_t(e)])][r] = s.U.val[size_t(e)];
    for (int64_t j = 0; j < k; ++j)
        for (int64_t e = s.M.outer[size_t(j)]; e < s.M.outer[size_t(j) + 1]; ++e) {
            const int64_t r = s.M.inner[size_t(e)];
            if (r == j) continue;
            mrow[size_t(r)][j] = s.M.val[size_t(e)];
            users[size_t(j)].insert(r);
        }
    std::vector<char> keep(static_cast<size_t>(k), 1);
    for (int64_t j = 0; j < k; ++j) {
        if (s.V.outer[size_t(j)] != s.V.outer[size_t(j) + 1]) continue;
        const std::map<int64_t, double> deps = mrow[size_t(j)];
        const std::map<int64_t, double> uj = std::move(ucol[size_t(j)]);
        for (const auto& [i, a] : deps) {
            auto& ui = ucol[size_t(i)];
            for (const auto& [row, v] : uj) {
                double& slot = ui[row];
                slot += -a * v;
                if (slot == 0.0) ui.erase(row);
            }
        }
        const std::set<int64_t> refs = users[size_t(j)];
        for (int64_t r : refs) {
            auto& row = mrow[size_t(r)];
            const auto it = row.find(j);
            const double b = it->second;
            row.erase(it);
            for (const auto& [i, a] : deps) {
                double& slot = row[i];
                const bool fresh = slot == 0.0;
                slot -= b * a;
                if (slot == 0.0) row.erase(i);
                else if (fresh) users[size_t(i)].insert(r);
            }
        }
        for (const auto& [i, a] : deps) {
            (void)a;
            users[size_t(i)].erase(j);
        }
        ucol[size_t(j)].clear();
        mrow[size_t(j)].clear();
        users[size_t(j)].clear();
        keep[size_t(j)] = 0;
    }
    std::vector<int64_t> remap(static_cast<size_t>(k), -1);
    int64_t kept = 0;
    for (int64_t j = 0; j < k; ++j)
        if (keep[size_t(j)]) remap[size_t(j)] = kept++;
    Factors out;
    out.Ahat = s.Ahat;
    out.technique = s.technique;
    out.postprocessed = true;
    out.n1 = s.n1;
    out.n2 = s.n2;
    std::vector<std::tuple<int64_t, int64_t, double>> ut, mt;
    ColBuilder vb(s.V.rows, kept, false);
    for (int64_t j = 0; j < k; ++j) {
        if (!keep[size_t(j)]) continue;
        const int64_t nj = remap[size_t(j)];
        for (const auto& [row, v] : ucol[size_t(j)])
            if (v != 0.0) ut.emplace_back(row, nj, v);
        mt.emplace_back(nj, nj, 1.0);
        for (const auto& [i, a] : mrow[size_t(j)]) mt.emplace_back(nj, remap[size_t(i)], a);
        for (int64_t e = s.V.outer[size_t(j)]; e < s.V.outer[size_t(j) + 1]; ++e)
            vb.push(s.V.inner[size_t(e)], s.V.val[size_t(e)]);
        vb.end();
    }
    out.U = compress(s.U.rows, kept, true, ut);
    out.M = compress(kept, kept, false, mt);
    out.V = vb.m;
    validate(out);
    const int64_t before = s.Ahat.nnz() + s.U.nnz() + s.M.nnz() + s.V.nnz();
    const int64_t after = out.Ahat.nnz() + out.U.nnz() + out.M.nnz() + out.V.nnz();
    if (after > before) fail(CONTRACT, "postprocessing increased the stored size");
    return out;
}

// --------------------------------------------------------------- bundles ---
namespace {
void writeMtx(const std::string& path, const Compressed& m) {  // matrix_market.hpp:15-30
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) fail(IO, "cannot open '" + path + "' for writing");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%lld %lld %lld\n", (long long)m.rows, (long long)m.cols, (long long)m.nnz());
    for (int64_t o = 0; o < m.outerSize(); ++o)
        for (int64_t e = m.outer[size_t(o)]; e < m.outer[size_t(o) + 1]; ++e) {
            const long long r = m.rowMajor ? o : m.inner[size_t(e)], c = m.rowMajor ? m.inner[size_t(e)] : o;
            std::fprintf(f, "%lld %lld %.17g\n", r + 1, c + 1, m.val[size_t(e)]);
        }
    if (std::fclose(f) != 0) fail(IO, "write failed for '" + path + "'");
}

Compressed readMtx(const std::string& path, bool rowMajor) {  // matrix_market.hpp:33-71
    std::ifstream in(path);
    if (!in) fail(IO, "cannot open '" + path + "'");
    std::string line;
    if (!std::getline(in, line)) fail(PARSE, path + ": empty file");
    if (line.rfind("%%MatrixMarket", 0) != 0) fail(PARSE, path + ": missing MatrixMarket banner");
    {
        std::istringstream hs(line);
        std::string tag, object, format, field, sym;
        hs >> tag >> object >> format >> field >> sym;
        if (object != "matrix" || format != "coordinate" || field != "real" || sym != "general")
            fail(PARSE, path + ": unsupported MatrixMarket flavor '" + line + "'");
    }
    while (std::getline(in, line))
        if (!line.empty() && line[0] != '%') break;
    long long rows = 0, cols = 0, nnz = 0;
    {
        std::istringstream hs(line);
        if (!(hs >> rows >> cols >> nnz) || rows < 0 || cols < 0 || nnz < 0)
            fail(PARSE, path + ": bad size line '" + line + "'");
    }
    std::vector<std::tuple<int64_t, int64_t, double>> t;
    t.reserve(size_t(nnz));
    for (long long q = 0; q < nnz; ++q) {
        long long i = 0, j = 0;
        double v = 0;
        if (!(in >> i >> j >> v)) fail(PARSE, path + ": truncated after " + std::to_string(q) + " entries");
        if (i < 1 || i > rows || j < 1 || j > cols)
            fail(PARSE, path + ": entry (" + std::to_string(i) + "," + std::to_string(j) + ") outside " +
                            std::to_string(rows) + "x" + std::to_string(cols));
        t.emplace_back(i - 1, j - 1, v);
    }
    return compress(rows, cols, rowMajor, std::move(t));
}

// Tiny key scanner for the flat header.json written below.
std::string headerValue(const std::string& text, const std::string& key) {
    const std::string pat = "\"" + key + "\"";
    const size_t p = text.find(pat);
    if (p == std::string::npos) return "";
    size_t q = text.find(':', p + pat.size());
    if (q == std::string::npos) return "";
    ++q;
    while (q < text.size() && std::isspace(static_cast<unsigned char>(text[q]))) ++q;
    size_t e = q;
    if (e < text.size() && text[e] == '"') {
        const size_t c = text.find('"', e + 1);
        return text.substr(e, c - e + 1);
    }
    while (e < text.size() && text[e] != ',' && text[e] != '\n' && text[e] != '}') ++e;
    std::string v = text.substr(q, e - q);
    while (!v.empty() && std::isspace(static_cast<unsigned char>(v.back()))) v.pop_back();
    return v;
}
}  // namespace

void writeBundle(const Factors& s, const std::string& dir) {  // bundle_io.hpp:27-53
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    if (ec) fail(IO, "cannot create '" + dir + "': " + ec.message());
    const std::filesystem::path base(dir);
    {
        std::FILE* f = std::fopen((base / "header.json").string().c_str(), "w");
        if (!f) fail(IO, "cannot open '" + (base / "header.json").string() + "' for writing");
        std::fprintf(f,
                     "{\n  \"cols\": %lld,\n  \"k\": %lld,\n  \"nonzeros\": {\n    \"ahat\": %lld,\n    \"m\": %lld,\n"
                     "    \"u\": %lld,\n    \"v\": %lld\n  },\n  \"postprocessed\": %s,\n  \"rows\": %lld,\n"
                     "  \"schema_version\": 1,\n  \"technique\": \"%s\"\n}\n",
                     (long long)s.cols(), (long long)s.k(), (long long)s.Ahat.nnz(), (long long)s.M.nnz(),
                     (long long)s.U.nnz(), (long long)s.V.nnz(), s.postprocessed ? "true" : "false",
                     (long long)s.rows(), s.technique == 0 ? "a" : "b");
        std::fclose(f);
    }
    writeMtx((base / "ahat.mtx").string(), s.Ahat);
    writeMtx((base / "u.mtx").string(), s.U);
    writeMtx((base / "m.mtx").string(), s.M);
    writeMtx((base / "v.mtx").string(), s.V);
}

Factors readBundle(const std::string& dir) {  // bundle_io.hpp:57-94
    const std::filesystem::path base(dir);
    std::ifstream in(base / "header.json");
    if (!in) fail(IO, "cannot open '" + (base / "header.json").string() + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string h = ss.str();
    if (headerValue(h, "schema_version").empty()) fail(PARSE, "bundle header missing schema_version");
    if (headerValue(h, "schema_version") != "1") fail(PARSE, "unsupported bundle schema_version " + headerValue(h, "schema_version"));
    for (const char* key : {"technique", "postprocessed", "rows", "cols", "k"})
        if (headerValue(h, key).empty()) fail(PARSE, std::string("bundle header missing '") + key + "'");
    Factors s;
    const std::string tech = headerValue(h, "technique");
    if (tech == "\"a\"" || tech == "\"A\"") s.technique = 0;
    else if (tech == "\"b\"" || tech == "\"B\"") s.technique = 1;
    else fail(PARSE, "unknown technique '" + tech + "', expected 'a' or 'b'");
    s.postprocessed = headerValue(h, "postprocessed") == "true";
    s.Ahat = readMtx((base / "ahat.mtx").string(), true);
    s.U = readMtx((base / "u.mtx").string(), true);
    s.M = readMtx((base / "m.mtx").string(), false);
    s.V = readMtx((base / "v.mtx").string(), false);
    if (s.rows() != std::atoll(headerValue(h, "rows").c_str()) || s.cols() != std::atoll(headerValue(h, "cols").c_str()) ||
        s.k() != std::atoll(headerValue(h, "k").c_str()))
        fail(PARSE, "bundle factors disagree with header dimensions");
    try {
        validate(s);
    } catch (const Error& e) {
        fail(PARSE, "bundle factors are inconsistent: " + e.msg);
    }
    return s;
}

}  // namespace krh

// ==================================================================== C ABI
struct krh_instance {
    krh::Instance in;
    std::vector<uint8_t> cards[2] = {};  // card ids per hand, filled by krh_instance_kron_view
};
struct krh_factors {
    krh::Factors f;
};

namespace {
thread_local int g_code = 0;
thread_local std::string g_msg;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const krh::Error& e) {
        g_code = e.code;
        g_msg = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_code = 7;
        g_msg = e.what();
        return 7;
    }
}
}  // namespace

extern "C" {

const char* krh_last_error(int* code) {
    if (code) *code = g_code;
    return g_msg.c_str();
}

int krh_instance_from_json(const char* path, krh_instance** out) {
    return guard([&] { *out = new krh_instance{krh::readInstanceJson(path)}; });
}

int krh_instance_builtin(const char* name, uint64_t seed, int hands, int shared, const char* board, int deck, int tree,
                         krh_instance** out) {
    return guard([&] {
        const std::string n(name);
        krh::Instance in;
        if (n == "golden") in = krh::goldenInstance();
        else if (n == "twenty_card") in = krh::twentyCardInstance();
        else if (n == "bluffing") in = krh::bluffingInstance();
        else if (n == "all_tie") in = krh::allTieInstance();
        else if (n == "random_small") {
            std::mt19937_64 rng(seed);
            for (int q = 0; q < shared; ++q) (void)krh::randomSmallInstance(rng, hands);
            in = krh::randomSmallInstance(rng, hands);
        } else if (n == "bench") in = krh::benchInstance(seed, hands, shared);
        else if (n == "river_full") {
            krh::BettingConfig cfg = krh::referenceBettingConfig();
            if (tree == 3) cfg = krh::threeBetConfig();
            if (tree == 91) {  // menus {0.33, 0.75, 1.5}, raise cap 3 -> n = 91
                cfg = krh::threeBetConfig();
                for (int p = 0; p < 2; ++p)
                    for (auto& m : cfg.menu[p]) m = {0.33, 0.75, 1.5};
            }
            in = krh::fullRangeRiver(board, deck, seed, cfg);
        }
        else throw krh::Error{krh::INVALID_INPUT, "unknown built-in instance '" + n + "'"};
        *out = new krh_instance{std::move(in)};
    });
}

void krh_instance_free(krh_instance* h) { delete h; }

int krh_instance_custom(const int32_t board[5], int deck, const uint8_t* cards1, const double* w1, int m1,
                        const uint8_t* cards2, const double* w2, int m2, double stack, double pot,
                        const double* menu, int nmenu, int all_in, int raise_cap, krh_instance** out) {
    return guard([&] {
        if (!board || !out || m1 < 0 || m2 < 0 || nmenu < 0 || (nmenu && !menu))
            throw krh::Error{krh::INVALID_INPUT, "bad arguments to krh_instance_custom"};
        std::vector<int> dk;
        if (deck == 26) {
            for (int r = 0; r < 13; ++r)
                for (int q = 0; q < 2; ++q) dk.push_back(r * 4 + q);
        } else if (deck == 52) {
            dk = krh::standardDeck();
        } else {
            throw krh::Error{krh::INVALID_INPUT, "deck must be 52 or 26"};
        }
        std::array<int, 5> bd{};
        for (int i = 0; i < 5; ++i) {
            if (board[i] < 0 || board[i] >= 52) throw krh::Error{krh::INVALID_INPUT, "board card out of range"};
            bd[size_t(i)] = board[i];
        }
        auto hands = [](const uint8_t* c, int m) {
            std::vector<krh::Hand> h;
            for (int i = 0; i < m; ++i) {
                if (c[2 * i] >= 52 || c[2 * i + 1] >= 52 || c[2 * i] == c[2 * i + 1])
                    throw krh::Error{krh::INVALID_INPUT, "bad hand cards"};
                h.push_back(krh::Hand::of(c[2 * i], c[2 * i + 1]));
            }
            return h;
        };
        krh::BettingConfig cfg;
        cfg.stack1 = cfg.stack2 = stack;
        cfg.pot = pot;
        for (int p = 0; p < 2; ++p)
            for (auto& m : cfg.menu[p]) m.assign(menu, menu + nmenu);
        cfg.allIn = all_in != 0;
        if (raise_cap >= 0) cfg.raiseCap = raise_cap;
        *out = new krh_instance{krh::makeInstance(bd, dk, hands(cards1, m1), std::vector<double>(w1, w1 + m1),
                                                  hands(cards2, m2), std::vector<double>(w2, w2 + m2), cfg)};
    });
}

int krh_instance_dims(const krh_instance* h, int64_t out[16]) {
    return guard([&] {
        const auto& in = h->in;
        int folds = 0;
        for (const auto& t : in.sk.terminals) folds += t.fold;
        int64_t acts[2] = {0, 0};
        for (int p = 0; p < 2; ++p)
            for (int id : in.sk.playerNodes[p]) acts[p] += int64_t(in.sk.nodes[size_t(id)].actions.size());
        const int64_t v[16] = {in.m(0), in.m(1), in.n(0), in.n(1), in.rows(), in.cols(), int64_t(in.sk.nodes.size()),
                               int64_t(in.sk.playerNodes[0].size()), int64_t(in.sk.playerNodes[1].size()),
                               int64_t(in.sk.terminals.size()), folds, int64_t(in.sk.terminals.size()) - folds,
                               in.F.nnz(), in.S.nnz(), acts[0], acts[1]};
        std::memcpy(out, v, sizeof v);
    });
}

double krh_instance_beta(const krh_instance* h) { return h->in.beta; }
double krh_instance_pot(const krh_instance* h) { return 2 * h->in.config.pot; }

int krh_instance_hands(const krh_instance* h, int player, char* out) {
    return guard([&] {
        const auto& hs = h->in.hands[player == 0 ? 0 : 1];
        for (size_t i = 0; i < hs.size(); ++i) std::memcpy(out + 4 * i, hs[i].code().data(), 4);
    });
}

int krh_instance_vectors(const krh_instance* h, double* mu1, double* mu2, double* lam1, double* lam2) {
    return guard([&] {
        const auto& in = h->in;
        std::memcpy(mu1, in.mu[0].data(), 8 * in.mu[0].size());
        std::memcpy(mu2, in.mu[1].data(), 8 * in.mu[1].size());
        std::memcpy(lam1, in.lambda[0].data(), 8 * in.lambda[0].size());
        std::memcpy(lam2, in.lambda[1].data(), 8 * in.lambda[1].size());
    });
}

int krh_instance_treeplex(const krh_instance* h, int player, int32_t* parent, int32_t* aptr, int32_t* aseq) {
    return guard([&] {
        const auto& sk = h->in.sk;
        const int p = player == 0 ? 0 : 1;
        int a = 0, v = 0;
        aptr[0] = 0;
        for (int id : sk.playerNodes[p]) {
            const auto& nd = sk.nodes[size_t(id)];
            parent[v] = nd.parentSeq[p];
            for (const auto& act : nd.actions) aseq[a++] = act.seq;
            aptr[++v] = a;
        }
    });
}

int64_t krh_dense_nnz(const krh_instance* h) { return krh::densePayoffNonzeros(h->in); }

int krh_instance_kron_view(const krh_instance* h, kr_kron_board* out) {
    return guard([&] {
        const auto& in = h->in;
        auto& cards = const_cast<krh_instance*>(h)->cards;
        for (int p = 0; p < 2; ++p) {
            cards[p].clear();
            for (const auto& hd : in.hands[p]) {
                cards[p].push_back(hd.hi);
                cards[p].push_back(hd.lo);
            }
        }
        auto view = [](const krh::Compressed& m) {
            return kr_compressed{m.outerSize(), m.outer.data(), m.inner.data(), m.val.data()};
        };
        out->m1 = in.m(0);
        out->m2 = in.m(1);
        out->n1 = in.n(0);
        out->n2 = in.n(1);
        out->key1 = in.key[0].data();
        out->key2 = in.key[1].data();
        out->cards1 = cards[0].data();
        out->cards2 = cards[1].data();
        out->lambda1 = in.lambda[0].data();
        out->lambda2 = in.lambda[1].data();
        out->F = view(in.F);
        out->S = view(in.S);
    });
}

int krh_sparsify(const krh_instance* h, int technique, int post, int peel_iters, krh_factors** out) {
    return guard([&] {
        krh::Factors f;
        if (technique == 0) {
            f = krh::techniqueA(h->in, peel_iters);
            if (post) f = krh::postprocess(f);
        } else {
            f = post ? krh::techniqueBPost(h->in) : krh::techniqueB(h->in);
        }
        *out = new krh_factors{std::move(f)};
    });
}

int krh_postprocess(const krh_factors* f, krh_factors** out) {
    return guard([&] { *out = new krh_factors{krh::postprocess(f->f)}; });
}

int krh_factors_from_arrays(const kr_factors* kf, int technique, int postprocessed, krh_factors** out) {
    return guard([&] {
        auto grab = [](const kr_compressed& c, bool rowMajor, int64_t rows, int64_t cols) {
            krh::Compressed m;
            m.rowMajor = rowMajor;
            m.rows = rows;
            m.cols = cols;
            m.outer.assign(c.outer, c.outer + c.outer_size + 1);
            const int64_t nnz = c.outer[c.outer_size];
            m.inner.assign(c.inner, c.inner + nnz);
            m.val.assign(c.val, c.val + nnz);
            return m;
        };
        krh::Factors f;
        f.Ahat = grab(kf->ahat, true, kf->rows, kf->cols);
        f.U = grab(kf->u, true, kf->rows, kf->k);
        f.M = grab(kf->m, false, kf->k, kf->k);
        f.V = grab(kf->v, false, kf->cols, kf->k);
        f.technique = technique;
        f.postprocessed = postprocessed != 0;
        f.n1 = kf->n1;
        f.n2 = kf->n2;
        *out = new krh_factors{std::move(f)};
    });
}

void krh_factors_free(krh_factors* f) { delete f; }

int krh_factors_dims(const krh_factors* h, int64_t out[9]) {
    return guard([&] {
        const auto& f = h->f;
        const int64_t v[9] = {f.rows(), f.cols(), f.k(), f.Ahat.nnz(), f.U.nnz(), f.M.nnz(), f.V.nnz(),
                              f.technique, f.postprocessed ? 1 : 0};
        std::memcpy(out, v, sizeof v);
    });
}

int krh_factors_view(const krh_factors* h, kr_factors* out) {
    return guard([&] {
        const auto& f = h->f;
        auto view = [](const krh::Compressed& m) {
            return kr_compressed{m.outerSize(), m.outer.data(), m.inner.data(), m.val.data()};
        };
        out->rows = f.rows();
        out->cols = f.cols();
        out->k = f.k();
        out->ahat = view(f.Ahat);
        out->u = view(f.U);
        out->m = view(f.M);
        out->v = view(f.V);
        out->n1 = f.n1;
        out->n2 = f.n2;
    });
}

int krh_factors_validate(const krh_factors* f) {
    return guard([&] { krh::validate(f->f); });
}

int krh_bundle_write(const krh_factors* f, const char* dir) {
    return guard([&] { krh::writeBundle(f->f, dir); });
}

int krh_bundle_read(const char* dir, krh_factors** out) {
    return guard([&] { *out = new krh_factors{krh::readBundle(dir)}; });
}

}  // extern "C"
