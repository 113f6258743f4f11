// kr_oracle.hpp — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// A plain C++20 restatement of the reference `kronriver` library's algorithm
// for the gradient-oracle hot path (arXiv 2112.03804): cards -> betting
// skeleton -> Kronecker payoff -> Technique A/B sparsification (+postprocess)
// -> factored matvec -> DCFR solver / best response.  Every function cites the
// reference file:line it follows (paths relative to /root/reference/proj).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this code, and only as the checker.  The product path
// (paper_2112_03804_b200/) never includes or links it.
//
// The reference cannot be compiled here (Eigen3, Catch2 and CLI11 are absent),
// so this restatement replaces Eigen's storage with an explicit sorted
// compressed format that mirrors `makeSparse` (linalg.hpp:18-25):
// setFromTriplets (duplicates summed in triplet order, inner indices sorted
// ascending), prune(0,0) (exact zeros dropped), makeCompressed.
//
// Parity is PINNED by the reference's published golden numbers
// (README.md:75-82): twenty_card B-post factor counts
// ahat=28350 u=2205 m=1649 v=23556 k=835, dense nnz 152916, and the
// 600-iteration solve from the B bundle: exploitability 0.000189332132512,
// gradient_flops 67228200 — see tests/test_oracle_golden.py.
//
// Build flags mirror the reference Release build (CMakeLists.txt:6-8,20):
// -O3 with no -march (x86-64 baseline, hence no FMA), plus
// -ffp-contract=off to forbid contraction explicitly.
#pragma once

#include <algorithm>
#include <array>
#include <cassert>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <numeric>
#include <optional>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace kro {

// ---------------------------------------------------------------- errors ---
// errors.hpp:11-58 — stable codes.
struct Error : std::runtime_error {
    std::string code;
    Error(std::string c, const std::string& m) : std::runtime_error(m), code(std::move(c)) {}
};
struct InvalidInputError : Error { explicit InvalidInputError(const std::string& m) : Error("INVALID_INPUT", m) {} };
struct ParseError : Error { explicit ParseError(const std::string& m) : Error("PARSE", m) {} };
struct GuardError : Error { explicit GuardError(const std::string& m) : Error("GUARD_EXCEEDED", m) {} };
struct DegenerateBeliefsError : Error { explicit DegenerateBeliefsError(const std::string& m) : Error("DEGENERATE_BELIEFS", m) {} };
struct ContractError : Error { explicit ContractError(const std::string& m) : Error("CONTRACT", m) {} };

using Vec = std::vector<double>;

// ------------------------------------------------------------- sparse -----
// Compressed sparse storage standing in for Eigen::SparseMatrix
// (linalg.hpp:12-16).  `rowMajor` selects CSR (outer = rows) or CSC.
struct Triplet {
    int64_t r, c;
    double v;
};

struct SpMat {
    bool rowMajor = true;
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> outer{0};  // outerSize()+1
    std::vector<int32_t> inner;
    std::vector<double> val;

    int64_t outerSize() const { return rowMajor ? rows : cols; }
    int64_t nnz() const { return static_cast<int64_t>(val.size()); }
    double coeff(int64_t r, int64_t c) const {
        int64_t o = rowMajor ? r : c, in = rowMajor ? c : r;
        for (int64_t e = outer[o]; e < outer[o + 1]; ++e)
            if (inner[e] == in) return val[e];
        return 0.0;
    }
};

// makeSparse (linalg.hpp:18-25): setFromTriplets + prune(0,0) + makeCompressed.
inline SpMat makeSparse(int64_t rows, int64_t cols, const std::vector<Triplet>& t, bool rowMajor) {
    SpMat m;
    m.rowMajor = rowMajor;
    m.rows = rows;
    m.cols = cols;
    int64_t nOuter = rowMajor ? rows : cols;
    std::vector<int64_t> cnt(static_cast<size_t>(nOuter) + 1, 0);
    for (const Triplet& x : t) {
        if (x.r < 0 || x.r >= rows || x.c < 0 || x.c >= cols)
            throw ContractError("triplet outside matrix");
        cnt[static_cast<size_t>(rowMajor ? x.r : x.c) + 1]++;
    }
    for (int64_t o = 0; o < nOuter; ++o) cnt[o + 1] += cnt[o];
    // stable bucket by outer index keeps triplet order inside each bucket
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    std::vector<std::pair<int32_t, double>> tmp(t.size());
    for (size_t k = 0; k < t.size(); ++k) {
        int64_t o = rowMajor ? t[k].r : t[k].c;
        int64_t in = rowMajor ? t[k].c : t[k].r;
        tmp[static_cast<size_t>(pos[o]++)] = {static_cast<int32_t>(in), t[k].v};
    }
    m.outer.assign(static_cast<size_t>(nOuter) + 1, 0);
    m.inner.reserve(t.size());
    m.val.reserve(t.size());
    for (int64_t o = 0; o < nOuter; ++o) {
        auto b = tmp.begin() + cnt[o], e = tmp.begin() + cnt[o + 1];
        std::stable_sort(b, e, [](const auto& a, const auto& c) { return a.first < c.first; });
        for (auto it = b; it != e;) {
            int32_t in = it->first;
            double s = it->second;
            ++it;
            while (it != e && it->first == in) {  // duplicates summed in insertion order
                s = s + it->second;
                ++it;
            }
            if (s != 0.0) {  // prune(0.0, 0.0)
                m.inner.push_back(in);
                m.val.push_back(s);
            }
        }
        m.outer[static_cast<size_t>(o) + 1] = static_cast<int64_t>(m.val.size());
    }
    return m;
}

inline std::vector<Triplet> toTriplets(const SpMat& m) {
    std::vector<Triplet> t;
    t.reserve(m.val.size());
    for (int64_t o = 0; o < m.outerSize(); ++o)
        for (int64_t e = m.outer[o]; e < m.outer[o + 1]; ++e)
            t.push_back(m.rowMajor ? Triplet{o, m.inner[e], m.val[e]} : Triplet{m.inner[e], o, m.val[e]});
    return t;
}

// SpMatR(X.transpose()) style conversion: same matrix, other storage order,
// or the transpose kept in the same storage order.
inline SpMat transposed(const SpMat& m, bool rowMajorOut) {
    std::vector<Triplet> t = toTriplets(m);
    for (auto& x : t) std::swap(x.r, x.c);
    return makeSparse(m.cols, m.rows, t, rowMajorOut);
}

// ---------------------------------------------------------------- cards ---
// cards.hpp:17-56: rank 2..14, suit c=0 d=1 h=2 s=3, ordered rank then suit.
struct Card {
    int8_t rank = 2, suit = 0;
    Card() = default;
    Card(int r, int s) : rank(static_cast<int8_t>(r)), suit(static_cast<int8_t>(s)) {
        if (r < 2 || r > 14 || s < 0 || s > 3)
            throw InvalidInputError("card out of range: rank=" + std::to_string(r) + " suit=" + std::to_string(s));
    }
    int id() const { return (rank - 2) * 4 + suit; }
    std::string code() const {
        static constexpr char kR[] = "23456789TJQKA", kS[] = "cdhs";
        return {kR[rank - 2], kS[suit]};
    }
    static Card fromCode(std::string_view c) {
        static constexpr std::string_view kR = "23456789TJQKA", kS = "cdhs";
        if (c.size() != 2) throw InvalidInputError("bad card code '" + std::string(c) + "'");
        auto r = kR.find(c[0]), s = kS.find(c[1]);
        if (r == std::string_view::npos || s == std::string_view::npos)
            throw InvalidInputError("bad card code '" + std::string(c) + "'");
        return Card(static_cast<int>(r) + 2, static_cast<int>(s));
    }
    friend auto operator<=>(const Card&, const Card&) = default;
};

// cards.hpp:60-95: canonical high card first.
struct Hand {
    Card high, low;
    Hand() = default;
    Hand(Card a, Card b) {
        if (a == b) throw InvalidInputError("hand repeats card " + a.code());
        if (a < b) std::swap(a, b);
        high = a;
        low = b;
    }
    bool contains(Card c) const { return c == high || c == low; }
    bool overlaps(const Hand& o) const { return contains(o.high) || contains(o.low); }
    std::string code() const { return high.code() + low.code(); }
    static Hand fromCode(std::string_view c) {
        if (c.size() != 4) throw InvalidInputError("bad hand code '" + std::string(c) + "'");
        return Hand(Card::fromCode(c.substr(0, 2)), Card::fromCode(c.substr(2, 2)));
    }
    friend auto operator<=>(const Hand&, const Hand&) = default;
};

struct Board {
    std::array<Card, 5> cards{};
    Board() = default;
    explicit Board(std::array<Card, 5> cs) : cards(cs) {
        for (int i = 0; i < 5; ++i)
            for (int j = i + 1; j < 5; ++j)
                if (cards[i] == cards[j]) throw InvalidInputError("board repeats card " + cards[i].code());
    }
    bool contains(Card c) const { return std::find(cards.begin(), cards.end(), c) != cards.end(); }
    bool overlaps(const Hand& h) const { return contains(h.high) || contains(h.low); }
    static Board fromCode(std::string_view c) {
        if (c.size() != 10) throw InvalidInputError("bad board code");
        std::array<Card, 5> cs;
        for (int i = 0; i < 5; ++i) cs[i] = Card::fromCode(c.substr(2 * i, 2));
        return Board(cs);
    }
    friend bool operator==(const Board&, const Board&) = default;
};

struct Deck {
    std::vector<Card> cards;
    static Deck standard52() {
        Deck d;
        for (int r = 2; r <= 14; ++r)
            for (int s = 0; s < 4; ++s) d.cards.emplace_back(r, s);
        return d;
    }
    bool contains(Card c) const { return std::find(cards.begin(), cards.end(), c) != cards.end(); }
    void validate() const {
        for (size_t i = 0; i < cards.size(); ++i)
            for (size_t j = i + 1; j < cards.size(); ++j)
                if (cards[i] == cards[j]) throw InvalidInputError("deck repeats card " + cards[i].code());
    }
};

// cards.hpp:167-194 packed key; 200-217 helpers; 223-304 evaluate7.
inline uint32_t packRank(int cat, int a, int b = 0, int c = 0, int d = 0, int e = 0) {
    return (uint32_t(cat) << 20) | (uint32_t(a) << 16) | (uint32_t(b) << 12) | (uint32_t(c) << 8) |
           (uint32_t(d) << 4) | uint32_t(e);
}
inline int straightTop(uint32_t mask) {
    for (int top = 14; top >= 6; --top) {
        uint32_t run = 0x1Fu << (top - 4);
        if ((mask & run) == run) return top;
    }
    constexpr uint32_t kWheel = (1u << 14) | (1u << 5) | (1u << 4) | (1u << 3) | (1u << 2);
    return (mask & kWheel) == kWheel ? 5 : 0;
}
inline void topRanks(uint32_t mask, int ex1, int ex2, int want, int* out) {
    int got = 0;
    for (int r = 14; r >= 2 && got < want; --r) {
        if (r == ex1 || r == ex2) continue;
        if (mask & (1u << r)) out[got++] = r;
    }
    while (got < want) out[got++] = 0;
}
inline uint32_t evaluate7(const Hand& h, const Board& b) {
    std::array<Card, 7> cs = {h.high, h.low, b.cards[0], b.cards[1], b.cards[2], b.cards[3], b.cards[4]};
    uint64_t seen = 0;
    for (const Card& c : cs) {
        uint64_t bit = 1ull << c.id();
        if (seen & bit) throw InvalidInputError("hand shares card " + c.code() + " with board");
        seen |= bit;
    }
    int rankCnt[15] = {}, suitCnt[4] = {};
    uint32_t suitMask[4] = {}, rankMask = 0;
    for (const Card& c : cs) {
        ++rankCnt[c.rank];
        ++suitCnt[c.suit];
        suitMask[c.suit] |= 1u << c.rank;
        rankMask |= 1u << c.rank;
    }
    int flushSuit = -1;
    for (int s = 0; s < 4; ++s)
        if (suitCnt[s] >= 5) flushSuit = s;
    if (flushSuit >= 0)
        if (int st = straightTop(suitMask[flushSuit]); st > 0) return packRank(8, st);
    int quad = 0, trip1 = 0, trip2 = 0, pair1 = 0, pair2 = 0;
    for (int r = 14; r >= 2; --r) {
        switch (rankCnt[r]) {
            case 4: quad = r; break;
            case 3:
                if (!trip1) trip1 = r;
                else if (!trip2) trip2 = r;
                break;
            case 2:
                if (!pair1) pair1 = r;
                else if (!pair2) pair2 = r;
                break;
            default: break;
        }
    }
    int k[5];
    if (quad) {
        topRanks(rankMask, quad, 0, 1, k);
        return packRank(7, quad, k[0]);
    }
    if (trip1 && (trip2 || pair1)) return packRank(6, trip1, trip2 > pair1 ? trip2 : pair1);
    if (flushSuit >= 0) {
        topRanks(suitMask[flushSuit], 0, 0, 5, k);
        return packRank(5, k[0], k[1], k[2], k[3], k[4]);
    }
    if (int st = straightTop(rankMask); st > 0) return packRank(4, st);
    if (trip1) {
        topRanks(rankMask, trip1, 0, 2, k);
        return packRank(3, trip1, k[0], k[1]);
    }
    if (pair1 && pair2) {
        topRanks(rankMask, pair1, pair2, 1, k);
        return packRank(2, pair1, pair2, k[0]);
    }
    if (pair1) {
        topRanks(rankMask, pair1, 0, 3, k);
        return packRank(1, pair1, k[0], k[1], k[2]);
    }
    topRanks(rankMask, 0, 0, 5, k);
    return packRank(0, k[0], k[1], k[2], k[3], k[4]);
}

// cards.hpp:308-319
inline int gammaSign(const Hand& h1, const Hand& h2, const Board& b) {
    if (b.overlaps(h1)) throw InvalidInputError("hand " + h1.code() + " shares a card with the board");
    if (b.overlaps(h2)) throw InvalidInputError("hand " + h2.code() + " shares a card with the board");
    if (h1.overlaps(h2)) return 0;
    uint32_t r1 = evaluate7(h1, b), r2 = evaluate7(h2, b);
    return r1 > r2 ? 1 : (r1 < r2 ? -1 : 0);
}

// -------------------------------------------------------------- skeleton ---
// skeleton.hpp:19-126
constexpr double kMoneyTol = 1e-6;
enum BetContext { FirstAction = 0, FacingCheck = 1, FacingBet = 2, AfterOneRaise = 3, AfterMultipleRaises = 4 };
constexpr int kBetContexts = 5;
inline const char* betContextName(int c) {
    static const char* n[] = {"first_action", "facing_check", "facing_bet", "after_one_raise",
                              "after_multiple_raises"};
    return n[c];
}

struct BettingConfig {
    double stack1 = 0, stack2 = 0, potContribution = 0;
    std::array<std::vector<double>, kBetContexts> menu1{}, menu2{};
    bool allIn = true;
    std::optional<int> raiseCap{};
    const std::vector<double>& menu(int p, int ctx) const { return (p == 0 ? menu1 : menu2)[ctx]; }
    double cap() const { return potContribution + std::min(stack1, stack2); }
    void validate() const {
        if (!(stack1 > 0) || !(stack2 > 0)) throw InvalidInputError("stacks must be positive");
        if (!(potContribution > 0)) throw InvalidInputError("pot contribution must be positive");
        for (const auto* ms : {&menu1, &menu2})
            for (const auto& m : *ms)
                for (double f : m)
                    if (!(f > 0) || !std::isfinite(f))
                        throw InvalidInputError("bet fractions must be positive and finite");
        if (raiseCap && *raiseCap < 0) throw InvalidInputError("raise cap must be nonnegative");
    }
};

enum ActKind { Check, Fold, Call, Bet, Raise, AllIn };
struct SkAction {
    ActKind kind = Check;
    double fraction = 0, target = 0;
    int seq = 0;
    bool toTerminal = false;
    int child = -1;
};
struct SkNode {
    int player = 0;
    double contrib1 = 0, contrib2 = 0;
    int context = 0;
    int parentSeq1 = 0, parentSeq2 = 0;
    std::vector<SkAction> actions;
    int parentSeq(int p) const { return p == 0 ? parentSeq1 : parentSeq2; }
};
struct SkTerminal {
    bool fold = false;
    int folder = -1;
    double q1 = 0, q2 = 0;
    int seq1 = 0, seq2 = 0;
    std::string path;
};
struct Skeleton {
    BettingConfig config;
    std::vector<SkNode> nodes;
    std::vector<SkTerminal> terminals;
    std::array<int, 2> seqCount{0, 0};
    std::array<std::vector<int>, 2> playerNodes{};
    std::array<std::vector<int>, 2> seqParent{};
    int sequences(int p) const { return seqCount[p]; }
    int decisionNodes(int p) const { return static_cast<int>(playerNodes[p].size()); }
};

inline std::string fractionToken(double f) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%g", f);
    return buf;
}

// skeleton.hpp:136-311 SkeletonBuilder
struct SkeletonBuilder {
    const BettingConfig& cfg;
    Skeleton out;
    double cap;
    explicit SkeletonBuilder(const BettingConfig& c) : cfg(c), cap(c.cap()) {
        out.config = c;
        out.seqParent[0].push_back(0);
        out.seqParent[1].push_back(0);
    }
    int newSeq(int p, int parent) {
        int s = ++out.seqCount[p];
        out.seqParent[p].push_back(parent);
        return s;
    }
    int addTerminal(SkTerminal t) {
        out.terminals.push_back(std::move(t));
        return static_cast<int>(out.terminals.size()) - 1;
    }
    int build(int player, double c1, double c2, int bets, bool checked, int ps1, int ps2, const std::string& path) {
        double own = player == 0 ? c1 : c2;
        double other = player == 0 ? c2 : c1;
        bool equal = std::abs(c1 - c2) <= kMoneyTol;
        int ctx;
        if (equal) ctx = checked ? FacingCheck : FirstAction;
        else if (bets <= 1) ctx = FacingBet;
        else if (bets == 2) ctx = AfterOneRaise;
        else ctx = AfterMultipleRaises;

        int nodeIdx = static_cast<int>(out.nodes.size());
        out.nodes.emplace_back();
        out.playerNodes[player].push_back(nodeIdx);
        {
            SkNode& n = out.nodes.back();
            n.player = player;
            n.contrib1 = c1;
            n.contrib2 = c2;
            n.context = ctx;
            n.parentSeq1 = ps1;
            n.parentSeq2 = ps2;
        }
        int ownParent = player == 0 ? ps1 : ps2;
        std::vector<SkAction> acts;
        if (equal) {
            SkAction a;
            a.kind = Check;
            a.target = own;
            acts.push_back(a);
        } else {
            SkAction f;
            f.kind = Fold;
            f.target = own;
            acts.push_back(f);
            SkAction c;
            c.kind = Call;
            c.target = other;
            acts.push_back(c);
        }
        bool open = !cfg.raiseCap || bets < *cfg.raiseCap;
        if (open) {
            struct Cand {
                double target, fraction;
                ActKind kind;
            };
            std::vector<Cand> cands;
            double maxc = std::max(c1, c2);
            for (double f : cfg.menu(player, ctx)) {
                double t = equal ? own + f * (c1 + c2) : other + f * (2.0 * other);
                if (t > cap - kMoneyTol) t = cap;
                if (t <= maxc + kMoneyTol) continue;
                cands.push_back({t, f, equal ? Bet : Raise});
            }
            if (cfg.allIn && cap > maxc + kMoneyTol) cands.push_back({cap, 0.0, AllIn});
            std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.target < b.target; });
            for (size_t i = 0; i < cands.size(); ++i) {
                if (i > 0 && std::abs(cands[i].target - cands[i - 1].target) <= kMoneyTol) continue;
                SkAction a;
                a.target = cands[i].target;
                a.fraction = cands[i].fraction;
                a.kind = std::abs(a.target - cap) <= kMoneyTol ? AllIn : cands[i].kind;
                acts.push_back(a);
            }
        }
        for (SkAction& a : acts) a.seq = newSeq(player, ownParent);
        for (SkAction& a : acts) {
            int nps1 = player == 0 ? a.seq : ps1;
            int nps2 = player == 1 ? a.seq : ps2;
            double nc1 = player == 0 ? a.target : c1;
            double nc2 = player == 1 ? a.target : c2;
            std::string tok;
            switch (a.kind) {
                case Check: tok = "k"; break;
                case Fold: tok = "f"; break;
                case Call: tok = "c"; break;
                case Bet: tok = "b" + fractionToken(a.fraction); break;
                case Raise: tok = "r" + fractionToken(a.fraction); break;
                case AllIn: tok = "a"; break;
            }
            std::string cp = path.empty() ? tok : path + "/" + tok;
            switch (a.kind) {
                case Check:
                    if (checked) {
                        SkTerminal t;
                        t.q1 = c1;
                        t.q2 = c2;
                        t.seq1 = nps1;
                        t.seq2 = nps2;
                        t.path = cp;
                        a.toTerminal = true;
                        a.child = addTerminal(std::move(t));
                    } else {
                        a.child = build(1 - player, c1, c2, bets, true, nps1, nps2, cp);
                    }
                    break;
                case Fold: {
                    SkTerminal t;
                    t.fold = true;
                    t.folder = player;
                    t.q1 = c1;
                    t.q2 = c2;
                    t.seq1 = nps1;
                    t.seq2 = nps2;
                    t.path = cp;
                    a.toTerminal = true;
                    a.child = addTerminal(std::move(t));
                    break;
                }
                case Call: {
                    SkTerminal t;
                    t.q1 = nc1;
                    t.q2 = nc2;
                    t.seq1 = nps1;
                    t.seq2 = nps2;
                    t.path = cp;
                    a.toTerminal = true;
                    a.child = addTerminal(std::move(t));
                    break;
                }
                default:
                    a.child = build(1 - player, nc1, nc2, bets + 1, false, nps1, nps2, cp);
                    break;
            }
        }
        out.nodes[nodeIdx].actions = std::move(acts);
        return nodeIdx;
    }
};

// skeleton.hpp:316-321
inline Skeleton buildSkeleton(const BettingConfig& cfg) {
    cfg.validate();
    SkeletonBuilder b(cfg);
    b.build(0, cfg.potContribution, cfg.potContribution, 0, false, 0, 0, "");
    return std::move(b.out);
}

// skeleton.hpp:332-349
inline std::pair<SpMat, SpMat> payoffComponents(const Skeleton& sk) {
    std::vector<Triplet> ft, st;
    for (const SkTerminal& t : sk.terminals) {
        if (t.seq1 <= 0 || t.seq2 <= 0) throw ContractError("terminal missing a sequence for one player");
        int i = t.seq1 - 1, j = t.seq2 - 1;
        if (t.fold) ft.push_back({i, j, t.folder == 1 ? t.q2 : -t.q1});
        else st.push_back({i, j, t.q1});
    }
    return {makeSparse(sk.sequences(0), sk.sequences(1), ft, true),
            makeSparse(sk.sequences(0), sk.sequences(1), st, true)};
}

// ------------------------------------------------------------------ kron ---
// kron.hpp:18-37
struct RiverInstance {
    Board board;
    std::array<std::vector<Hand>, 2> hands{};
    std::array<std::vector<double>, 2> beliefs{};
    BettingConfig config;
    Deck deck = Deck::standard52();
    int handCount(int p) const { return static_cast<int>(hands[p].size()); }
};

// kron.hpp:39-98
inline RiverInstance makeRiverInstance(const Board& board, std::vector<Hand> h1, std::vector<double> b1,
                                       std::vector<Hand> h2, std::vector<double> b2, const BettingConfig& cfg,
                                       Deck deck = Deck::standard52()) {
    cfg.validate();
    deck.validate();
    for (const Card& c : board.cards)
        if (!deck.contains(c)) throw InvalidInputError("board card " + c.code() + " not in the deck");
    RiverInstance inst;
    inst.board = board;
    inst.config = cfg;
    inst.deck = std::move(deck);
    std::array<std::vector<Hand>*, 2> hs = {&h1, &h2};
    std::array<std::vector<double>*, 2> bs = {&b1, &b2};
    for (int p = 0; p < 2; ++p) {
        auto& hands = *hs[p];
        auto& w = *bs[p];
        if (hands.empty()) throw InvalidInputError("player " + std::to_string(p + 1) + " has no hands");
        if (hands.size() != w.size()) throw InvalidInputError("hand/weight count mismatch");
        for (double x : w)
            if (!(x >= 0) || !std::isfinite(x)) throw InvalidInputError("belief weights must be finite and nonnegative");
        for (const Hand& h : hands) {
            if (!inst.deck.contains(h.high) || !inst.deck.contains(h.low))
                throw InvalidInputError("hand " + h.code() + " uses a card outside the deck");
            if (inst.board.overlaps(h)) throw InvalidInputError("hand " + h.code() + " shares a card with the board");
        }
        std::vector<size_t> order(hands.size());
        std::iota(order.begin(), order.end(), size_t{0});
        std::vector<uint32_t> strength(hands.size());
        for (size_t i = 0; i < hands.size(); ++i) strength[i] = evaluate7(hands[i], inst.board);
        std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
            if (strength[a] != strength[b]) return strength[a] < strength[b];
            return hands[a] < hands[b];
        });
        for (size_t i : order) {
            inst.hands[p].push_back(hands[i]);
            inst.beliefs[p].push_back(w[i]);
        }
        for (size_t i = 1; i < inst.hands[p].size(); ++i)
            if (inst.hands[p][i] == inst.hands[p][i - 1])
                throw InvalidInputError("duplicate hand " + inst.hands[p][i].code());
    }
    return inst;
}

// kron.hpp:104-132 — W and Hcross held row-major dense (m1 x m2).
struct KronPayoff {
    Skeleton skeleton;
    SpMat F, S;
    int n1 = 0, n2 = 0;
    std::array<std::vector<Hand>, 2> hands{};
    Vec mu1, mu2;
    double beta = 0;
    Vec lambda1, lambda2;
    std::vector<double> W, Hcross;
    int m1() const { return static_cast<int>(hands[0].size()); }
    int m2() const { return static_cast<int>(hands[1].size()); }
    int handCount(int p) const { return p == 0 ? m1() : m2(); }
    int64_t rows() const { return int64_t(m1()) * n1; }
    int64_t cols() const { return int64_t(m2()) * n2; }
    double w(int i, int j) const { return W[size_t(i) * m2() + j]; }
    double hx(int i, int j) const { return Hcross[size_t(i) * m2() + j]; }
    double pi(int i, int j) const { return lambda1[i] * lambda2[j] * (1.0 - hx(i, j)); }  // kron.hpp:129-131
};

// kron.hpp:134-166
inline KronPayoff assemble(const RiverInstance& inst) {
    KronPayoff kp;
    kp.skeleton = buildSkeleton(inst.config);
    auto [F, S] = payoffComponents(kp.skeleton);
    kp.F = std::move(F);
    kp.S = std::move(S);
    kp.n1 = kp.skeleton.sequences(0);
    kp.n2 = kp.skeleton.sequences(1);
    kp.hands = inst.hands;
    int m1 = inst.handCount(0), m2 = inst.handCount(1);
    kp.mu1 = inst.beliefs[0];
    kp.mu2 = inst.beliefs[1];
    kp.W.assign(size_t(m1) * m2, 0.0);
    kp.Hcross.assign(size_t(m1) * m2, 0.0);
    double beta = 0;
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j) {
            const Hand& a = inst.hands[0][i];
            const Hand& b = inst.hands[1][j];
            if (inst.board.overlaps(a) || inst.board.overlaps(b)) throw InvalidInputError("hand shares a card with the board");
            bool ok = !a.overlaps(b);
            kp.Hcross[size_t(i) * m2 + j] = ok ? 0.0 : 1.0;
            kp.W[size_t(i) * m2 + j] = ok ? gammaSign(a, b, inst.board) : 0.0;
            if (ok) beta += kp.mu1[i] * kp.mu2[j];
        }
    if (!(beta > 0)) throw DegenerateBeliefsError("no compatible hand pair carries belief mass");
    kp.beta = beta;
    double sb = std::sqrt(beta);
    kp.lambda1.resize(m1);
    kp.lambda2.resize(m2);
    for (int i = 0; i < m1; ++i) kp.lambda1[i] = kp.mu1[i] / sb;
    for (int j = 0; j < m2; ++j) kp.lambda2[j] = kp.mu2[j] / sb;
    return kp;
}

// kron.hpp:170-192 — row-major dense.
inline std::vector<double> denseExpand(const KronPayoff& kp, double guard = 5e7) {
    double cells = double(kp.rows()) * double(kp.cols());
    if (cells > guard) throw GuardError("dense payoff exceeds guard");
    int64_t C = kp.cols();
    std::vector<double> A(size_t(kp.rows()) * C, 0.0);
    for (int i = 0; i < kp.m1(); ++i)
        for (int j = 0; j < kp.m2(); ++j) {
            double p = kp.pi(i, j);
            if (p == 0.0) continue;
            double g = kp.w(i, j);
            int64_t r0 = int64_t(i) * kp.n1, c0 = int64_t(j) * kp.n2;
            for (int64_t k = 0; k < kp.F.rows; ++k)
                for (int64_t e = kp.F.outer[k]; e < kp.F.outer[k + 1]; ++e)
                    A[size_t(r0 + k) * C + c0 + kp.F.inner[e]] += p * kp.F.val[e];
            if (g != 0.0)
                for (int64_t k = 0; k < kp.S.rows; ++k)
                    for (int64_t e = kp.S.outer[k]; e < kp.S.outer[k + 1]; ++e)
                        A[size_t(r0 + k) * C + c0 + kp.S.inner[e]] += p * g * kp.S.val[e];
        }
    return A;
}

// kron.hpp:198-207
inline int64_t densePayoffNonzeros(const KronPayoff& kp) {
    int64_t nF = kp.F.nnz(), nS = kp.S.nnz(), total = 0;
    for (int i = 0; i < kp.m1(); ++i)
        for (int j = 0; j < kp.m2(); ++j) {
            if (kp.pi(i, j) == 0.0) continue;
            total += nF + (kp.w(i, j) != 0.0 ? nS : 0);
        }
    return total;
}

// Eigen's SparseMatrix*Vec: per row, sequential sum over the stored entries.
inline Vec spmvRows(const SpMat& A, const double* x) {
    Vec y(size_t(A.rows), 0.0);
    for (int64_t r = 0; r < A.rows; ++r) {
        double acc = 0;
        for (int64_t e = A.outer[r]; e < A.outer[r + 1]; ++e) acc += A.val[e] * x[A.inner[e]];
        y[r] = acc;
    }
    return y;
}

// kron.hpp:211-231 (block formula; Eigen evaluates p*vF + (p*W)*vS per element)
inline Vec referenceMatvec(const KronPayoff& kp, const Vec& x) {
    if (int64_t(x.size()) != kp.cols()) throw InvalidInputError("matvec input has the wrong size");
    int m1 = kp.m1(), m2 = kp.m2(), n1 = kp.n1, n2 = kp.n2;
    std::vector<Vec> vF(m2), vS(m2);
    for (int j = 0; j < m2; ++j) {
        vF[j] = spmvRows(kp.F, x.data() + size_t(j) * n2);
        vS[j] = spmvRows(kp.S, x.data() + size_t(j) * n2);
    }
    Vec y(size_t(kp.rows()), 0.0);
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j) {
            double p = kp.pi(i, j);
            if (p == 0.0) continue;
            double pw = p * kp.w(i, j);
            for (int a = 0; a < n1; ++a) y[size_t(i) * n1 + a] += p * vF[j][a] + pw * vS[j][a];
        }
    return y;
}

// kron.hpp:234-254
inline Vec referenceMatvecT(const KronPayoff& kp, const Vec& y) {
    if (int64_t(y.size()) != kp.rows()) throw InvalidInputError("matvec input has the wrong size");
    int m1 = kp.m1(), m2 = kp.m2(), n1 = kp.n1, n2 = kp.n2;
    SpMat Ft = transposed(kp.F, true), St = transposed(kp.S, true);
    std::vector<Vec> uF(m1), uS(m1);
    for (int i = 0; i < m1; ++i) {
        uF[i] = spmvRows(Ft, y.data() + size_t(i) * n1);
        uS[i] = spmvRows(St, y.data() + size_t(i) * n1);
    }
    Vec x(size_t(kp.cols()), 0.0);
    for (int j = 0; j < m2; ++j)
        for (int i = 0; i < m1; ++i) {
            double p = kp.pi(i, j);
            if (p == 0.0) continue;
            double pw = p * kp.w(i, j);
            for (int b = 0; b < n2; ++b) x[size_t(j) * n2 + b] += p * uF[i][b] + pw * uS[i][b];
        }
    return x;
}

// -------------------------------------------------------------- sparsify ---
// sparsify.hpp:17-22 — rectangle factorization of W (int8 working copy).
struct WFactorization {
    SpMat What, U, V;
    int rank() const { return static_cast<int>(U.cols); }
};

struct Rect {
    int gain = 0, value = 0, r0 = 0, r1 = 0, c0 = 0, c1 = 0;
};

// sparsify.hpp:34-60
inline Rect bestRect(const std::vector<int8_t>& R, int rows, int cols, int v) {
    Rect best;
    std::vector<int> height(size_t(cols), 0), stack;
    for (int i = 0; i < rows; ++i) {
        for (int j = 0; j < cols; ++j) height[j] = R[size_t(i) * cols + j] == v ? height[j] + 1 : 0;
        stack.clear();
        for (int j = 0; j <= cols; ++j) {
            int h = j < cols ? height[j] : 0;
            while (!stack.empty() && height[stack.back()] >= h) {
                int top = stack.back();
                stack.pop_back();
                int hh = height[top];
                int left = stack.empty() ? 0 : stack.back() + 1;
                int width = j - left;
                int gain = hh * width - (hh + width);
                if (gain > best.gain) best = {gain, v, i - hh + 1, i, left, j - 1};
            }
            if (j < cols) stack.push_back(j);
        }
    }
    return best;
}

// sparsify.hpp:68-103 (W row-major dense rows x cols)
inline WFactorization sparsifyW(const std::vector<double>& W, int rows, int cols, int maxIters = 1000) {
    std::vector<int8_t> R(size_t(rows) * cols);
    for (size_t k = 0; k < R.size(); ++k) {
        double w = W[k];
        if (w != -1.0 && w != 0.0 && w != 1.0) throw InvalidInputError("showdown matrix entries must be -1, 0 or +1");
        R[k] = static_cast<int8_t>(w);
    }
    std::vector<Triplet> ut, vt;
    int rank = 0;
    for (int it = 0; it < maxIters; ++it) {
        Rect plus = bestRect(R, rows, cols, 1), minus = bestRect(R, rows, cols, -1);
        Rect best = plus.gain >= minus.gain ? plus : minus;
        if (best.gain <= 0) break;
        for (int i = best.r0; i <= best.r1; ++i) {
            for (int j = best.c0; j <= best.c1; ++j) R[size_t(i) * cols + j] = 0;
            ut.push_back({i, rank, double(best.value)});
        }
        for (int j = best.c0; j <= best.c1; ++j) vt.push_back({j, rank, 1.0});
        ++rank;
    }
    std::vector<Triplet> wt;
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j)
            if (R[size_t(i) * cols + j] != 0) wt.push_back({i, j, double(R[size_t(i) * cols + j])});
    WFactorization out;
    out.What = makeSparse(rows, cols, wt, true);
    out.U = makeSparse(rows, rank, ut, true);
    out.V = makeSparse(cols, rank, vt, true);
    return out;
}

enum class Technique { A, B };

// sparsify.hpp:110-121
struct Sparsification {
    SpMat Ahat;  // CSR
    SpMat U;     // CSR
    SpMat M;     // CSC
    SpMat V;     // CSC
    Technique technique = Technique::A;
    bool postprocessed = false;
    int64_t rows() const { return Ahat.rows; }
    int64_t cols() const { return Ahat.cols; }
    int64_t k() const { return M.rows; }
};

struct SizeReport {
    int64_t ahat = 0, u = 0, m = 0, v = 0;
    int64_t total() const { return ahat + u + m + v; }
};
inline SizeReport size(const Sparsification& s) { return {s.Ahat.nnz(), s.U.nnz(), s.M.nnz(), s.V.nnz()}; }

// sparsify.hpp:133-145
inline void validateSparsification(const Sparsification& s) {
    int64_t k = s.M.rows;
    if (s.M.cols != k) throw ContractError("M is not square");
    if (s.U.rows != s.Ahat.rows || s.U.cols != k) throw ContractError("U dimensions do not match Ahat/M");
    if (s.V.rows != s.Ahat.cols || s.V.cols != k) throw ContractError("V dimensions do not match Ahat/M");
    for (int64_t j = 0; j < k; ++j) {
        int64_t e = s.M.outer[j];
        if (e == s.M.outer[j + 1] || s.M.inner[e] != j || s.M.val[e] != 1.0)
            throw ContractError("M is not unit lower triangular at column " + std::to_string(j));
    }
}

// sparsify.hpp:149-158
inline void appendScaledKron(std::vector<Triplet>& out, int64_t i, int64_t j, double scale, const SpMat& Q,
                             int64_t qRows, int64_t qCols) {
    int64_t r0 = i * qRows, c0 = j * qCols;
    for (int64_t k = 0; k < Q.outerSize(); ++k)
        for (int64_t e = Q.outer[k]; e < Q.outer[k + 1]; ++e) {
            double v = scale * Q.val[e];
            if (v != 0.0) out.push_back({r0 + k, c0 + Q.inner[e], v});
        }
}

// sparsify.hpp:165-240
inline Sparsification techniqueA(const KronPayoff& kp, const WFactorization& wf) {
    int m1 = kp.m1(), m2 = kp.m2();
    if (wf.What.rows != m1 || wf.What.cols != m2 || wf.U.rows != m1 || wf.V.rows != m2 || wf.U.cols != wf.V.cols)
        throw ContractError("W factorization dimensions do not match the payoff");
    {
        std::vector<double> rebuilt(size_t(m1) * m2, 0.0);
        for (int64_t r = 0; r < m1; ++r)
            for (int64_t e = wf.What.outer[r]; e < wf.What.outer[r + 1]; ++e)
                rebuilt[size_t(r) * m2 + wf.What.inner[e]] += wf.What.val[e];
        SpMat Vc = transposed(wf.V, true);  // rank x m2 rows
        for (int64_t r = 0; r < m1; ++r)
            for (int64_t e = wf.U.outer[r]; e < wf.U.outer[r + 1]; ++e) {
                int64_t q = wf.U.inner[e];
                for (int64_t f = Vc.outer[q]; f < Vc.outer[q + 1]; ++f)
                    rebuilt[size_t(r) * m2 + Vc.inner[f]] += wf.U.val[e] * Vc.val[f];
            }
        for (size_t c = 0; c < rebuilt.size(); ++c)
            if (std::abs(rebuilt[c] - kp.W[c]) > 1e-12) throw ContractError("W factorization does not reconstruct W");
    }
    int r = wf.rank();
    int64_t n1 = kp.n1, n2 = kp.n2;
    int64_t k = int64_t(r) * n1 + n1;
    Sparsification s;
    s.technique = Technique::A;
    std::vector<Triplet> at;
    for (int64_t b = 0; b < wf.What.rows; ++b)
        for (int64_t e = wf.What.outer[b]; e < wf.What.outer[b + 1]; ++e) {
            int64_t c = wf.What.inner[e];
            appendScaledKron(at, b, c, kp.lambda1[b] * kp.lambda2[c] * wf.What.val[e], kp.S, n1, n2);
        }
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j)
            if (kp.hx(i, j) != 0.0) appendScaledKron(at, i, j, -kp.lambda1[i] * kp.lambda2[j], kp.F, n1, n2);
    s.Ahat = makeSparse(int64_t(m1) * n1, int64_t(m2) * n2, at, true);

    std::vector<Triplet> ut;
    for (int64_t b = 0; b < wf.U.rows; ++b)
        for (int64_t e = wf.U.outer[b]; e < wf.U.outer[b + 1]; ++e) {
            double v = kp.lambda1[b] * wf.U.val[e];
            if (v == 0.0) continue;
            for (int64_t d = 0; d < n1; ++d) ut.push_back({b * n1 + d, int64_t(wf.U.inner[e]) * n1 + d, v});
        }
    for (int i = 0; i < m1; ++i) {
        double v = kp.lambda1[i];
        if (v == 0.0) continue;
        for (int64_t d = 0; d < n1; ++d) ut.push_back({i * n1 + d, int64_t(r) * n1 + d, v});
    }
    s.U = makeSparse(s.Ahat.rows, k, ut, true);

    std::vector<Triplet> mt;
    for (int64_t d = 0; d < k; ++d) mt.push_back({d, d, 1.0});
    s.M = makeSparse(k, k, mt, false);

    SpMat St = transposed(kp.S, true), Ft = transposed(kp.F, true);
    std::vector<Triplet> vt;
    for (int64_t b = 0; b < wf.V.rows; ++b)
        for (int64_t e = wf.V.outer[b]; e < wf.V.outer[b + 1]; ++e) {
            double scale = kp.lambda2[b] * wf.V.val[e];
            if (scale == 0.0) continue;
            for (int64_t c = 0; c < St.rows; ++c)
                for (int64_t f = St.outer[c]; f < St.outer[c + 1]; ++f)
                    vt.push_back({b * n2 + c, int64_t(wf.V.inner[e]) * n1 + St.inner[f], scale * St.val[f]});
        }
    for (int j = 0; j < m2; ++j) {
        double scale = kp.lambda2[j];
        if (scale == 0.0) continue;
        for (int64_t c = 0; c < Ft.rows; ++c)
            for (int64_t f = Ft.outer[c]; f < Ft.outer[c + 1]; ++f)
                vt.push_back({int64_t(j) * n2 + c, int64_t(r) * n1 + Ft.inner[f], scale * Ft.val[f]});
    }
    s.V = makeSparse(s.Ahat.cols, k, vt, false);
    validateSparsification(s);
    return s;
}

// sparsify.hpp:246-312
inline Sparsification techniqueB(const KronPayoff& kp) {
    int m1 = kp.m1(), m2 = kp.m2();
    int64_t n1 = kp.n1, n2 = kp.n2;
    int64_t k = int64_t(m1) * n1 + n1;
    std::vector<double> Y(size_t(m1) * m2);
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j) Y[size_t(i) * m2 + j] = i == 0 ? kp.w(i, j) : kp.w(i, j) - kp.w(i - 1, j);
    Sparsification s;
    s.technique = Technique::B;
    std::vector<Triplet> at;
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j)
            if (kp.hx(i, j) != 0.0) appendScaledKron(at, i, j, -kp.lambda1[i] * kp.lambda2[j], kp.F, n1, n2);
    s.Ahat = makeSparse(int64_t(m1) * n1, int64_t(m2) * n2, at, true);

    std::vector<Triplet> ut;
    for (int i = 0; i < m1; ++i) {
        double v = kp.lambda1[i];
        if (v == 0.0) continue;
        for (int64_t d = 0; d < n1; ++d) {
            ut.push_back({i * n1 + d, i * n1 + d, v});
            ut.push_back({i * n1 + d, int64_t(m1) * n1 + d, v});
        }
    }
    s.U = makeSparse(s.Ahat.rows, k, ut, true);

    std::vector<Triplet> mt;
    for (int64_t d = 0; d < k; ++d) mt.push_back({d, d, 1.0});
    for (int i = 1; i < m1; ++i)
        for (int64_t d = 0; d < n1; ++d) mt.push_back({int64_t(i) * n1 + d, int64_t(i - 1) * n1 + d, -1.0});
    s.M = makeSparse(k, k, mt, false);

    SpMat St = transposed(kp.S, true), Ft = transposed(kp.F, true);
    std::vector<Triplet> vt;
    for (int i = 0; i < m1; ++i)
        for (int j = 0; j < m2; ++j) {
            double scale = kp.lambda2[j] * Y[size_t(i) * m2 + j];
            if (scale == 0.0) continue;
            for (int64_t c = 0; c < St.rows; ++c)
                for (int64_t f = St.outer[c]; f < St.outer[c + 1]; ++f)
                    vt.push_back({int64_t(j) * n2 + c, int64_t(i) * n1 + St.inner[f], scale * St.val[f]});
        }
    for (int j = 0; j < m2; ++j) {
        double scale = kp.lambda2[j];
        if (scale == 0.0) continue;
        for (int64_t c = 0; c < Ft.rows; ++c)
            for (int64_t f = Ft.outer[c]; f < Ft.outer[c + 1]; ++f)
                vt.push_back({int64_t(j) * n2 + c, int64_t(m1) * n1 + Ft.inner[f], scale * Ft.val[f]});
    }
    s.V = makeSparse(s.Ahat.cols, k, vt, false);
    validateSparsification(s);
    return s;
}

// sparsify.hpp:318-406 — std::map / std::set iteration order reproduced.
inline Sparsification postprocess(const Sparsification& s) {
    validateSparsification(s);
    int64_t k = s.k();
    std::vector<std::map<int64_t, double>> ucol(static_cast<size_t>(k));
    for (int64_t b = 0; b < s.U.rows; ++b)
        for (int64_t e = s.U.outer[b]; e < s.U.outer[b + 1]; ++e) ucol[s.U.inner[e]][b] = s.U.val[e];
    std::vector<std::map<int64_t, double>> mrow(static_cast<size_t>(k));
    std::vector<std::set<int64_t>> colRows(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j)
        for (int64_t e = s.M.outer[j]; e < s.M.outer[j + 1]; ++e)
            if (s.M.inner[e] != j) {
                mrow[s.M.inner[e]][j] = s.M.val[e];
                colRows[j].insert(s.M.inner[e]);
            }
    std::vector<bool> alive(static_cast<size_t>(k), true);
    for (int64_t j = 0; j < k; ++j) {
        if (s.V.outer[j] != s.V.outer[j + 1]) continue;  // V column j carries data
        auto subs = mrow[j];
        const auto uj = std::move(ucol[j]);
        for (const auto& [i, a] : subs) {
            auto& ui = ucol[i];
            for (const auto& [row, v] : uj) {
                double& slot = ui[row];
                slot += -a * v;
                if (slot == 0.0) ui.erase(row);
            }
        }
        auto refs = colRows[j];
        for (int64_t r : refs) {
            auto& row = mrow[r];
            auto itb = row.find(j);
            double b = itb->second;
            row.erase(itb);
            for (const auto& [i, a] : subs) {
                double& slot = row[i];
                bool fresh = slot == 0.0;
                slot -= b * a;
                if (slot == 0.0) row.erase(i);
                else if (fresh) colRows[i].insert(r);
            }
        }
        for (const auto& [i, a] : subs) {
            (void)a;
            colRows[i].erase(j);
        }
        ucol[j].clear();
        mrow[j].clear();
        colRows[j].clear();
        alive[j] = false;
    }
    std::vector<int64_t> remap(static_cast<size_t>(k), -1);
    int64_t kept = 0;
    for (int64_t j = 0; j < k; ++j)
        if (alive[j]) remap[j] = kept++;
    Sparsification out;
    out.Ahat = s.Ahat;
    out.technique = s.technique;
    out.postprocessed = true;
    std::vector<Triplet> ut, mt, vt;
    for (int64_t j = 0; j < k; ++j) {
        if (!alive[j]) continue;
        int64_t nj = remap[j];
        for (const auto& [row, v] : ucol[j])
            if (v != 0.0) ut.push_back({row, nj, v});
        mt.push_back({nj, nj, 1.0});
        for (const auto& [i, a] : mrow[j]) mt.push_back({nj, remap[i], a});
        for (int64_t e = s.V.outer[j]; e < s.V.outer[j + 1]; ++e) vt.push_back({s.V.inner[e], nj, s.V.val[e]});
    }
    out.U = makeSparse(s.U.rows, kept, ut, true);
    out.M = makeSparse(kept, kept, mt, false);
    out.V = makeSparse(s.V.rows, kept, vt, false);
    validateSparsification(out);
    if (size(out).total() > size(s).total()) throw ContractError("postprocessing increased the stored size");
    return out;
}

// ---------------------------------------------------------------- engine ---
// engine.hpp:14-18
struct GradientWorkspace {
    Vec y, z;
    int64_t flops = 0, totalFlops = 0;
};

// engine.hpp:21-28
inline bool isIdentity(const SpMat& M) {
    if (M.nnz() != M.rows) return false;
    for (int64_t j = 0; j < M.cols; ++j) {
        int64_t e = M.outer[j];
        if (e == M.outer[j + 1] || M.inner[e] != j || M.val[e] != 1.0) return false;
    }
    return true;
}

// engine.hpp:31-41
inline void solveUnitLower(const SpMat& M, Vec& z) {
    if (int64_t(z.size()) != M.rows) throw InvalidInputError("solve rhs has the wrong size");
    for (int64_t j = 0; j < M.cols; ++j) {
        int64_t e = M.outer[j], end = M.outer[j + 1];
        if (e == end || M.inner[e] != j || M.val[e] != 1.0)
            throw ContractError("M is not unit lower triangular at column " + std::to_string(j));
        double zj = z[j];
        if (zj == 0.0) continue;
        for (++e; e < end; ++e) z[M.inner[e]] -= M.val[e] * zj;
    }
}

// engine.hpp:44-54
inline void solveUnitLowerT(const SpMat& M, Vec& z) {
    if (int64_t(z.size()) != M.rows) throw InvalidInputError("solve rhs has the wrong size");
    for (int64_t j = M.cols - 1; j >= 0; --j) {
        int64_t e = M.outer[j], end = M.outer[j + 1];
        if (e == end || M.inner[e] != j || M.val[e] != 1.0)
            throw ContractError("M is not unit lower triangular at column " + std::to_string(j));
        double acc = 0;
        for (++e; e < end; ++e) acc += M.val[e] * z[M.inner[e]];
        z[j] -= acc;
    }
}

// engine.hpp:58-93
inline Vec matvec(const Sparsification& s, const Vec& x, GradientWorkspace& ws) {
    if (int64_t(x.size()) != s.cols())
        throw InvalidInputError("matvec input has size " + std::to_string(x.size()) + ", expected " +
                                std::to_string(s.cols()));
    int64_t k = s.k();
    ws.flops = 0;
    ws.y.assign(size_t(k), 0.0);
    const double* xp = x.data();
    for (int64_t t = 0; t < k; ++t) {
        double acc = 0;
        for (int64_t e = s.V.outer[t]; e < s.V.outer[t + 1]; ++e) acc += s.V.val[e] * xp[s.V.inner[e]];
        ws.y[t] = acc;
    }
    ws.flops += s.V.nnz();
    if (!isIdentity(s.M)) {
        solveUnitLower(s.M, ws.y);
        ws.flops += s.M.nnz() - k;
    }
    const Vec& z = ws.y;
    Vec out(size_t(s.rows()));
    for (int64_t i = 0; i < s.rows(); ++i) {
        double acc = 0;
        for (int64_t e = s.U.outer[i]; e < s.U.outer[i + 1]; ++e) acc += s.U.val[e] * z[s.U.inner[e]];
        for (int64_t e = s.Ahat.outer[i]; e < s.Ahat.outer[i + 1]; ++e) acc += s.Ahat.val[e] * xp[s.Ahat.inner[e]];
        out[i] = acc;
    }
    ws.flops += s.U.nnz() + s.Ahat.nnz();
    ws.totalFlops += ws.flops;
    return out;
}

// engine.hpp:96-133
inline Vec matvecTranspose(const Sparsification& s, const Vec& y, GradientWorkspace& ws) {
    if (int64_t(y.size()) != s.rows())
        throw InvalidInputError("matvec input has size " + std::to_string(y.size()) + ", expected " +
                                std::to_string(s.rows()));
    int64_t k = s.k();
    ws.flops = 0;
    ws.z.assign(size_t(k), 0.0);
    for (int64_t i = 0; i < s.rows(); ++i) {
        double yi = y[i];
        if (yi == 0.0) continue;
        for (int64_t e = s.U.outer[i]; e < s.U.outer[i + 1]; ++e) ws.z[s.U.inner[e]] += s.U.val[e] * yi;
    }
    ws.flops += s.U.nnz();
    if (!isIdentity(s.M)) {
        solveUnitLowerT(s.M, ws.z);
        ws.flops += s.M.nnz() - k;
    }
    Vec out(size_t(s.cols()), 0.0);
    for (int64_t i = 0; i < s.rows(); ++i) {
        double yi = y[i];
        if (yi == 0.0) continue;
        for (int64_t e = s.Ahat.outer[i]; e < s.Ahat.outer[i + 1]; ++e) out[s.Ahat.inner[e]] += s.Ahat.val[e] * yi;
    }
    ws.flops += s.Ahat.nnz();
    for (int64_t t = 0; t < k; ++t) {
        double zt = ws.z[t];
        if (zt == 0.0) continue;
        for (int64_t e = s.V.outer[t]; e < s.V.outer[t + 1]; ++e) out[s.V.inner[e]] += s.V.val[e] * zt;
    }
    ws.flops += s.V.nnz();
    ws.totalFlops += ws.flops;
    return out;
}

// ---------------------------------------------------------------- solver ---
// solver.hpp:21-27 GradientEngine and the engines at 30-99.
struct GradientEngine {
    virtual ~GradientEngine() = default;
    virtual Vec Ax(const Vec& x2) const = 0;
    virtual Vec ATx(const Vec& x1) const = 0;
    virtual int64_t flops() const { return 0; }
};
struct FactoredEngine : GradientEngine {
    const Sparsification* s;
    mutable GradientWorkspace ws;
    explicit FactoredEngine(const Sparsification& sp) : s(&sp) {}
    Vec Ax(const Vec& x) const override { return matvec(*s, x, ws); }
    Vec ATx(const Vec& y) const override { return matvecTranspose(*s, y, ws); }
    int64_t flops() const override { return ws.totalFlops; }
};
struct ReferenceEngine : GradientEngine {
    const KronPayoff* kp;
    explicit ReferenceEngine(const KronPayoff& k) : kp(&k) {}
    Vec Ax(const Vec& x) const override { return referenceMatvec(*kp, x); }
    Vec ATx(const Vec& y) const override { return referenceMatvecT(*kp, y); }
};
// DenseEngine (solver.hpp:43-51): Eigen's dense GEMV; its accumulation order
// is Eigen's, so it is compared with tolerance only.
struct DenseEngine : GradientEngine {
    std::vector<double> A;
    int64_t rows, cols;
    DenseEngine(std::vector<double> a, int64_t r, int64_t c) : A(std::move(a)), rows(r), cols(c) {}
    Vec Ax(const Vec& x) const override {
        Vec y(size_t(rows), 0.0);
        for (int64_t i = 0; i < rows; ++i) {
            double acc = 0;
            for (int64_t j = 0; j < cols; ++j) acc += A[size_t(i) * cols + j] * x[j];
            y[i] = acc;
        }
        return y;
    }
    Vec ATx(const Vec& y) const override {
        Vec x(size_t(cols), 0.0);
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < cols; ++j) x[j] += A[size_t(i) * cols + j] * y[i];
        return x;
    }
};

// solver.hpp:101-109
struct DcfrParams {
    double alpha = 1.5, beta = 0.0, gamma = 2.0;
    int maxIters = 1000;
    double targetExploitability = 0.0;
    int checkpointEvery = 50;
    int threads = 1;
    // Update rule (NOT in the reference, whose only solver is DCFR; SPEC.md:438
    // lists CFR+ as a non-goal).  0 = DCFR as solver.hpp:343-404.  1 = CFR+
    // style: each player's regrets are discounted right after its sweep and
    // its strategy is regret-matched on the discounted regrets (with alpha =
    // +inf, beta = -inf: R <- max(R + r, 0), i.e. regret matching+).  2 = PRM+
    // (predictive): as 1, but the strategy is regret-matched on R + r, the
    // last instantaneous regret serving as the prediction.
    int rule = 0;
};

// t^e / (t^e + 1) (solver.hpp:378-379), extended to e = +-inf by its limit
// (1 for +inf, 0 for -inf) where std::pow would give inf / inf.
inline double discountFactor(int t, double e) {
    if (std::isinf(e)) return e > 0 ? 1.0 : 0.0;
    double te = std::pow(double(t), e);
    return te / (te + 1);
}
struct TracePoint {
    int iteration = 0;
    double seconds = 0, exploitability = 0, br1 = 0, br2 = 0;
};
struct DcfrResult {
    Vec avg1, avg2;
    int iterations = 0;
    double exploitability = 0;
    std::vector<TracePoint> trace;
    int64_t gradientFlops = 0;
};

struct RegretTable {  // solver.hpp:145-159
    int player = 0, n = 0, handCount = 0;
    Vec regret, avg;
    void init(int p, int n_, int h) {
        player = p;
        n = n_;
        handCount = h;
        regret.assign(size_t(n) * h, 0.0);
        avg.assign(size_t(n) * h, 0.0);
    }
};

// solver.hpp:166-194
inline void regretMatch(const double* regrets, const std::vector<SkAction>& acts, int off, double* probs) {
    size_t count = acts.size();
    double best = regrets[off + acts[0].seq - 1];
    double maxAbs = std::abs(best);
    for (size_t a = 1; a < count; ++a) {
        double r = regrets[off + acts[a].seq - 1];
        best = std::max(best, r);
        maxAbs = std::max(maxAbs, std::abs(r));
    }
    double tol = 1e-9 * (1 + maxAbs);
    if (best > tol) {
        double sumPos = 0;
        for (size_t a = 0; a < count; ++a) {
            double r = regrets[off + acts[a].seq - 1];
            if (r > 0) sumPos += r;
        }
        for (size_t a = 0; a < count; ++a) {
            double r = regrets[off + acts[a].seq - 1];
            probs[a] = r > 0 ? r / sumPos : 0.0;
        }
        return;
    }
    int ties = 0;
    for (size_t a = 0; a < count; ++a)
        if (regrets[off + acts[a].seq - 1] >= best - tol) ++ties;
    for (size_t a = 0; a < count; ++a) probs[a] = regrets[off + acts[a].seq - 1] >= best - tol ? 1.0 / ties : 0.0;
}

// solver.hpp:197-218, regret-matching `regrets` (the table's own by default)
inline Vec sequenceForm(const Skeleton& sk, const RegretTable& rt, const Vec* regrets = nullptr) {
    const Vec& R = regrets ? *regrets : rt.regret;
    Vec x(size_t(rt.handCount) * rt.n, 0.0);
    const auto& nodes = sk.playerNodes[rt.player];
    std::vector<double> reach(size_t(rt.n) + 1), probs;
    for (int h = 0; h < rt.handCount; ++h) {
        int off = h * rt.n;
        reach[0] = 1.0;
        for (int idx : nodes) {
            const SkNode& v = sk.nodes[idx];
            double mass = reach[v.parentSeq(rt.player)];
            probs.resize(v.actions.size());
            regretMatch(R.data(), v.actions, off, probs.data());
            for (size_t a = 0; a < v.actions.size(); ++a) {
                double m = mass * probs[a];
                reach[v.actions[a].seq] = m;
                x[off + v.actions[a].seq - 1] = m;
            }
        }
    }
    return x;
}

// solver.hpp:222-260 (single-threaded: the reference's partition is bitwise
// neutral, test_solver.cpp:255-269)
inline void cfrSweep(const Skeleton& sk, RegretTable& rt, const Vec& g, Vec* inst = nullptr) {
    const auto& nodes = sk.playerNodes[rt.player];
    if (inst) inst->assign(rt.regret.size(), 0.0);
    std::vector<double> seqVal(size_t(rt.n) + 1), probs;
    for (int h = 0; h < rt.handCount; ++h) {
        int off = h * rt.n;
        std::fill(seqVal.begin(), seqVal.end(), 0.0);
        for (auto it = nodes.rbegin(); it != nodes.rend(); ++it) {
            const SkNode& v = sk.nodes[*it];
            probs.resize(v.actions.size());
            regretMatch(rt.regret.data(), v.actions, off, probs.data());
            double nodeVal = 0;
            for (size_t a = 0; a < v.actions.size(); ++a) {
                int seq = v.actions[a].seq;
                double ev = g[off + seq - 1] + seqVal[seq];
                seqVal[seq] = ev;
                nodeVal += probs[a] * ev;
            }
            for (const auto& act : v.actions) {
                const double d = seqVal[act.seq] - nodeVal;
                rt.regret[off + act.seq - 1] += d;
                if (inst) (*inst)[off + act.seq - 1] = d;
            }
            seqVal[v.parentSeq(rt.player)] += nodeVal;
        }
    }
}

// solver.hpp:262-264
inline void discount(RegretTable& rt, double pos, double neg) {
    for (double& r : rt.regret) r *= r > 0 ? pos : neg;
}

// solver.hpp:266-286
inline void validateSequenceStrategy(const Skeleton& sk, int player, int handCount, const Vec& x, double tol = 1e-9) {
    int n = sk.sequences(player);
    if (int64_t(x.size()) != int64_t(handCount) * n) throw InvalidInputError("strategy vector has the wrong size");
    for (double v : x)
        if (v < -tol) throw InvalidInputError("strategy vector has negative entries");
    for (int h = 0; h < handCount; ++h) {
        int off = h * n;
        for (int idx : sk.playerNodes[player]) {
            const SkNode& v = sk.nodes[idx];
            int p = v.parentSeq(player);
            double parentMass = p == 0 ? 1.0 : x[off + p - 1];
            double sum = 0;
            for (const auto& a : v.actions) sum += x[off + a.seq - 1];
            if (std::abs(sum - parentMass) > tol * (1 + std::abs(parentMass)))
                throw InvalidInputError("strategy violates flow conservation at a node");
        }
    }
}

// solver.hpp:292-321
inline double bestResponseValue(const KronPayoff& kp, const GradientEngine& eng, int player, const Vec& opp) {
    if (player != 0 && player != 1) throw InvalidInputError("player must be 0 or 1");
    const Skeleton& sk = kp.skeleton;
    validateSequenceStrategy(sk, 1 - player, kp.handCount(1 - player), opp);
    Vec g;
    if (player == 0) {
        g = eng.Ax(opp);
    } else {
        g = eng.ATx(opp);
        for (double& v : g) v = -v;
    }
    int n = player == 0 ? kp.n1 : kp.n2;
    const auto& nodes = sk.playerNodes[player];
    double total = 0;
    std::vector<double> seqVal(size_t(n) + 1);
    for (int h = 0; h < kp.handCount(player); ++h) {
        int off = h * n;
        std::fill(seqVal.begin(), seqVal.end(), 0.0);
        for (auto it = nodes.rbegin(); it != nodes.rend(); ++it) {
            const SkNode& v = sk.nodes[*it];
            double best = 0;
            bool first = true;
            for (const auto& a : v.actions) {
                double ev = g[off + a.seq - 1] + seqVal[a.seq];
                if (first || ev > best) best = ev;
                first = false;
            }
            seqVal[v.parentSeq(player)] += best;
        }
        total += seqVal[0];
    }
    return total;
}

// solver.hpp:325-331
inline double exploitability(const KronPayoff& kp, const GradientEngine& eng, const Vec& x1, const Vec& x2,
                             double* br1Out = nullptr, double* br2Out = nullptr) {
    double br1 = bestResponseValue(kp, eng, 0, x2);
    double br2 = bestResponseValue(kp, eng, 1, x1);
    if (br1Out) *br1Out = br1;
    if (br2Out) *br2Out = br2;
    double pot = 2 * kp.skeleton.config.potContribution;
    return (br1 + br2) / 2 / pot;
}

// solver.hpp:334-338
inline Vec uniformStrategy(const KronPayoff& kp, int player) {
    RegretTable rt;
    rt.init(player, player == 0 ? kp.n1 : kp.n2, kp.handCount(player));
    return sequenceForm(kp.skeleton, rt);
}

// One player's half-iteration: sweep, then (rules 1, 2) the discount of its
// own regrets, then its new strategy.  Rule 0 leaves the discount to the end
// of the iteration, as solver.hpp:378-380 does.
inline Vec playerUpdate(const Skeleton& sk, RegretTable& rt, const Vec& g, int rule, double pos, double neg) {
    if (rule == 0) {
        cfrSweep(sk, rt, g);
        return sequenceForm(sk, rt);
    }
    Vec r;
    cfrSweep(sk, rt, g, rule == 2 ? &r : nullptr);
    discount(rt, pos, neg);
    if (rule == 1) return sequenceForm(sk, rt);
    for (size_t e = 0; e < r.size(); ++e) r[e] = rt.regret[e] + r[e];  // prediction: R + last regret
    return sequenceForm(sk, rt, &r);
}

// solver.hpp:343-404
inline DcfrResult dcfrSolve(const KronPayoff& kp, const GradientEngine& eng, const DcfrParams& params) {
    if (params.maxIters < 1) throw InvalidInputError("iteration budget must be positive");
    if (params.checkpointEvery < 1) throw InvalidInputError("checkpoint period must be positive");
    const Skeleton& sk = kp.skeleton;
    RegretTable rt1, rt2;
    rt1.init(0, kp.n1, kp.handCount(0));
    rt2.init(1, kp.n2, kp.handCount(1));
    double weightSum = 0;
    DcfrResult res;
    int64_t flops0 = eng.flops();
    Vec x1 = sequenceForm(sk, rt1), x2 = sequenceForm(sk, rt2);
    for (int t = 1; t <= params.maxIters; ++t) {
        double pos = discountFactor(t, params.alpha), neg = discountFactor(t, params.beta);
        Vec g1 = eng.Ax(x2);
        x1 = playerUpdate(sk, rt1, g1, params.rule, pos, neg);
        Vec g2 = eng.ATx(x1);
        for (double& v : g2) v = -v;
        x2 = playerUpdate(sk, rt2, g2, params.rule, pos, neg);
        if (params.rule == 0) {
            discount(rt1, pos, neg);
            discount(rt2, pos, neg);
        }
        double shrink = std::pow(double(t) / (t + 1), params.gamma);
        for (size_t e = 0; e < x1.size(); ++e) rt1.avg[e] += x1[e];
        for (size_t e = 0; e < x2.size(); ++e) rt2.avg[e] += x2[e];
        weightSum += 1;
        for (double& v : rt1.avg) v *= shrink;
        for (double& v : rt2.avg) v *= shrink;
        weightSum *= shrink;
        if (t % params.checkpointEvery == 0 || t == params.maxIters) {
            Vec a1(rt1.avg.size()), a2(rt2.avg.size());
            for (size_t e = 0; e < a1.size(); ++e) a1[e] = rt1.avg[e] / weightSum;
            for (size_t e = 0; e < a2.size(); ++e) a2[e] = rt2.avg[e] / weightSum;
            TracePoint tp;
            tp.iteration = t;
            tp.exploitability = exploitability(kp, eng, a1, a2, &tp.br1, &tp.br2);
            res.trace.push_back(tp);
            res.iterations = t;
            res.exploitability = tp.exploitability;
            if (params.targetExploitability > 0 && tp.exploitability <= params.targetExploitability) break;
        }
    }
    res.avg1.resize(rt1.avg.size());
    res.avg2.resize(rt2.avg.size());
    for (size_t e = 0; e < res.avg1.size(); ++e) res.avg1[e] = rt1.avg[e] / weightSum;
    for (size_t e = 0; e < res.avg2.size(); ++e) res.avg2[e] = rt2.avg[e] / weightSum;
    res.gradientFlops = eng.flops() - flops0;
    return res;
}

// The loop body of dcfrSolve (solver.hpp:365-392) split into begin /
// iterate / checkpoint so a multi-rank test driver can combine boards between
// checkpoints; the arithmetic is the same statements in the same order.
struct DcfrState {
    const KronPayoff* kp;
    const GradientEngine* eng;
    DcfrParams p;
    RegretTable rt1, rt2;
    Vec x1, x2;
    double weightSum = 0;
    int t = 0;
    DcfrState(const KronPayoff& k, const GradientEngine& e) : kp(&k), eng(&e) {}
    void begin(const DcfrParams& params) {
        p = params;
        rt1.init(0, kp->n1, kp->handCount(0));
        rt2.init(1, kp->n2, kp->handCount(1));
        weightSum = 0;
        t = 0;
        x1 = sequenceForm(kp->skeleton, rt1);
        x2 = sequenceForm(kp->skeleton, rt2);
    }
    void iterate(int n) {
        const Skeleton& sk = kp->skeleton;
        for (int q = 0; q < n; ++q) {
            const int tt = ++t;
            double pos = discountFactor(tt, p.alpha), neg = discountFactor(tt, p.beta);
            Vec g1 = eng->Ax(x2);
            x1 = playerUpdate(sk, rt1, g1, p.rule, pos, neg);
            Vec g2 = eng->ATx(x1);
            for (double& v : g2) v = -v;
            x2 = playerUpdate(sk, rt2, g2, p.rule, pos, neg);
            if (p.rule == 0) {
                discount(rt1, pos, neg);
                discount(rt2, pos, neg);
            }
            double shrink = std::pow(double(tt) / (tt + 1), p.gamma);
            for (size_t e = 0; e < x1.size(); ++e) rt1.avg[e] += x1[e];
            for (size_t e = 0; e < x2.size(); ++e) rt2.avg[e] += x2[e];
            weightSum += 1;
            for (double& v : rt1.avg) v *= shrink;
            for (double& v : rt2.avg) v *= shrink;
            weightSum *= shrink;
        }
    }
    void checkpoint(double* br1, double* br2) const {
        Vec a1(rt1.avg.size()), a2(rt2.avg.size());
        for (size_t e = 0; e < a1.size(); ++e) a1[e] = rt1.avg[e] / weightSum;
        for (size_t e = 0; e < a2.size(); ++e) a2[e] = rt2.avg[e] / weightSum;
        *br1 = bestResponseValue(*kp, *eng, 0, a2);
        *br2 = bestResponseValue(*kp, *eng, 1, a1);
    }
};

// ------------------------------------------------------------- instances ---
// instances.hpp:19-29
inline BettingConfig referenceBettingConfig() {
    BettingConfig c;
    c.stack1 = c.stack2 = 18125;
    c.potContribution = 1875;
    for (int x = 0; x < kBetContexts; ++x) {
        c.menu1[x] = {0.75};
        c.menu2[x] = {0.75};
    }
    c.allIn = true;
    return c;
}

// instances.hpp:33-43
inline RiverInstance goldenInstance() {
    Board b = Board::fromCode("2c7d9hJc3s");
    std::vector<Hand> h1 = {Hand::fromCode("AcAd"), Hand::fromCode("KcKd"), Hand::fromCode("5c5d")};
    std::vector<Hand> h2 = {Hand::fromCode("AhAs"), Hand::fromCode("QcQd"), Hand::fromCode("7c7h")};
    return makeRiverInstance(b, h1, {0.5, 0.3, 0.2}, h2, {0.4, 0.4, 0.2}, referenceBettingConfig());
}

// instances.hpp:48-68
inline RiverInstance twentyCardInstance() {
    Deck deck;
    for (int r = 2; r <= 6; ++r)
        for (int s = 0; s < 4; ++s) deck.cards.emplace_back(r, s);
    Board board = Board::fromCode("2c2d4h5s6c");
    std::vector<Card> rest;
    for (const Card& c : deck.cards)
        if (!board.contains(c)) rest.push_back(c);
    std::vector<Hand> hands;
    for (size_t i = 0; i < rest.size(); ++i)
        for (size_t j = i + 1; j < rest.size(); ++j) hands.emplace_back(rest[i], rest[j]);
    std::vector<double> w(hands.size(), 1.0);
    return makeRiverInstance(board, hands, w, hands, w, referenceBettingConfig(), deck);
}

// instances.hpp:73-84
inline RiverInstance bluffingInstance() {
    Board board = Board::fromCode("2c2d2h3c3d");
    BettingConfig cfg;
    cfg.stack1 = cfg.stack2 = 40;
    cfg.potContribution = 10;
    cfg.menu1[FirstAction] = {1.0};
    cfg.allIn = false;
    std::vector<Hand> h1 = {Hand::fromCode("3h3s"), Hand::fromCode("4c5c")};
    std::vector<Hand> h2 = {Hand::fromCode("AcAd")};
    return makeRiverInstance(board, h1, {0.5, 0.5}, h2, {1.0}, cfg);
}

// instances.hpp:88-101
inline RiverInstance allTieInstance() {
    Board board = Board::fromCode("AsKsQsJsTs");
    BettingConfig cfg;
    cfg.stack1 = cfg.stack2 = 40;
    cfg.potContribution = 10;
    cfg.menu1[FirstAction] = {1.0};
    cfg.menu2[FacingCheck] = {1.0};
    cfg.allIn = false;
    std::vector<Hand> h1 = {Hand::fromCode("2c3c"), Hand::fromCode("4d5d")};
    std::vector<Hand> h2 = {Hand::fromCode("2h3h"), Hand::fromCode("4h5h")};
    return makeRiverInstance(board, h1, {0.5, 0.5}, h2, {0.5, 0.5}, cfg);
}

// instances.hpp:105-148 (same libstdc++ distributions => same draws)
inline RiverInstance randomSmallInstance(std::mt19937_64& rng, int handsPerSide = 0) {
    Deck full = Deck::standard52();
    for (int attempt = 0; attempt < 100; ++attempt) {
        std::shuffle(full.cards.begin(), full.cards.end(), rng);
        int deckSize = std::uniform_int_distribution<int>(12, 20)(rng);
        Deck deck;
        deck.cards.assign(full.cards.begin(), full.cards.begin() + deckSize);
        Board board({deck.cards[0], deck.cards[1], deck.cards[2], deck.cards[3], deck.cards[4]});
        std::vector<Card> rest(deck.cards.begin() + 5, deck.cards.end());
        std::vector<Hand> pairs;
        for (size_t i = 0; i < rest.size(); ++i)
            for (size_t j = i + 1; j < rest.size(); ++j) pairs.emplace_back(rest[i], rest[j]);
        auto draw = [&](int count) {
            std::vector<Hand> pool = pairs;
            std::shuffle(pool.begin(), pool.end(), rng);
            pool.resize(size_t(count));
            return pool;
        };
        int maxHands = std::min<int>(12, int(pairs.size()));
        if (handsPerSide > maxHands) continue;
        auto drawCount = [&] {
            return handsPerSide > 0 ? handsPerSide : std::uniform_int_distribution<int>(2, maxHands)(rng);
        };
        std::vector<Hand> h1 = draw(drawCount());
        std::vector<Hand> h2 = draw(drawCount());
        bool compatiblePair = false;
        for (const Hand& a : h1)
            for (const Hand& b : h2)
                if (!a.overlaps(b)) compatiblePair = true;
        if (!compatiblePair) continue;
        std::uniform_real_distribution<double> weight(0.1, 1.0);
        std::vector<double> w1, w2;
        for (size_t i = 0; i < h1.size(); ++i) w1.push_back(weight(rng));
        for (size_t i = 0; i < h2.size(); ++i) w2.push_back(weight(rng));
        return makeRiverInstance(board, h1, w1, h2, w2, referenceBettingConfig(), deck);
    }
    throw InvalidInputError("failed to draw a usable random instance");
}

// instances.hpp:159-194
inline RiverInstance benchInstance(uint64_t seed, int handsPerSide, int sharedCards = 0) {
    if (handsPerSide < 1) throw InvalidInputError("handsPerSide must be positive");
    if (sharedCards < 0 || sharedCards > 40) throw InvalidInputError("sharedCards out of range");
    std::mt19937_64 rng(seed);
    Deck deck = Deck::standard52();
    std::shuffle(deck.cards.begin(), deck.cards.end(), rng);
    Board board({deck.cards[0], deck.cards[1], deck.cards[2], deck.cards[3], deck.cards[4]});
    std::vector<Card> rest(deck.cards.begin() + 5, deck.cards.end());
    std::vector<Card> shared(rest.begin(), rest.begin() + sharedCards);
    size_t half = (rest.size() - size_t(sharedCards)) / 2;
    std::vector<Card> pool1(rest.begin() + sharedCards, rest.begin() + sharedCards + half);
    std::vector<Card> pool2(rest.begin() + sharedCards + half, rest.end());
    pool1.insert(pool1.end(), shared.begin(), shared.end());
    pool2.insert(pool2.end(), shared.begin(), shared.end());
    auto drawHands = [&](const std::vector<Card>& pool) {
        std::vector<Hand> pairs;
        for (size_t i = 0; i < pool.size(); ++i)
            for (size_t j = i + 1; j < pool.size(); ++j) pairs.emplace_back(pool[i], pool[j]);
        if (pairs.size() < size_t(handsPerSide)) throw InvalidInputError("pool too small for the requested hand count");
        std::shuffle(pairs.begin(), pairs.end(), rng);
        pairs.resize(size_t(handsPerSide));
        return pairs;
    };
    std::vector<Hand> h1 = drawHands(pool1), h2 = drawHands(pool2);
    std::uniform_real_distribution<double> weight(0.25, 1.0);
    std::vector<double> w1, w2;
    for (int i = 0; i < handsPerSide; ++i) w1.push_back(weight(rng));
    for (int i = 0; i < handsPerSide; ++i) w2.push_back(weight(rng));
    return makeRiverInstance(board, h1, w1, h2, w2, referenceBettingConfig());
}

// ---- synthetic configs of BASELINE.json / SURVEY.md §8(d) (not in the
// reference; defined here so the oracle and the product build the same games)

// 3-bet tree: menus {0.5, 1.0} in all contexts, all-in, raise cap 3.
inline BettingConfig threeBetConfig() {
    BettingConfig c;
    c.stack1 = c.stack2 = 18125;
    c.potContribution = 1875;
    for (int x = 0; x < kBetContexts; ++x) {
        c.menu1[x] = {0.5, 1.0};
        c.menu2[x] = {0.5, 1.0};
    }
    c.allIn = true;
    c.raiseCap = 3;
    return c;
}

// Full-range river on `board`: every hand of `deck` disjoint from the board,
// in canonical (ascending Hand) order; beliefs uniform_real(0.25,1) from
// mt19937_64(seed), player 1's all drawn before player 2's.
inline RiverInstance fullRangeRiver(const Board& board, const Deck& deck, uint64_t seed, const BettingConfig& cfg) {
    std::vector<Card> rest;
    for (const Card& c : deck.cards)
        if (!board.contains(c)) rest.push_back(c);
    std::sort(rest.begin(), rest.end());
    std::vector<Hand> hands;
    for (size_t i = 0; i < rest.size(); ++i)
        for (size_t j = i + 1; j < rest.size(); ++j) hands.emplace_back(rest[i], rest[j]);
    std::sort(hands.begin(), hands.end());
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> weight(0.25, 1.0);
    std::vector<double> w1, w2;
    for (size_t i = 0; i < hands.size(); ++i) w1.push_back(weight(rng));
    for (size_t i = 0; i < hands.size(); ++i) w2.push_back(weight(rng));
    return makeRiverInstance(board, hands, w1, hands, w2, cfg, deck);
}

}  // namespace kro
