// kr_host.hpp — host side of the B200 gradient oracle (namespace krh).
//
// Everything upstream of the hot path, restated from the reference kronriver
// library (paths under /root/reference/proj/include/kronriver/):
//   cards / 7-card evaluation      cards.hpp:17-329
//   betting skeleton               skeleton.hpp:44-387
//   river instance + payoff        kron.hpp:18-207
//   Technique A / B, postprocess   sparsify.hpp:17-406
//   instance JSON, bundles         instance_io.hpp, bundle_io.hpp, matrix_market.hpp
//   built-in games                 instances.hpp:19-194
// Factors are produced in the reference's storage order and bit-for-bit equal
// to it (tests/test_host_builder.py checks against the CPU oracle).  The
// design differs where the reference is O(m1 m2) in evaluator calls or sorts
// triplets: hand strengths are evaluated once per hand, and factors are
// generated directly in compressed order (Technique B's postprocessed form in
// closed form: chains of strength-distinct hands per showdown sequence).
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <random>
#include <string>
#include <vector>

namespace krh {

// ---------------------------------------------------------------- errors ---
enum Status { OK = 0, INVALID_INPUT = 1, PARSE = 2, IO = 3, GUARD = 4, DEGENERATE = 5, CONTRACT = 6 };
struct Error {
    int code;
    std::string msg;
};

// ---------------------------------------------------------------- cards ----
// Card id = (rank-2)*4 + suit, suits c d h s; id order == (rank, suit) order.
using CardId = uint8_t;
int cardFromCode(const std::string& code);  // throws Error
std::string cardCode(int id);

struct Hand {  // canonical: hi > lo (cards.hpp:60-95)
    uint8_t hi = 0, lo = 0;
    static Hand of(int a, int b);
    uint64_t mask() const { return (1ull << hi) | (1ull << lo); }
    std::string code() const { return cardCode(hi) + cardCode(lo); }
    bool operator<(const Hand& o) const { return hi != o.hi ? hi < o.hi : lo < o.lo; }
    bool operator==(const Hand& o) const { return hi == o.hi && lo == o.lo; }
};
Hand handFromCode(const std::string& code);

// Packed strength key of hand + 5 board cards (cards.hpp:223-304).
uint32_t strengthKey(const Hand& h, const std::array<int, 5>& board);

// -------------------------------------------------------------- skeleton ---
constexpr int kContexts = 5;
extern const char* const kContextNames[kContexts];

struct BettingConfig {  // skeleton.hpp:44-78
    double stack1 = 0, stack2 = 0, pot = 0;
    std::array<std::vector<double>, kContexts> menu[2];
    bool allIn = true;
    std::optional<int> raiseCap;
    void validate() const;
};

struct Action {
    int kind = 0;  // 0 check 1 fold 2 call 3 bet 4 raise 5 all-in
    double fraction = 0, target = 0;
    int seq = 0;
    bool terminal = false;
    int child = -1;
};
struct Node {
    int player = 0, context = 0, parentSeq[2] = {0, 0};
    double c1 = 0, c2 = 0;
    std::vector<Action> actions;
};
struct Terminal {
    bool fold = false;
    int folder = -1;
    double q1 = 0, q2 = 0;
    int seq1 = 0, seq2 = 0;
    std::string path;
};
struct Skeleton {  // skeleton.hpp:114-126
    BettingConfig config;
    std::vector<Node> nodes;
    std::vector<Terminal> terminals;
    int nseq[2] = {0, 0};
    std::vector<int> playerNodes[2];
};
Skeleton buildSkeleton(const BettingConfig& cfg);

// ------------------------------------------------------------ compressed ---
struct Compressed {  // Eigen-compatible compressed storage, inner ascending
    bool rowMajor = true;
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> outer{0};
    std::vector<int32_t> inner;
    std::vector<double> val;
    int64_t outerSize() const { return rowMajor ? rows : cols; }
    int64_t nnz() const { return int64_t(val.size()); }
};

// ---------------------------------------------------------------- payoff ---
struct Instance {  // RiverInstance (kron.hpp:18-37) + KronPayoff (104-132)
    std::array<int, 5> board{};
    std::vector<int> deck;
    std::vector<Hand> hands[2];     // strength-sorted, weakest first
    std::vector<double> mu[2];      // raw beliefs, sorted order
    std::vector<uint32_t> key[2];   // strength keys
    BettingConfig config;
    Skeleton sk;
    Compressed F, S;                // n1 x n2 CSR
    double beta = 0;
    std::vector<double> lambda[2];
    int m(int p) const { return int(hands[p].size()); }
    int n(int p) const { return sk.nseq[p]; }
    int64_t rows() const { return int64_t(m(0)) * n(0); }
    int64_t cols() const { return int64_t(m(1)) * n(1); }
    bool compatible(int i, int j) const { return (hands[0][i].mask() & hands[1][j].mask()) == 0; }
    // showdown sign gamma(h1_i, h2_j) for compatible pairs (cards.hpp:308-319)
    int sign(int i, int j) const {
        if (!compatible(i, j)) return 0;
        return key[0][i] > key[1][j] ? 1 : (key[0][i] < key[1][j] ? -1 : 0);
    }
};

// makeRiverInstance + assemble (kron.hpp:39-98, 134-166).
Instance makeInstance(const std::array<int, 5>& board, std::vector<int> deck, std::vector<Hand> h1,
                      std::vector<double> w1, std::vector<Hand> h2, std::vector<double> w2, const BettingConfig& cfg);
int64_t densePayoffNonzeros(const Instance& in);  // kron.hpp:198-207

// Built-in games (instances.hpp) and the synthetic configs of SURVEY §8(d).
Instance goldenInstance();
Instance twentyCardInstance();
Instance bluffingInstance();
Instance allTieInstance();
Instance randomSmallInstance(std::mt19937_64& rng, int handsPerSide);
Instance benchInstance(uint64_t seed, int handsPerSide, int sharedCards);
BettingConfig referenceBettingConfig();
BettingConfig threeBetConfig();
Instance fullRangeRiver(const std::string& board, int deckKind, uint64_t seed, const BettingConfig& cfg);
Instance readInstanceJson(const std::string& path);

// --------------------------------------------------------------- factors ---
struct Factors {  // Sparsification (sparsify.hpp:110-121)
    Compressed Ahat, U, M, V;  // CSR, CSR, CSC, CSC
    int technique = 1;          // 0 = A, 1 = B
    bool postprocessed = false;
    int32_t n1 = 0, n2 = 0;     // layout hint for the engine
    int64_t rows() const { return Ahat.rows; }
    int64_t cols() const { return Ahat.cols; }
    int64_t k() const { return M.rows; }
};

Factors techniqueB(const Instance& in);          // sparsify.hpp:246-312
Factors techniqueBPost(const Instance& in);      // == postprocess(techniqueB(in)), closed form
Factors techniqueA(const Instance& in, int peelIters);  // sparsifyW + techniqueA (68-103, 165-240)
Factors postprocess(const Factors& s);           // sparsify.hpp:318-406
void validate(const Factors& s);                 // sparsify.hpp:133-145

void writeBundle(const Factors& s, const std::string& dir);
Factors readBundle(const std::string& dir);

}  // namespace krh
