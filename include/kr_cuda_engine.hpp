// kr_cuda_engine.hpp — C++ host adapter over the kr_* C ABI.
//
// The reference's solver reaches the payoff only through
//   class GradientEngine { virtual Vec Ax(const Vec&) const = 0;
//                          virtual Vec ATx(const Vec&) const = 0;
//                          virtual int64_t flops() const; }   (solver.hpp:21-27)
// CudaEngine below is that interface over libkrcuda.so (the B200 engine), and
// CudaSolver is dcfrSolve (solver.hpp:343-404) on the device.  Error codes
// coming back through the ABI are rethrown as exceptions carrying the
// reference's stable codes (errors.hpp:11-58).  Header-only; link
// libkrcuda.so.  INTEGRATION.md shows the same adapter written against
// kronriver's Eigen types.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "kr_engine.h"

namespace krb200 {

struct Error : std::runtime_error {
    std::string code;
    Error(std::string c, const std::string& m) : std::runtime_error(m), code(std::move(c)) {}
};

inline const char* statusCode(int s) {
    switch (s) {
        case KR_INVALID_INPUT: return "INVALID_INPUT";
        case KR_PARSE: return "PARSE";
        case KR_IO: return "IO";
        case KR_GUARD_EXCEEDED: return "GUARD_EXCEEDED";
        case KR_DEGENERATE_BELIEFS: return "DEGENERATE_BELIEFS";
        case KR_CONTRACT: return "CONTRACT";
        case KR_NO_DEVICE: return "NO_DEVICE";
        default: return "CUDA";
    }
}

inline void check(int status) {
    if (status != KR_OK) {
        int code = 0;
        const char* msg = kr_last_error(&code);
        throw Error(statusCode(status), msg ? msg : "");
    }
}

using Vec = std::vector<double>;

class GradientEngine {  // solver.hpp:21-27
public:
    virtual ~GradientEngine() = default;
    virtual Vec Ax(const Vec& x2) const = 0;
    virtual Vec ATx(const Vec& x1) const = 0;
    virtual int64_t flops() const { return 0; }
};

class CudaEngine : public GradientEngine {
public:
    // One Sparsification, or several boards stacked block-diagonally.
    explicit CudaEngine(const kr_factors& f, int device = 0) { check(kr_engine_create(&f, device, 0, &e_)); }
    CudaEngine(const std::vector<kr_factors>& boards, int device = 0) {
        check(kr_engine_create_boards(boards.data(), int(boards.size()), device, 0, &e_));
    }
    // Engines over KronPayoff pieces: the implicit Kronecker engine
    // (kr_engine_create_kron, products within 1e-12) or the Kronecker-factored
    // one (kr_engine_create_kfactored: Technique B post from its Kronecker
    // factors, products bitwise those of the factored engine).
    enum class Kind { Implicit, KFactored };
    explicit CudaEngine(const std::vector<kr_kron_board>& boards, int device = 0, Kind kind = Kind::Implicit) {
        if (kind == Kind::KFactored) check(kr_engine_create_kfactored(boards.data(), int(boards.size()), device, 0, &e_));
        else check(kr_engine_create_kron(boards.data(), int(boards.size()), device, 0, &e_));
    }
    ~CudaEngine() override {
        if (e_) kr_engine_destroy(e_);
    }
    CudaEngine(const CudaEngine&) = delete;
    CudaEngine& operator=(const CudaEngine&) = delete;

    int64_t rows() const { return dim(0); }
    int64_t cols() const { return dim(1); }
    kr_engine* handle() const { return e_; }

    Vec Ax(const Vec& x2) const override {  // engine.hpp:58-93
        Vec y(static_cast<size_t>(rows()));
        check(kr_engine_ax(e_, x2.data(), int64_t(x2.size()), y.data(), int64_t(y.size())));
        return y;
    }
    Vec ATx(const Vec& x1) const override {  // engine.hpp:96-133
        Vec x(static_cast<size_t>(cols()));
        check(kr_engine_atx(e_, x1.data(), int64_t(x1.size()), x.data(), int64_t(x.size())));
        return x;
    }
    int64_t flops() const override { return kr_engine_flops(e_); }

private:
    int64_t dim(int i) const {
        int64_t d[8];
        check(kr_engine_dims(e_, d));
        return d[i];
    }
    kr_engine* e_ = nullptr;
};

struct DcfrParams {  // solver.hpp:101-109 (+ rule: KR_RULE_*, 0 = the reference's DCFR)
    double alpha = 1.5, beta = 0.0, gamma = 2.0;
    int maxIters = 1000;
    double targetExploitability = 0.0;
    int checkpointEvery = 50;
    int rule = KR_RULE_DCFR;
};

struct TracePoint {
    int iteration = 0;
    double exploitability = 0;
};

struct DcfrResult {  // solver.hpp:133-140
    Vec avg1, avg2;
    int iterations = 0;
    double exploitability = 0;
    std::vector<TracePoint> trace;
    int64_t gradientFlops = 0;
    double deviceSeconds = 0;
};

// Treeplex of one player: parent sequence per decision node (preorder), the
// action ranges and their 1-based sequence ids (skeleton.hpp:89-126).
struct Treeplex {
    int32_t nSeq = 0;
    std::vector<int32_t> parent, actionPtr, actionSeq;
    kr_treeplex view() const {
        return kr_treeplex{nSeq, int32_t(parent.size()), parent.data(), actionPtr.data(), actionSeq.data()};
    }
};

class CudaSolver {
public:
    CudaSolver(CudaEngine& eng, const Treeplex& p1, const Treeplex& p2, const std::vector<int32_t>& hands1,
               const std::vector<int32_t>& hands2, double pot)
        : rows_(eng.rows()), cols_(eng.cols()), nboards_(int(hands1.size())) {
        const kr_treeplex t1 = p1.view(), t2 = p2.view();
        check(kr_solver_create(eng.handle(), &t1, &t2, nboards_, hands1.data(), hands2.data(), pot, &s_));
    }
    ~CudaSolver() {
        if (s_) kr_solver_destroy(s_);
    }
    CudaSolver(const CudaSolver&) = delete;
    CudaSolver& operator=(const CudaSolver&) = delete;

    // Board sharding (kr_solver_set_comm): this solver holds c's rank's shard
    // of boardsPerRank; runs then cover every board of every rank.
    void setComm(kr_comm* c, const std::vector<int32_t>& boardsPerRank) {
        check(kr_solver_set_comm(s_, c, c ? boardsPerRank.data() : nullptr));
    }

    DcfrResult run(const DcfrParams& p) {  // dcfrSolve (solver.hpp:343-404)
        const int cap = p.maxIters / (p.checkpointEvery > 0 ? p.checkpointEvery : 1) + 2;
        std::vector<int32_t> it(static_cast<size_t>(cap));
        std::vector<double> ex(static_cast<size_t>(cap));
        DcfrResult out;
        out.avg1.resize(size_t(rows_));
        out.avg2.resize(size_t(cols_));
        kr_dcfr_params prm{p.alpha, p.beta, p.gamma, p.maxIters, p.targetExploitability, p.checkpointEvery, p.rule};
        kr_dcfr_result r{};
        r.trace_cap = cap;
        r.trace_iter = it.data();
        r.trace_expl = ex.data();
        r.avg1 = out.avg1.data();
        r.avg2 = out.avg2.data();
        check(kr_solver_run(s_, &prm, &r));
        out.iterations = r.iterations;
        out.exploitability = r.exploitability;
        out.gradientFlops = r.gradient_flops;
        out.deviceSeconds = r.seconds;
        for (int i = 0; i < r.trace_len && i < cap; ++i) out.trace.push_back({it[size_t(i)], ex[size_t(i)]});
        return out;
    }

    // bestResponseValue (solver.hpp:292-321)
    double bestResponseValue(int player, const Vec& opp) {
        double v = 0;
        check(kr_solver_best_response(s_, player, opp.data(), int64_t(opp.size()), &v, nullptr));
        return v;
    }

private:
    int64_t rows_, cols_;
    int nboards_;
    kr_solver* s_ = nullptr;
};

}  // namespace krb200
