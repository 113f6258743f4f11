// krb200 — C++ command-line driver over the product's two C ABIs, mirroring
// the reference CLI's sparsify / solve subcommands (tools/main.cpp:98-162)
// with the gradient oracle and the solver step on the B200:
//
//   krb200 sparsify --instance F [--technique a|b] [--out DIR]
//   krb200 solve    --instance F [--bundle DIR] [--technique a|b] [--iters N]
//                   [--target-expl X] [--checkpoint-every N] [--out DIR]
//                   [--engine factored|implicit] [--rule dcfr|cfr+|prm+]
//   krb200 solve-turn [--turn Ks7d4c2h] [--boards 48] [--gpus N] [--iters N]
//                   [--checkpoint-every N] [--engine kfactored|factored|implicit]
//
// solve-turn: config 3, a turn's river boards under a
// uniform chance root, boards sharded contiguously over N GPUs of this node
// (one host thread and one solver per GPU, an NCCL communicator over the
// device list: kr_comm_init_all); the checkpoint values are all-gathered and
// folded in board order, so the trace is bitwise the one-GPU trace.
//
// --engine implicit applies the payoff without factors (kr_engine_create_kron);
// --rule selects the update rule (dcfr is the reference's; cfr+ and prm+ are
// presets with alpha = +inf, beta = -inf, gamma = 1).
//
// Errors print `error code=... msg="..."` and exit 2, as the reference does
// (main.cpp:420-426).
#include <chrono>
#include <cmath>
#include <memory>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <vector>

#include "kr_cuda_engine.hpp"
#include "kr_host.h"

namespace {

struct Options {
    std::string cmd, instance, bundle, technique = "b", out = "out", engine = "factored", rule = "dcfr";
    std::string turn = "Ks7d4c2h";
    int iters = 1000, checkpointEvery = 50, boards = 48, gpus = 1;
    double targetExpl = 0;
    bool engineSet = false;
};

void hcheck(int status) {
    if (status != 0) {
        int code = 0;
        const char* msg = krh_last_error(&code);
        throw krb200::Error(krb200::statusCode(status), msg ? msg : "");
    }
}

struct Instance {
    krh_instance* h = nullptr;
    int64_t d[16] = {};
    explicit Instance(const std::string& path) {
        hcheck(krh_instance_from_json(path.c_str(), &h));
        hcheck(krh_instance_dims(h, d));
    }
    explicit Instance(krh_instance* owned) : h(owned) { hcheck(krh_instance_dims(h, d)); }
    ~Instance() { krh_instance_free(h); }
    krb200::Treeplex treeplex(int p) const {
        krb200::Treeplex t;
        t.nSeq = int32_t(d[2 + p]);
        t.parent.resize(size_t(d[7 + p]));
        t.actionPtr.resize(size_t(d[7 + p]) + 1);
        t.actionSeq.resize(size_t(d[14 + p]));
        hcheck(krh_instance_treeplex(h, p, t.parent.data(), t.actionPtr.data(), t.actionSeq.data()));
        return t;
    }
};

struct Factors {
    krh_factors* h = nullptr;
    ~Factors() { krh_factors_free(h); }
    kr_factors view() const {
        kr_factors v;
        hcheck(krh_factors_view(h, &v));
        return v;
    }
    void dims(int64_t out[9]) const { hcheck(krh_factors_dims(h, out)); }
};

int runSparsify(const Options& o) {
    Instance inst(o.instance);
    Factors f;
    const auto t0 = std::chrono::steady_clock::now();
    hcheck(krh_sparsify(inst.h, o.technique == "a" ? 0 : 1, 1, 1000, &f.h));
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    hcheck(krh_bundle_write(f.h, o.out.c_str()));
    int64_t d[9];
    f.dims(d);
    const long long dense = krh_dense_nnz(inst.h), size = d[3] + d[4] + d[5] + d[6];
    std::printf("%-20s %14s %10s %9s %8s\n", "game", "unsparsified", "size", "time", "ratio");
    std::printf("%-20s %14lld %10lld %8.3fs %8.2f\n", std::filesystem::path(o.instance).stem().string().c_str(),
                dense, size, secs, size ? double(dense) / double(size) : 0.0);
    std::printf("factors: ahat=%lld u=%lld m=%lld v=%lld k=%lld technique=%s postprocessed=1\n", (long long)d[3],
                (long long)d[4], (long long)d[5], (long long)d[6], (long long)d[2], d[7] == 0 ? "a" : "b");
    std::printf("bundle: %s\n", o.out.c_str());
    return 0;
}

int runSolve(const Options& o) {
    Instance inst(o.instance);
    Factors f;
    if (o.engine != "factored" && o.engine != "implicit")
        throw krb200::Error("INVALID_INPUT", "--engine must be factored or implicit");
    if (o.rule != "dcfr" && o.rule != "cfr+" && o.rule != "prm+")
        throw krb200::Error("INVALID_INPUT", "--rule must be dcfr, cfr+ or prm+");
    if (o.engine == "implicit") {
    } else if (!o.bundle.empty()) {
        hcheck(krh_bundle_read(o.bundle.c_str(), &f.h));
        int64_t d[9];
        f.dims(d);
        if (d[0] != inst.d[4] || d[1] != inst.d[5])
            throw krb200::Error("INVALID_INPUT", "bundle shape does not match the instance");
    } else {
        hcheck(krh_sparsify(inst.h, o.technique == "a" ? 0 : 1, 1, 1000, &f.h));
    }
    std::unique_ptr<krb200::CudaEngine> engp;
    if (o.engine == "implicit") {
        kr_kron_board kb;
        hcheck(krh_instance_kron_view(inst.h, &kb));
        engp = std::make_unique<krb200::CudaEngine>(std::vector<kr_kron_board>{kb});
    } else {
        engp = std::make_unique<krb200::CudaEngine>(f.view());
    }
    krb200::CudaEngine& eng = *engp;
    krb200::CudaSolver solver(eng, inst.treeplex(0), inst.treeplex(1), {int32_t(inst.d[0])}, {int32_t(inst.d[1])},
                              krh_instance_pot(inst.h));
    krb200::DcfrParams p;
    if (o.rule != "dcfr") {
        p.alpha = HUGE_VAL;
        p.beta = -HUGE_VAL;
        p.gamma = 1.0;
        p.rule = o.rule == "cfr+" ? KR_RULE_CFRP : KR_RULE_PRMP;
    }
    p.maxIters = o.iters;
    p.targetExploitability = o.targetExpl;
    p.checkpointEvery = o.checkpointEvery;
    const krb200::DcfrResult r = solver.run(p);
    std::filesystem::create_directories(o.out);
    const std::string trace = o.out + "/trace.csv", profile = o.out + "/profile.json";
    if (std::FILE* t = std::fopen(trace.c_str(), "w")) {  // solver.hpp:121-131 format
        std::fprintf(t, "iteration,seconds,exploitability\n");
        for (const auto& q : r.trace) std::fprintf(t, "%d,%.6f,%.12g\n", q.iteration, 0.0, q.exploitability);
        std::fclose(t);
    }
    if (std::FILE* pf = std::fopen(profile.c_str(), "w")) {
        std::fprintf(pf, "{\n  \"exploitability\": %.17g,\n  \"gradient_flops\": %lld,\n  \"iterations\": %d,\n",
                     r.exploitability, (long long)r.gradientFlops, r.iterations);
        std::fprintf(pf, "  \"schema_version\": 1,\n  \"device_seconds\": %.6f\n}\n", r.deviceSeconds);
        std::fclose(pf);
    }
    std::printf("solve: iterations=%d exploitability=%.12g gradient_flops=%lld trace=%s profile=%s\n", r.iterations,
                r.exploitability, (long long)r.gradientFlops, trace.c_str(), profile.c_str());
    if (o.engine != "factored" || o.rule != "dcfr")
        std::printf("engine=%s rule=%s device_seconds=%.6f\n", o.engine.c_str(), o.rule.c_str(), r.deviceSeconds);
    return 0;
}

// The river cards under a turn and their belief seeds (config 3: seed 1000 +
// card id, as paper_2112_03804_b200.host.turn_boards).
std::vector<std::pair<std::string, uint64_t>> turnBoards(const std::string& turn, int n) {
    const std::string ranks = "23456789TJQKA", suits = "cdhs";
    std::vector<std::pair<std::string, uint64_t>> out;
    for (size_t r = 0; r < ranks.size(); ++r)
        for (size_t s = 0; s < suits.size(); ++s) {
            const std::string c = std::string(1, ranks[r]) + suits[s];
            bool used = false;
            for (size_t i = 0; i + 1 < turn.size(); i += 2) used = used || turn.substr(i, 2) == c;
            if (!used && int(out.size()) < n) out.push_back({c, 1000 + uint64_t(r * 4 + s)});
        }
    return out;
}

int runSolveTurn(const Options& o) {
    const std::string engine = o.engineSet ? o.engine : "kfactored";
    if (engine != "factored" && engine != "kfactored" && engine != "implicit")
        throw krb200::Error("INVALID_INPUT", "--engine must be kfactored, factored or implicit");
    int ndev = kr_device_count();
    if (o.gpus < 1 || o.gpus > ndev)
        throw krb200::Error("INVALID_INPUT", "--gpus must be between 1 and the visible device count");
    const auto specs = turnBoards(o.turn, o.boards);
    const int nb = int(specs.size()), world = o.gpus;
    std::vector<int32_t> bpr(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) bpr[size_t(r)] = nb / world + (r < nb % world ? 1 : 0);
    std::vector<kr_comm*> comms(static_cast<size_t>(world), nullptr);
    if (world > 1) {
        std::vector<int> devs(static_cast<size_t>(world));
        for (int r = 0; r < world; ++r) devs[size_t(r)] = r;
        krb200::check(kr_comm_init_all(world, devs.data(), comms.data()));
    }
    std::vector<krb200::DcfrResult> res(static_cast<size_t>(world));
    std::vector<std::string> errs(static_cast<size_t>(world));
    auto rankMain = [&](int r) {
        try {
            const int b0 = [&] { int s = 0; for (int q = 0; q < r; ++q) s += bpr[size_t(q)]; return s; }();
            std::vector<std::unique_ptr<Instance>> insts;
            std::vector<Factors> fs(static_cast<size_t>(bpr[size_t(r)]));
            std::vector<kr_kron_board> kb;
            std::vector<kr_factors> fv;
            std::vector<int32_t> h1, h2;
            for (int b = b0; b < b0 + bpr[size_t(r)]; ++b) {
                const std::string board = o.turn + specs[size_t(b)].first;
                krh_instance* h = nullptr;
                hcheck(krh_instance_builtin("river_full", specs[size_t(b)].second, 0, 0, board.c_str(), 52, 3, &h));
                auto in = std::make_unique<Instance>(h);
                kr_kron_board k;
                hcheck(krh_instance_kron_view(in->h, &k));
                kb.push_back(k);
                if (engine == "factored") {
                    hcheck(krh_sparsify(in->h, 1, 1, 1000, &fs[size_t(b - b0)].h));
                    fv.push_back(fs[size_t(b - b0)].view());
                }
                h1.push_back(int32_t(in->d[0]));
                h2.push_back(int32_t(in->d[1]));
                insts.push_back(std::move(in));
            }
            std::unique_ptr<krb200::CudaEngine> eng;
            if (engine == "factored") eng = std::make_unique<krb200::CudaEngine>(fv, r);
            else eng = std::make_unique<krb200::CudaEngine>(kb, r, engine == "kfactored"
                                                                     ? krb200::CudaEngine::Kind::KFactored
                                                                     : krb200::CudaEngine::Kind::Implicit);
            krb200::CudaSolver solver(*eng, insts[0]->treeplex(0), insts[0]->treeplex(1), h1, h2,
                                      krh_instance_pot(insts[0]->h));
            if (world > 1) solver.setComm(comms[size_t(r)], bpr);
            krb200::DcfrParams p;
            p.maxIters = o.iters;
            p.checkpointEvery = o.checkpointEvery;
            res[size_t(r)] = solver.run(p);
        } catch (const std::exception& e) {
            errs[size_t(r)] = e.what();
        }
    };
    std::vector<std::thread> th;
    for (int r = 0; r < world; ++r) th.emplace_back(rankMain, r);
    for (auto& t : th) t.join();
    for (kr_comm* c : comms)
        if (c) kr_comm_destroy(c);
    for (const auto& e : errs)
        if (!e.empty()) throw krb200::Error("CUDA", e);
    const krb200::DcfrResult& r = res[0];
    double secs = 0;
    for (const auto& q : res) secs = std::max(secs, q.deviceSeconds);
    for (const auto& q : r.trace) std::printf("checkpoint iteration=%d exploitability=%.17g\n", q.iteration, q.exploitability);
    std::printf("solve-turn: turn=%s boards=%d gpus=%d engine=%s iterations=%d exploitability=%.17g "
                "device_seconds=%.6f iters_per_s=%.1f\n",
                o.turn.c_str(), nb, world, engine.c_str(), r.iterations, r.exploitability, secs,
                secs > 0 ? r.iterations / secs : 0.0);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    Options o;
    if (argc < 2) {
        std::fprintf(stderr, "usage: krb200 {sparsify|solve|solve-turn} [options]\n");
        return 1;
    }
    o.cmd = argv[1];
    for (int i = 2; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--instance") o.instance = v;
        else if (k == "--bundle") o.bundle = v;
        else if (k == "--technique") o.technique = v;
        else if (k == "--out") o.out = v;
        else if (k == "--iters") o.iters = std::atoi(v.c_str());
        else if (k == "--target-expl") o.targetExpl = std::atof(v.c_str());
        else if (k == "--checkpoint-every") o.checkpointEvery = std::atoi(v.c_str());
        else if (k == "--engine") {
            o.engine = v;
            o.engineSet = true;
        } else if (k == "--turn") o.turn = v;
        else if (k == "--boards") o.boards = std::atoi(v.c_str());
        else if (k == "--gpus") o.gpus = std::atoi(v.c_str());
        else if (k == "--rule") o.rule = v;
        else {
            std::fprintf(stderr, "unknown option %s\n", k.c_str());
            return 1;
        }
    }
    try {
        if (o.cmd == "sparsify") return runSparsify(o);
        if (o.cmd == "solve") return runSolve(o);
        if (o.cmd == "solve-turn") return runSolveTurn(o);
        std::fprintf(stderr, "unknown subcommand %s\n", o.cmd.c_str());
        return 1;
    } catch (const krb200::Error& e) {
        std::fprintf(stderr, "error code=%s msg=\"%s\"\n", e.code.c_str(), e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error code=INTERNAL msg=\"%s\"\n", e.what());
        return 3;
    }
}
