// krb200 — C++ command-line driver over the product's two C ABIs, mirroring
// the reference CLI's sparsify / solve subcommands (tools/main.cpp:98-162)
// with the gradient oracle and the solver step on the B200:
//
//   krb200 sparsify --instance F [--technique a|b] [--out DIR]
//   krb200 solve    --instance F [--bundle DIR] [--technique a|b] [--iters N]
//                   [--target-expl X] [--checkpoint-every N] [--out DIR]
//                   [--engine factored|implicit] [--rule dcfr|cfr+|prm+]
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
    int iters = 1000, checkpointEvery = 50;
    double targetExpl = 0;
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

}  // namespace

int main(int argc, char** argv) {
    Options o;
    if (argc < 2) {
        std::fprintf(stderr, "usage: krb200 {sparsify|solve} --instance F [options]\n");
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
        else if (k == "--engine") o.engine = v;
        else if (k == "--rule") o.rule = v;
        else {
            std::fprintf(stderr, "unknown option %s\n", k.c_str());
            return 1;
        }
    }
    try {
        if (o.cmd == "sparsify") return runSparsify(o);
        if (o.cmd == "solve") return runSolve(o);
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
