// C++ host API of the B200-native core, mirroring the reference's
// include/sskm/engine.hpp entry points over the C-ABI in sskm_b200.h.
//
//   reference (proj/include/sskm/engine.hpp)        here
//   RunConfig                    (:20-41)           sskm_b200::RunConfig (same fields + device, seeds)
//   IterationStats               (:43-57)           sskm_b200::IterationStats (= sskm_iteration_stats)
//   ClusteringResult             (:132-142)         sskm_b200::ClusteringResult (+ Cᵀ centroids)
//   run(const CorpusMatrix&, const RunConfig&)  (:148)    sskm_b200::run(const CsrCorpus&, const RunConfig&)
//   compute_centroids / detect_unchanged (:93, :106)       Engine::update()
//   assign (:124)                                          Engine::assign()
//
// Errors keep the reference's types: configuration / shape problems throw
// std::invalid_argument (engine.cpp:47-64), device failures std::runtime_error.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sskm_b200.h"

namespace sskm_b200 {

enum class Mode { kBaseline = SSKM_MODE_BASELINE, kNcc = SSKM_MODE_NCC, kNccIndex = SSKM_MODE_NCC_INDEX };

inline Mode parse_mode(const std::string& name) {
    if (name == "baseline") return Mode::kBaseline;
    if (name == "ncc") return Mode::kNcc;
    if (name == "ncc+index") return Mode::kNccIndex;
    throw std::invalid_argument("unknown mode '" + name + "' (expected baseline, ncc, or ncc+index)");
}

struct RunConfig {
    std::uint32_t k = 2;
    Mode mode = Mode::kBaseline;
    std::vector<double> lambdas{0.1, 0.25, 0.4, 0.6};
    double conv_sq_dist = 0.0001;
    double ncc_epsilon = 0.0;
    std::uint32_t index_activation_threshold = 100;
    std::uint32_t max_iters = 100;
    std::uint64_t seed = 0;
    std::uint32_t threads = 0;   // accepted for API parity; the GPU grid replaces it
    int device = 0;              // CUDA device ordinal
    std::vector<int> devices;    // several GPUs of this node (documents sharded; needs init_seeds)
    std::vector<std::uint32_t> init_seeds;  // empty: k-means++ (engine.cpp:66-130)

    sskm_run_config c() const {
        sskm_run_config r{};
        r.k = k;
        r.mode = static_cast<std::int32_t>(mode);
        r.lambdas = lambdas.empty() ? nullptr : lambdas.data();
        r.n_lambdas = static_cast<std::uint32_t>(lambdas.size());
        r.conv_sq_dist = conv_sq_dist;
        r.ncc_epsilon = ncc_epsilon;
        r.index_activation_threshold = index_activation_threshold;
        r.max_iters = max_iters;
        r.seed = seed;
        r.threads = threads;
        r.device = device;
        return r;
    }

    // RunConfig::validate (engine.cpp:47-64)
    void validate(std::size_t n_docs) const;
};

using IterationStats = sskm_iteration_stats;

enum class StopReason { kNoReassignments = 0, kCentroidDrift = 1, kMaxIterations = 2 };

inline const char* stop_reason_name(StopReason r) {
    switch (r) {
        case StopReason::kNoReassignments: return "no_reassignments";
        case StopReason::kCentroidDrift: return "centroid_drift";
        case StopReason::kMaxIterations: return "max_iterations";
    }
    return "?";
}

// Unit-length document rows as CSR (corpus.hpp:26-32), fp32 values.
struct CsrCorpus {
    std::vector<std::int64_t> indptr{0};
    std::vector<std::int32_t> indices;
    std::vector<float> values;
    std::uint32_t dims = 0;
    std::size_t size() const { return indptr.size() - 1; }
};

struct ClusteringResult {
    std::vector<std::uint32_t> assignments;
    std::vector<double> sims;
    std::vector<float> centroids_t;  // d × k row-major (Cᵀ)
    std::vector<IterationStats> iterations;
    double objective = 0.0;
    StopReason stop_reason = StopReason::kMaxIterations;

    std::uint64_t total_dot_products() const {
        std::uint64_t t = 0;
        for (const auto& it : iterations) t += it.dot_products;
        return t;
    }
};

inline void check(int rc) {
    if (rc == SSKM_OK) return;
    const std::string msg = sskm_last_error();
    if (rc == SSKM_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void RunConfig::validate(std::size_t n_docs) const {
    const sskm_run_config r = c();
    check(sskm_validate(&r, n_docs));
}

// sskm::run (engine.hpp:148) on one GPU.
inline ClusteringResult run(const CsrCorpus& data, const RunConfig& cfg, bool with_centroids = true) {
    const sskm_run_config r = cfg.c();
    check(sskm_validate(&r, data.size()));
    if (!cfg.init_seeds.empty() && cfg.init_seeds.size() != cfg.k)
        throw std::invalid_argument("init_seeds must hold exactly k document ids");
    ClusteringResult out;
    out.assignments.resize(data.size());
    out.sims.resize(data.size());
    if (with_centroids) out.centroids_t.resize(static_cast<std::size_t>(data.dims) * cfg.k);
    out.iterations.resize(cfg.max_iters);
    std::uint32_t n_it = 0;
    std::int32_t stop = 0;
    if (!cfg.devices.empty()) {  // multi-device context (sskm_multi_*): bitwise the single-GPU result
        if (cfg.init_seeds.empty()) throw std::invalid_argument("a multi-device run needs init_seeds");
        check(sskm_cluster_csr_multi(&r, static_cast<std::int32_t>(cfg.devices.size()), cfg.devices.data(),
                                     static_cast<std::int64_t>(data.size()), data.dims, data.indptr.data(),
                                     data.indices.data(), data.values.data(), cfg.init_seeds.data(),
                                     out.assignments.data(), out.sims.data(),
                                     with_centroids ? out.centroids_t.data() : nullptr, out.iterations.data(),
                                     cfg.max_iters, &n_it, &stop, &out.objective));
    } else {
        check(sskm_cluster_csr(&r, static_cast<std::int64_t>(data.size()), data.dims, data.indptr.data(),
                               data.indices.data(), data.values.data(),
                               cfg.init_seeds.empty() ? nullptr : cfg.init_seeds.data(), out.assignments.data(),
                               out.sims.data(), with_centroids ? out.centroids_t.data() : nullptr,
                               out.iterations.data(), cfg.max_iters, &n_it, &stop, &out.objective));
    }
    out.iterations.resize(n_it);
    out.stop_reason = static_cast<StopReason>(stop);
    return out;
}

// Per-iteration handle (the reference tests' Stepper shape, test_engine.cpp:54-100).
class Engine {
public:
    explicit Engine(int device = 0) { check(sskm_open(device, &ctx_)); }
    ~Engine() {
        if (ctx_) sskm_close(ctx_);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void upload(const CsrCorpus& d) {
        check(sskm_upload_csr(ctx_, static_cast<std::int64_t>(d.size()), d.dims, d.indptr.data(), d.indices.data(),
                              d.values.data(), 0, static_cast<std::int64_t>(d.size())));
        n_ = d.size();
        dims_ = d.dims;
    }
    void configure(const RunConfig& cfg) {
        const sskm_run_config r = cfg.c();
        check(sskm_configure(ctx_, &r));
        k_ = cfg.k;
    }
    void init_from_seeds(const std::vector<std::uint32_t>& seeds) { check(sskm_init_from_seeds(ctx_, seeds.data())); }
    std::vector<std::uint32_t> init_kmeanspp(std::uint64_t seed) {
        std::vector<std::uint32_t> s(k_);
        check(sskm_init_kmeanspp(ctx_, seed, s.data()));
        return s;
    }
    IterationStats update() { return call(sskm_update); }
    IterationStats assign() { return call(sskm_assign); }
    IterationStats step() { return call(sskm_step); }
    /// n iterations back to back, no stop rules (fixed-length runs).
    std::vector<IterationStats> step_n(std::uint32_t n) {
        std::vector<IterationStats> st(n);
        check(sskm_step_n(ctx_, n, st.data()));
        return st;
    }
    void state(std::vector<std::uint32_t>& a, std::vector<double>& sims, std::vector<std::uint8_t>& unchanged) {
        a.resize(n_);
        sims.resize(n_);
        unchanged.resize(k_);
        check(sskm_get_state(ctx_, a.data(), sims.data(), unchanged.data()));
    }
    std::vector<float> centroids_t() {
        std::vector<float> c(static_cast<std::size_t>(dims_) * k_);
        check(sskm_get_centroids(ctx_, c.data()));
        return c;
    }
    sskm_ctx* raw() { return ctx_; }

private:
    template <class F>
    IterationStats call(F f) {
        IterationStats st{};
        check(f(ctx_, &st));
        return st;
    }
    sskm_ctx* ctx_ = nullptr;
    std::size_t n_ = 0;
    std::uint32_t dims_ = 0, k_ = 0;
};

}  // namespace sskm_b200
