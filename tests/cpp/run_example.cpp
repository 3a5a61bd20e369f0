// C++ drop-in example: the reference's sskm::run call shape on the B200 core.
// Usage: run_example validate | run <k> | multi <k>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>

#include "sskm_b200.hpp"

static sskm_b200::CsrCorpus toy(std::size_t n, std::uint32_t d, unsigned seed) {
    std::mt19937 g(seed);
    sskm_b200::CsrCorpus c;
    c.dims = d;
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint32_t base = static_cast<std::uint32_t>((i % 4) * (d / 4));
        double norm = 0;
        std::vector<float> w;
        for (std::uint32_t t = 0; t < 5; ++t) {
            w.push_back(0.5f + (g() % 100) / 100.0f);
            norm += double(w.back()) * w.back();
        }
        for (std::uint32_t t = 0; t < 5; ++t) {
            c.indices.push_back(static_cast<std::int32_t>(base + t * 3));
            c.values.push_back(static_cast<float>(w[t] / std::sqrt(norm)));
        }
        c.indptr.push_back(static_cast<std::int64_t>(c.indices.size()));
    }
    return c;
}

int main(int argc, char** argv) {
    const char* what = argc > 1 ? argv[1] : "run";
    auto data = toy(400, 64, 7);
    sskm_b200::RunConfig cfg;
    if (!std::strcmp(what, "validate")) {
        try {
            cfg.k = 1;
            cfg.validate(data.size());
        } catch (const std::invalid_argument& e) {
            std::printf("invalid_argument: %s\n", e.what());
            return 2;  // the reference CLI's usage-error exit code (sskm_main.cpp:334-336)
        }
        return 0;
    }
    cfg.k = argc > 2 ? static_cast<std::uint32_t>(std::atoi(argv[2])) : 4;
    cfg.mode = sskm_b200::parse_mode("ncc");
    cfg.init_seeds = {0, 1, 2, 3};
    if (!std::strcmp(what, "multi")) cfg.devices = {0, 0};  // two document shards (on one device here)
    try {
        auto r = sskm_b200::run(data, cfg);
        std::printf("iterations=%zu stop=%s objective=%.12f dots=%llu a0=%u a1=%u a2=%u a3=%u\n", r.iterations.size(),
                    sskm_b200::stop_reason_name(r.stop_reason), r.objective,
                    static_cast<unsigned long long>(r.total_dot_products()), r.assignments[0], r.assignments[1],
                    r.assignments[2], r.assignments[3]);
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument: %s\n", e.what());
        return 2;
    } catch (const std::runtime_error& e) {
        std::printf("runtime_error: %s\n", e.what());
        return 1;
    }
    return 0;
}
