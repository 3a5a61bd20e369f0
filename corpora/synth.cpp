// Seeded synthetic TF-IDF corpus generator for the BASELINE configs
// (BASELINE.json "configs"). Benchmark/test input only — not on
// the hot path. Deterministic for any thread count: every document draws from
// its own counter-keyed SplitMix64 stream.
//
// Generator (pinned here, stated in DESIGN.md):
//   topics τ ∈ [0, K_true); topic τ is Zipf(s) over ranks 1..d mapped to term ids
//     by a keyed bijection perm_τ of [0, d) (multiply/xorshift rounds on the
//     next power of two, cycle-walked into [0, d));
//   doc i: τ = ⌊u·K_true⌋; L = max(1, round(exp(μ + σ·Z))), μ = ln(mean) − σ²/2,
//     Z = Box–Muller normal; L i.i.d. tokens rank r ~ Zipf(s) by inverse CDF;
//     term = perm_τ(r − 1); tf = multiplicity;
//   w = tf · ln(N / df) with df over the generated corpus; zero weights dropped;
//   rows L2-normalised in fp64 then stored fp32; CSR int64 indptr, int32 sorted
//   indices, fp32 values. Rows left empty (every term has df = N) are dropped.
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t s;
    explicit Rng(uint64_t key) : s(mix64(key)) {}
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // [0, 1)
};

struct Perm {
    uint32_t d, bits;
    uint64_t mask;
    uint64_t add[4], mul[4];
    Perm(uint32_t d_, uint64_t key) : d(d_) {
        bits = 1;
        while ((uint64_t(1) << bits) < d) ++bits;
        mask = (uint64_t(1) << bits) - 1;
        for (int r = 0; r < 4; ++r) {
            add[r] = mix64(key * 8 + 2 * r) & mask;
            mul[r] = mix64(key * 8 + 2 * r + 1) | 1ull;
        }
    }
    uint32_t operator()(uint32_t x) const {
        uint64_t y = x;
        do {
            for (int r = 0; r < 4; ++r) {
                y = (y + add[r]) & mask;
                y = (y * mul[r]) & mask;
                y ^= y >> ((bits + 1) / 2);
            }
        } while (y >= d);
        return static_cast<uint32_t>(y);
    }
};

struct Corpus {
    int64_t n = 0;
    uint32_t d = 0;
    std::vector<int64_t> indptr;
    std::vector<int32_t> idx;
    std::vector<float> val;
    int64_t dropped = 0;
};

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* sskm_synth_last_error(void) { return g_err.c_str(); }

// Generates the corpus; returns an opaque handle (NULL on error).
void* sskm_synth_generate(int64_t n_docs, uint32_t d, uint32_t k_true, double mean_len, double sigma,
                          double zipf_s, uint64_t seed, int threads) {
    try {
        if (n_docs <= 0 || d == 0 || k_true == 0 || !(mean_len > 0) || !(sigma >= 0) || !(zipf_s > 0))
            throw std::invalid_argument("bad generator parameters");
        if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        const uint64_t seed_key = mix64(seed ^ 0x5EEDC0DE5EEDC0DEull);
        // Zipf inverse CDF over ranks 1..d
        std::vector<double> cdf(d);
        double tot = 0.0;
        for (uint32_t r = 0; r < d; ++r) {
            tot += std::pow(static_cast<double>(r + 1), -zipf_s);
            cdf[r] = tot;
        }
        for (auto& c : cdf) c /= tot;
        cdf[d - 1] = 1.0;
        std::vector<Perm> perms;
        perms.reserve(k_true);
        for (uint32_t t = 0; t < k_true; ++t) perms.emplace_back(d, mix64(seed_key + 0x1000 + t));
        const double mu = std::log(mean_len) - 0.5 * sigma * sigma;
        const double max_len = 100.0 * mean_len + 100.0;

        // pass 1: distinct (term, tf) per document, per-thread chunks
        const int64_t n = n_docs;
        std::vector<int64_t> cnt(n + 1, 0);
        struct Chunk {
            std::vector<uint32_t> terms;
            std::vector<uint16_t> tf;
        };
        std::vector<Chunk> chunks(threads);
        std::vector<std::vector<uint32_t>> df_local(threads, std::vector<uint32_t>(d, 0));
        auto chunk_range = [&](int w) {
            const int64_t per = (n + threads - 1) / threads;
            return std::pair<int64_t, int64_t>(std::min<int64_t>(n, per * w), std::min<int64_t>(n, per * (w + 1)));
        };
        auto work1 = [&](int w) {
            auto [b, e] = chunk_range(w);
            std::vector<uint32_t> toks;
            Chunk& ch = chunks[w];
            auto& df = df_local[w];
            for (int64_t i = b; i < e; ++i) {
                Rng g(seed_key ^ mix64(static_cast<uint64_t>(i) + 0x9E37ull));
                const uint32_t topic = std::min<uint32_t>(k_true - 1, static_cast<uint32_t>(g.unit() * k_true));
                const double u1 = 1.0 - g.unit(), u2 = g.unit();
                const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
                double lf = std::exp(mu + sigma * z);
                if (lf > max_len) lf = max_len;
                const int64_t L = std::max<int64_t>(1, std::llround(lf));
                toks.resize(L);
                const Perm& P = perms[topic];
                for (int64_t t = 0; t < L; ++t) {
                    const double u = g.unit();
                    const uint32_t r = static_cast<uint32_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
                    toks[t] = P(std::min<uint32_t>(r, d - 1));
                }
                std::sort(toks.begin(), toks.end());
                int64_t m = 0;
                for (int64_t t = 0; t < L;) {
                    int64_t s = t;
                    while (t < L && toks[t] == toks[s]) ++t;
                    ch.terms.push_back(toks[s]);
                    ch.tf.push_back(static_cast<uint16_t>(std::min<int64_t>(t - s, 65535)));
                    ++df[toks[s]];
                    ++m;
                }
                cnt[i + 1] = m;
            }
        };
        {
            std::vector<std::thread> th;
            for (int w = 0; w < threads; ++w) th.emplace_back(work1, w);
            for (auto& t : th) t.join();
        }
        std::vector<uint32_t> df(d, 0);
        for (int w = 0; w < threads; ++w)
            for (uint32_t t = 0; t < d; ++t) df[t] += df_local[w][t];
        df_local.clear();
        df_local.shrink_to_fit();
        std::vector<int64_t> raw_ptr(n + 1, 0);
        for (int64_t i = 0; i < n; ++i) raw_ptr[i + 1] = raw_ptr[i] + cnt[i + 1];
        std::vector<double> idf(d);
        for (uint32_t t = 0; t < d; ++t)
            idf[t] = df[t] ? std::log(static_cast<double>(n) / static_cast<double>(df[t])) : 0.0;

        // pass 2: weights, drop zeros, normalise; rows counted then compacted
        std::vector<int64_t> keep(n + 1, 0);
        std::vector<std::vector<int32_t>> out_idx(threads);
        std::vector<std::vector<float>> out_val(threads);
        auto work2 = [&](int w) {
            auto [b, e] = chunk_range(w);
            const Chunk& ch = chunks[w];
            int64_t off = 0;
            std::vector<double> wts;
            std::vector<int32_t> ids;
            for (int64_t i = b; i < e; ++i) {
                const int64_t m = cnt[i + 1];
                wts.clear();
                ids.clear();
                for (int64_t q = 0; q < m; ++q) {
                    const uint32_t t = ch.terms[off + q];
                    const double wv = static_cast<double>(ch.tf[off + q]) * idf[t];
                    if (wv != 0.0) {
                        wts.push_back(wv);
                        ids.push_back(static_cast<int32_t>(t));
                    }
                }
                off += m;
                double s = 0.0;
                for (double x : wts) s += x * x;
                const double nrm = std::sqrt(s);
                int64_t kept = 0;
                for (size_t q = 0; q < wts.size(); ++q) {
                    const float v = static_cast<float>(wts[q] / nrm);
                    if (v != 0.0f) {
                        out_idx[w].push_back(ids[q]);
                        out_val[w].push_back(v);
                        ++kept;
                    }
                }
                keep[i + 1] = kept;
            }
        };
        {
            std::vector<std::thread> th;
            for (int w = 0; w < threads; ++w) th.emplace_back(work2, w);
            for (auto& t : th) t.join();
        }
        chunks.clear();
        auto* c = new Corpus();
        c->d = d;
        c->indptr.push_back(0);
        int64_t total = 0;
        for (int w = 0; w < threads; ++w) total += static_cast<int64_t>(out_idx[w].size());
        c->idx.reserve(total);
        c->val.reserve(total);
        for (int w = 0; w < threads; ++w) {
            c->idx.insert(c->idx.end(), out_idx[w].begin(), out_idx[w].end());
            c->val.insert(c->val.end(), out_val[w].begin(), out_val[w].end());
            std::vector<int32_t>().swap(out_idx[w]);
            std::vector<float>().swap(out_val[w]);
        }
        c->indptr.reserve(n + 1);
        for (int64_t i = 0; i < n; ++i) {
            if (keep[i + 1] == 0) {
                ++c->dropped;
                continue;
            }
            c->indptr.push_back(c->indptr.back() + keep[i + 1]);
        }
        c->n = static_cast<int64_t>(c->indptr.size()) - 1;
        return c;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void sskm_synth_sizes(void* h, int64_t* n, int64_t* nnz, uint32_t* d, int64_t* dropped) {
    auto* c = static_cast<Corpus*>(h);
    *n = c->n;
    *nnz = static_cast<int64_t>(c->idx.size());
    *d = c->d;
    *dropped = c->dropped;
}

void sskm_synth_export(void* h, int64_t* indptr, int32_t* idx, float* val) {
    auto* c = static_cast<Corpus*>(h);
    std::memcpy(indptr, c->indptr.data(), c->indptr.size() * sizeof(int64_t));
    if (!c->idx.empty()) {
        std::memcpy(idx, c->idx.data(), c->idx.size() * sizeof(int32_t));
        std::memcpy(val, c->val.data(), c->val.size() * sizeof(float));
    }
}

void sskm_synth_free(void* h) { delete static_cast<Corpus*>(h); }

}  // extern "C"
