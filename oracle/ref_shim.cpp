// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference library, compiled from
// the read-only sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libsskm_ref.so. It drives the reference's public per-iteration
// operations exactly like the reference tests' `Stepper`
// (proj/tests/test_engine.cpp:54-100) so the parity tests and the bench's
// reference arm can call the real C++ engine from Python (ctypes) on CSR
// inputs. Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
// --impl reference) may load it.
//
// Entry points mirror, one for one:
//   sref_corpus_from_csr      -> builds sskm::CorpusMatrix (corpus.hpp:26-32) in-process
//                                (load_matrix's 1e-9 norm check would reject fp32 rows,
//                                corpus.cpp:256-262, so it is bypassed as SURVEY §8c says)
//   sref_stepper_*            -> Stepper (test_engine.cpp:54-100) around
//                                compute_centroids / detect_unchanged / assign (engine.hpp:93-125)
//   sref_run                  -> sskm::run (engine.hpp:148)
//   sref_seed_kmeanspp        -> sskm::seed_kmeanspp (engine.hpp:74)
//   sref_dot / sref_normalize -> sparse_vector.hpp:58-63
//   sref_vectorize_*          -> sskm::vectorize_corpus (corpus.hpp:80-88) on in-memory texts
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "sskm/corpus.hpp"
#include "sskm/engine.hpp"
#include "sskm/prune_index.hpp"
#include "sskm/report.hpp"
#include "sskm/sparse_vector.hpp"
#include "sskm/synthetic.hpp"

using namespace sskm;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    } catch (...) {
        g_err = "unknown error";
        return 2;
    }
}

struct CStats {
    std::uint32_t iteration;
    std::uint32_t n_unchanged_centroids;
    std::uint64_t n_reassigned;
    std::uint64_t dot_products;
    std::uint64_t index_queries;
    std::uint64_t candidates_total;
    double wall_seconds;
    double index_build_seconds;
    double max_sq_drift;
    double objective;
    std::int32_t index_active;
    std::int32_t n_repaired;
};

void to_c(const IterationStats& s, CStats* o) {
    o->iteration = s.iteration;
    o->n_unchanged_centroids = s.n_unchanged_centroids;
    o->n_reassigned = s.n_reassigned;
    o->dot_products = s.dot_products;
    o->index_queries = s.index_queries;
    o->candidates_total = s.candidates_total;
    o->wall_seconds = s.wall_seconds;
    o->index_build_seconds = s.index_build_seconds;
    o->max_sq_drift = s.max_sq_drift;
    o->objective = s.objective;
    o->index_active = s.index_active ? 1 : 0;
    o->n_repaired = 0;
}

std::vector<SparseVector> centroids_from_csr(std::uint32_t k, std::uint32_t dims,
                                             const std::int64_t* ptr, const std::uint32_t* idx,
                                             const double* val) {
    std::vector<SparseVector> out;
    out.reserve(k);
    for (std::uint32_t j = 0; j < k; ++j) {
        std::vector<Entry> e;
        e.reserve(static_cast<std::size_t>(ptr[j + 1] - ptr[j]));
        for (std::int64_t p = ptr[j]; p < ptr[j + 1]; ++p) e.push_back({idx[p], val[p]});
        out.emplace_back(std::move(e), dims);
    }
    return out;
}

std::int64_t csr_nnz(const std::vector<SparseVector>& vs) {
    std::int64_t n = 0;
    for (const auto& v : vs) n += static_cast<std::int64_t>(v.nnz());
    return n;
}

void csr_export(const std::vector<SparseVector>& vs, std::int64_t* ptr, std::uint32_t* idx,
                double* val) {
    std::int64_t p = 0;
    ptr[0] = 0;
    for (std::size_t j = 0; j < vs.size(); ++j) {
        for (const Entry& e : vs[j].entries()) {
            idx[p] = e.dim;
            val[p] = e.weight;
            ++p;
        }
        ptr[j + 1] = p;
    }
}

// Stepper: the reference tests' per-iteration driver (test_engine.cpp:54-100),
// extended with seeding from given documents (the BASELINE init) and with
// teacher-forcing setters.
struct Stepper {
    const CorpusMatrix* data = nullptr;
    RunConfig config;
    ClusteringState state;
    std::vector<std::uint32_t> last_repaired;

    IterationStats step() {
        state.iteration += 1;
        auto update =
            compute_centroids(*data, state.assignments, state.sims, config.k, config.threads);
        std::uint32_t n_unchanged = 0;
        double drift = 0.0;
        if (state.iteration == 1) {
            state.unchanged.assign(config.k, 0);
        } else {
            auto ur = detect_unchanged(state.centroids, update.centroids, config.ncc_epsilon,
                                       config.threads);
            for (std::uint32_t j : update.repaired) {
                if (ur.unchanged[j]) {
                    ur.unchanged[j] = 0;
                    --ur.n_unchanged;
                }
            }
            state.unchanged = std::move(ur.unchanged);
            n_unchanged = ur.n_unchanged;
            drift = ur.max_sq_drift;
        }
        last_repaired = update.repaired;
        state.prev_centroids = std::move(state.centroids);
        state.centroids = std::move(update.centroids);
        return assign_now(n_unchanged, drift);
    }

    IterationStats assign_now(std::uint32_t n_unchanged, double drift) {
        MultiIndex index;
        const MultiIndex* index_ptr = nullptr;
        IterationStats st;
        if (config.mode == Mode::kNccIndex && state.iteration > 1 &&
            config.k - n_unchanged > config.index_activation_threshold) {
            auto tb = std::chrono::steady_clock::now();
            index = MultiIndex::build(state.centroids, config.lambdas);
            st.index_build_seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
            index_ptr = &index;
        }
        IterationStats a = assign(*data, state, config, index_ptr);
        a.max_sq_drift = drift;
        a.index_build_seconds = st.index_build_seconds;
        double obj = 0.0;  // run() sums the cached sims in document order (engine.cpp:403-405)
        for (double s : state.sims) obj += s;
        a.objective = obj;
        return a;
    }
};

}  // namespace

extern "C" {

const char* sref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- corpus ---
void* sref_corpus_from_csr(std::int64_t n, std::uint32_t dims, const std::int64_t* indptr,
                           const std::int32_t* indices, const double* values) {
    CorpusMatrix* m = nullptr;
    int rc = guard([&] {
        auto* mm = new CorpusMatrix();
        try {
            mm->dims = dims;
            mm->vectors.reserve(static_cast<std::size_t>(n));
            for (std::int64_t i = 0; i < n; ++i) {
                std::vector<Entry> e;
                e.reserve(static_cast<std::size_t>(indptr[i + 1] - indptr[i]));
                for (std::int64_t p = indptr[i]; p < indptr[i + 1]; ++p) {
                    e.push_back({static_cast<std::uint32_t>(indices[p]), values[p]});
                }
                mm->vectors.emplace_back(std::move(e), dims);
                mm->doc_ids.push_back(std::to_string(i));
            }
        } catch (...) {
            delete mm;
            throw;
        }
        m = mm;
    });
    return rc == 0 ? m : nullptr;
}

void sref_corpus_free(void* m) { delete static_cast<CorpusMatrix*>(m); }

std::int64_t sref_corpus_nnz(void* m) { return csr_nnz(static_cast<CorpusMatrix*>(m)->vectors); }
std::int64_t sref_corpus_n(void* m) { return static_cast<std::int64_t>(static_cast<CorpusMatrix*>(m)->size()); }
std::uint32_t sref_corpus_dims(void* m) { return static_cast<CorpusMatrix*>(m)->dims; }

void sref_corpus_export(void* m, std::int64_t* ptr, std::uint32_t* idx, double* val) {
    csr_export(static_cast<CorpusMatrix*>(m)->vectors, ptr, idx, val);
}

// The reference's own generator (synthetic.cpp:31-68); used for golden vectors.
void* sref_synthetic_zipf(std::uint64_t n_docs, std::uint32_t vocab, double avg_nnz, double s,
                          std::uint64_t seed) {
    CorpusMatrix* m = nullptr;
    int rc = guard([&] {
        m = new CorpusMatrix(synthetic_zipf_corpus({n_docs, vocab, avg_nnz, s, seed}));
    });
    return rc == 0 ? m : nullptr;
}

// ------------------------------------------------------------- vectorize ---
// vectorize_corpus (corpus.cpp:101-134) over texts given as one byte array with
// offsets; doc ids are the decimal input indices, so kept / dropped ids map
// back to positions. Vocabulary strings are exported in dim order.
struct VecOut {
    VectorizeResult r;
    std::vector<std::string> terms;  // by dim
    std::vector<std::int64_t> kept, dropped;
    double seconds = 0.0;
};

int sref_vectorize(std::int64_t n_docs, const char* text, const std::int64_t* offs, std::int64_t n_stop,
                   const char* stop_text, const std::int64_t* stop_offs, double max_df, void** out) {
    *out = nullptr;
    return guard([&] {
        std::vector<std::pair<std::string, std::string>> docs;
        docs.reserve(static_cast<std::size_t>(n_docs));
        for (std::int64_t d = 0; d < n_docs; ++d)
            docs.emplace_back(std::to_string(d), std::string(text + offs[d], text + offs[d + 1]));
        StopWords stop;
        for (std::int64_t w = 0; w < n_stop; ++w)
            stop.insert(std::string(stop_text + stop_offs[w], stop_text + stop_offs[w + 1]));
        auto* v = new VecOut();
        try {
            const auto t0 = std::chrono::steady_clock::now();
            v->r = vectorize_corpus(docs, stop, max_df);
            v->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            v->terms.resize(v->r.vocab.size());
            for (const auto& [term, dim] : v->r.vocab.term_to_dim) v->terms[dim] = term;
            for (const auto& id : v->r.matrix.doc_ids) v->kept.push_back(std::stoll(id));
            for (const auto& id : v->r.dropped_doc_ids) v->dropped.push_back(std::stoll(id));
        } catch (...) {
            delete v;
            throw;
        }
        *out = v;
    });
}

void sref_vec_sizes(void* h, std::int64_t* n_rows, std::int64_t* nnz, std::uint32_t* dims, std::uint32_t* n_docs,
                    std::int64_t* n_dropped, std::int64_t* vocab_bytes, double* seconds) {
    auto* v = static_cast<VecOut*>(h);
    *n_rows = static_cast<std::int64_t>(v->r.matrix.size());
    *nnz = csr_nnz(v->r.matrix.vectors);
    *dims = v->r.matrix.dims;
    *n_docs = v->r.vocab.n_docs;
    *n_dropped = static_cast<std::int64_t>(v->dropped.size());
    std::int64_t b = 0;
    for (const auto& t : v->terms) b += static_cast<std::int64_t>(t.size());
    *vocab_bytes = b;
    *seconds = v->seconds;
}

void sref_vec_export(void* h, std::int64_t* indptr, std::uint32_t* idx, double* val, std::int64_t* kept,
                     std::int64_t* dropped, std::uint32_t* doc_freq, char* vocab_text, std::int64_t* vocab_off) {
    auto* v = static_cast<VecOut*>(h);
    csr_export(v->r.matrix.vectors, indptr, idx, val);
    std::memcpy(kept, v->kept.data(), v->kept.size() * 8);
    if (!v->dropped.empty()) std::memcpy(dropped, v->dropped.data(), v->dropped.size() * 8);
    std::memcpy(doc_freq, v->r.vocab.doc_freq.data(), v->r.vocab.doc_freq.size() * 4);
    std::int64_t o = 0;
    vocab_off[0] = 0;
    for (std::size_t d = 0; d < v->terms.size(); ++d) {
        std::memcpy(vocab_text + o, v->terms[d].data(), v->terms[d].size());
        o += static_cast<std::int64_t>(v->terms[d].size());
        vocab_off[d + 1] = o;
    }
}

void sref_vec_free(void* h) { delete static_cast<VecOut*>(h); }


// ------------------------------------------------------------ primitives ---
int sref_dot(std::int64_t na, const std::uint32_t* ia, const double* va, std::int64_t nb,
             const std::uint32_t* ib, const double* vb, double* out) {
    return guard([&] {
        std::vector<Entry> a, b;
        for (std::int64_t p = 0; p < na; ++p) a.push_back({ia[p], va[p]});
        for (std::int64_t p = 0; p < nb; ++p) b.push_back({ib[p], vb[p]});
        *out = dot(SparseVector(std::move(a)), SparseVector(std::move(b)));
    });
}

// Normalizes in place; *n_out receives the surviving entry count.
int sref_normalize(std::int64_t n, std::uint32_t* idx, double* val, std::int64_t* n_out) {
    return guard([&] {
        std::vector<Entry> a;
        for (std::int64_t p = 0; p < n; ++p) a.push_back({idx[p], val[p]});
        SparseVector r = normalize(SparseVector(std::move(a)));
        std::int64_t q = 0;
        for (const Entry& e : r.entries()) {
            idx[q] = e.dim;
            val[q] = e.weight;
            ++q;
        }
        *n_out = q;
    });
}

// --------------------------------------------------------------- stepper ---
void* sref_stepper_new(void* corpus, std::uint32_t k, const char* mode, double ncc_epsilon,
                       double conv_sq_dist, std::uint32_t max_iters, std::uint32_t threads,
                       std::uint32_t index_activation_threshold) {
    Stepper* s = nullptr;
    int rc = guard([&] {
        auto* st = new Stepper();
        st->data = static_cast<CorpusMatrix*>(corpus);
        st->config.k = k;
        st->config.mode = parse_mode(mode);
        st->config.ncc_epsilon = ncc_epsilon;
        st->config.conv_sq_dist = conv_sq_dist;
        st->config.max_iters = max_iters;
        st->config.threads = threads;
        st->config.index_activation_threshold = index_activation_threshold;
        try {
            st->config.validate(st->data->size());
        } catch (...) {
            delete st;
            throw;
        }
        st->state.unchanged.assign(k, 0);
        s = st;
    });
    return rc == 0 ? s : nullptr;
}

// A stepper over a document SAMPLE for teacher-forced assign checks: k may
// exceed the sample size (config 4: k = 50,000). assign() itself never reads
// RunConfig::validate's k <= n condition (engine.cpp:218-322).
void* sref_stepper_new_sample(void* corpus, std::uint32_t k, const char* mode, double ncc_epsilon,
                              std::uint32_t threads) {
    Stepper* s = nullptr;
    int rc = guard([&] {
        auto* st = new Stepper();
        st->data = static_cast<CorpusMatrix*>(corpus);
        st->config.k = k;
        st->config.mode = parse_mode(mode);
        st->config.ncc_epsilon = ncc_epsilon;
        st->config.threads = threads;
        st->state.unchanged.assign(k, 0);
        s = st;
    });
    return rc == 0 ? s : nullptr;
}

void sref_stepper_free(void* s) { delete static_cast<Stepper*>(s); }

// BASELINE init: centroid j = document seeds[j], then the nearest-seed
// assignment with ties to the lowest seed index. That is exactly what
// seed_kmeanspp leaves behind for those seeds (engine.cpp:82-97); the
// reference's own full-scan assign computes it (engine.cpp:265-266).
int sref_stepper_init_seeds(void* h, const std::uint32_t* seeds, CStats* out) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        const std::size_t n = s->data->size();
        s->state.centroids.clear();
        for (std::uint32_t j = 0; j < s->config.k; ++j) {
            if (seeds[j] >= n) throw std::invalid_argument("seed out of range");
            s->state.centroids.push_back(s->data->vectors[seeds[j]]);
        }
        s->state.assignments.assign(n, 0);
        s->state.sims.assign(n, -2.0);
        s->state.unchanged.assign(s->config.k, 0);
        s->state.iteration = 0;
        IterationStats st = assign(*s->data, s->state, s->config, nullptr);
        if (out) to_c(st, out);
        s->state.iteration = 0;
    });
}

// k-means++ init exactly as run() does it (engine.cpp:349-352).
int sref_stepper_init_kmeanspp(void* h, std::uint64_t seed, std::uint32_t* seeds_out) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        SeedResult r = seed_kmeanspp(*s->data, s->config.k, seed, s->config.threads);
        s->state.assignments = std::move(r.assignments);
        s->state.sims = std::move(r.sims);
        s->state.unchanged.assign(s->config.k, 0);
        s->state.iteration = 0;
        if (seeds_out) std::memcpy(seeds_out, r.seeds.data(), r.seeds.size() * sizeof(std::uint32_t));
    });
}

int sref_stepper_step(void* h, CStats* out) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        IterationStats st = s->step();
        to_c(st, out);
        out->n_repaired = static_cast<std::int32_t>(s->last_repaired.size());
    });
}

// compute_centroids + detect_unchanged only (the first half of a step), so a
// caller can inspect / replace centroids before the assign half.
int sref_stepper_update(void* h, std::uint32_t* n_unchanged_out, double* drift_out) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        Stepper& S = *s;
        S.state.iteration += 1;
        auto update = compute_centroids(*S.data, S.state.assignments, S.state.sims, S.config.k,
                                        S.config.threads);
        std::uint32_t n_unchanged = 0;
        double drift = 0.0;
        if (S.state.iteration == 1) {
            S.state.unchanged.assign(S.config.k, 0);
        } else {
            auto ur = detect_unchanged(S.state.centroids, update.centroids, S.config.ncc_epsilon,
                                       S.config.threads);
            for (std::uint32_t j : update.repaired) {
                if (ur.unchanged[j]) {
                    ur.unchanged[j] = 0;
                    --ur.n_unchanged;
                }
            }
            S.state.unchanged = std::move(ur.unchanged);
            n_unchanged = ur.n_unchanged;
            drift = ur.max_sq_drift;
        }
        S.last_repaired = update.repaired;
        S.state.prev_centroids = std::move(S.state.centroids);
        S.state.centroids = std::move(update.centroids);
        *n_unchanged_out = n_unchanged;
        *drift_out = drift;
    });
}

int sref_stepper_assign(void* h, std::uint32_t n_unchanged, double drift, CStats* out) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        IterationStats st = s->assign_now(n_unchanged, drift);
        to_c(st, out);
    });
}

std::uint32_t sref_stepper_iteration(void* h) { return static_cast<Stepper*>(h)->state.iteration; }

int sref_stepper_get_state(void* h, std::uint32_t* a, double* sims, std::uint8_t* unchanged) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        if (a) std::memcpy(a, s->state.assignments.data(), s->state.assignments.size() * 4);
        if (sims) std::memcpy(sims, s->state.sims.data(), s->state.sims.size() * 8);
        if (unchanged) std::memcpy(unchanged, s->state.unchanged.data(), s->state.unchanged.size());
    });
}

int sref_stepper_set_state(void* h, const std::uint32_t* a, const double* sims,
                           const std::uint8_t* unchanged, std::uint32_t iteration) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        const std::size_t n = s->data->size();
        if (a) s->state.assignments.assign(a, a + n);
        if (sims) s->state.sims.assign(sims, sims + n);
        if (unchanged) s->state.unchanged.assign(unchanged, unchanged + s->config.k);
        s->state.iteration = iteration;
    });
}

int sref_stepper_repaired(void* h, std::uint32_t* out, std::int64_t* n) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        *n = static_cast<std::int64_t>(s->last_repaired.size());
        if (out) std::memcpy(out, s->last_repaired.data(), s->last_repaired.size() * 4);
    });
}

std::int64_t sref_stepper_centroids_nnz(void* h) {
    return csr_nnz(static_cast<Stepper*>(h)->state.centroids);
}

int sref_stepper_get_centroids(void* h, std::int64_t* ptr, std::uint32_t* idx, double* val) {
    return guard([&] { csr_export(static_cast<Stepper*>(h)->state.centroids, ptr, idx, val); });
}

// Selected centroids only (large k: the full export is GBs at config 4).
std::int64_t sref_stepper_cols_nnz(void* h, std::int64_t n, const std::uint32_t* cols) {
    const auto& c = static_cast<Stepper*>(h)->state.centroids;
    std::int64_t t = 0;
    for (std::int64_t q = 0; q < n; ++q) t += static_cast<std::int64_t>(c.at(cols[q]).nnz());
    return t;
}

int sref_stepper_get_cols(void* h, std::int64_t n, const std::uint32_t* cols, std::int64_t* ptr,
                          std::uint32_t* idx, double* val) {
    return guard([&] {
        const auto& c = static_cast<Stepper*>(h)->state.centroids;
        std::int64_t p = 0;
        ptr[0] = 0;
        for (std::int64_t q = 0; q < n; ++q) {
            for (const Entry& e : c.at(cols[q]).entries()) {
                idx[p] = e.dim;
                val[p] = e.weight;
                ++p;
            }
            ptr[q + 1] = p;
        }
    });
}

int sref_stepper_set_centroids(void* h, const std::int64_t* ptr, const std::uint32_t* idx,
                               const double* val) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        s->state.centroids = centroids_from_csr(s->config.k, s->data->dims, ptr, idx, val);
    });
}

// Standalone compute_centroids on caller-owned assignments (mutated by repair).
// Centroids come back through the stepper's centroid slot of `h`.
int sref_compute_centroids(void* h, std::uint32_t* assignments, const double* sims,
                           std::uint32_t* repaired, std::int64_t* n_repaired) {
    return guard([&] {
        auto* s = static_cast<Stepper*>(h);
        const std::size_t n = s->data->size();
        std::vector<std::uint32_t> a(assignments, assignments + n);
        std::vector<double> sm(sims, sims + n);
        CentroidUpdate u = compute_centroids(*s->data, a, sm, s->config.k, s->config.threads);
        std::memcpy(assignments, a.data(), n * 4);
        *n_repaired = static_cast<std::int64_t>(u.repaired.size());
        if (repaired) std::memcpy(repaired, u.repaired.data(), u.repaired.size() * 4);
        s->state.centroids = std::move(u.centroids);
    });
}

// ------------------------------------------------------------------- run ---
// Full sskm::run (k-means++ seeding) — the reference's own public entry.
int sref_run(void* corpus, std::uint32_t k, const char* mode, std::uint64_t seed,
             double conv_sq_dist, double ncc_epsilon, std::uint32_t index_activation_threshold,
             std::uint32_t max_iters, std::uint32_t threads, std::uint32_t* assignments,
             double* sims, CStats* stats, std::uint32_t stats_cap, std::uint32_t* n_iters,
             std::int32_t* stop_reason, double* objective) {
    return guard([&] {
        RunConfig cfg;
        cfg.k = k;
        cfg.mode = parse_mode(mode);
        cfg.seed = seed;
        cfg.conv_sq_dist = conv_sq_dist;
        cfg.ncc_epsilon = ncc_epsilon;
        cfg.index_activation_threshold = index_activation_threshold;
        cfg.max_iters = max_iters;
        cfg.threads = threads;
        const auto& data = *static_cast<CorpusMatrix*>(corpus);
        ClusteringResult r = run(data, cfg);
        std::memcpy(assignments, r.assignments.data(), r.assignments.size() * 4);
        std::memcpy(sims, r.sims.data(), r.sims.size() * 8);
        *n_iters = static_cast<std::uint32_t>(r.iterations.size());
        for (std::size_t t = 0; t < r.iterations.size() && t < stats_cap; ++t) to_c(r.iterations[t], &stats[t]);
        *stop_reason = static_cast<std::int32_t>(r.stop_reason);
        *objective = r.objective;
    });
}

int sref_seed_kmeanspp(void* corpus, std::uint32_t k, std::uint64_t seed, std::uint32_t threads,
                       std::uint32_t* seeds, std::uint32_t* assignments, double* sims) {
    return guard([&] {
        SeedResult r = seed_kmeanspp(*static_cast<CorpusMatrix*>(corpus), k, seed, threads);
        std::memcpy(seeds, r.seeds.data(), r.seeds.size() * 4);
        std::memcpy(assignments, r.assignments.data(), r.assignments.size() * 4);
        std::memcpy(sims, r.sims.data(), r.sims.size() * 8);
    });
}

// ---------------------------------------------------------- corpus IO ---
// load_matrix / write_matrix (corpus.cpp:182-272) and the run report JSON
// (report.cpp:24-79), for IO / report parity tests.
void* sref_load_matrix(const char* path) {
    CorpusMatrix* m = nullptr;
    int rc = guard([&] { m = new CorpusMatrix(load_matrix(path)); });
    return rc == 0 ? m : nullptr;
}

int sref_write_matrix(const char* path, void* corpus) {
    return guard([&] { write_matrix(path, *static_cast<CorpusMatrix*>(corpus)); });
}

// RunReport JSON for a result described by plain arrays.
int sref_report_json(std::uint32_t k, const char* mode, const double* lambdas, std::uint32_t n_lambdas,
                     double conv_sq_dist, double ncc_epsilon, std::uint32_t iat, std::uint32_t max_iters,
                     std::uint64_t seed, std::uint32_t threads, std::uint64_t n_docs, std::uint32_t dims,
                     const CStats* its, std::uint32_t n_it, double objective, std::int32_t stop,
                     const std::uint32_t* assignments, char* out, std::uint64_t cap, std::uint64_t* len) {
    return guard([&] {
        RunReport r;
        r.config.k = k;
        r.config.mode = parse_mode(mode);
        r.config.lambdas.assign(lambdas, lambdas + n_lambdas);
        r.config.conv_sq_dist = conv_sq_dist;
        r.config.ncc_epsilon = ncc_epsilon;
        r.config.index_activation_threshold = iat;
        r.config.max_iters = max_iters;
        r.config.seed = seed;
        r.config.threads = threads;
        r.n_docs = n_docs;
        r.dims = dims;
        for (std::uint32_t t = 0; t < n_it; ++t) {
            IterationStats s;
            s.iteration = its[t].iteration;
            s.n_reassigned = its[t].n_reassigned;
            s.n_unchanged_centroids = its[t].n_unchanged_centroids;
            s.dot_products = its[t].dot_products;
            s.index_queries = its[t].index_queries;
            s.candidates_total = its[t].candidates_total;
            s.wall_seconds = its[t].wall_seconds;
            s.index_build_seconds = its[t].index_build_seconds;
            s.index_active = its[t].index_active != 0;
            s.max_sq_drift = its[t].max_sq_drift;
            s.objective = its[t].objective;
            r.iterations.push_back(s);
        }
        r.objective = objective;
        r.stop_reason = static_cast<StopReason>(stop);
        r.cluster_sizes.assign(k, 0);
        for (std::uint64_t i = 0; i < n_docs; ++i) ++r.cluster_sizes[assignments[i]];
        const std::string j = to_json(r);
        *len = j.size();
        if (out && cap > j.size()) std::memcpy(out, j.c_str(), j.size() + 1);
    });
}

int sref_validate(std::uint64_t n_docs, std::uint32_t k, double conv_sq_dist, double ncc_epsilon,
                  std::uint32_t max_iters, const double* lambdas, std::uint32_t n_lambdas) {
    return guard([&] {
        RunConfig cfg;
        cfg.k = k;
        cfg.conv_sq_dist = conv_sq_dist;
        cfg.ncc_epsilon = ncc_epsilon;
        cfg.max_iters = max_iters;
        cfg.lambdas.assign(lambdas, lambdas + n_lambdas);
        cfg.validate(n_docs);
    });
}

}  // extern "C"
