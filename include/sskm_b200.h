/* sskm_b200 — C-ABI boundary of the B200-native sparse spherical k-means core.
 *
 * Plain pointers and sizes only (no torch / C++ types). Every entry point
 * returns an int status: SSKM_OK, SSKM_EINVAL (what the reference throws as
 * std::invalid_argument -> Python ValueError, CLI exit 2), or SSKM_ERUNTIME
 * (CUDA / resource failure -> std::runtime_error, CLI exit 1). The message of
 * the last failure on the calling thread is sskm_last_error().
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/include/sskm/engine.hpp unless noted). A context is
 * driven by one host thread; it owns device-resident corpus shard, centroids
 * and state on one GPU, so per-iteration calls move no bulk data over PCIe.
 */
#ifndef SSKM_B200_H
#define SSKM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSKM_OK 0
#define SSKM_EINVAL 1
#define SSKM_ERUNTIME 2

/* Mode, engine.hpp:13 (parse_mode, engine.cpp:21-27). */
#define SSKM_MODE_BASELINE 0
#define SSKM_MODE_NCC 1
#define SSKM_MODE_NCC_INDEX 2 /* assignment by the exact NCC kernels; when the reference would build its
                                 Lemma-1 index (engine.cpp:384-386) the index is rebuilt on the GPU and
                                 its queries replayed: index_* counters and dot_products are the reference's */

/* StopReason, engine.hpp:59 */
#define SSKM_STOP_NO_REASSIGNMENTS 0
#define SSKM_STOP_CENTROID_DRIFT 1
#define SSKM_STOP_MAX_ITERATIONS 2

/* RunConfig, engine.hpp:20-41 (+ GPU-only knobs that do not change the
 * meaning of the reference fields). */
typedef struct {
    uint32_t k;
    int32_t mode;
    const double* lambdas; /* validated like the reference; thresholds of the ncc+index index */
    uint32_t n_lambdas;
    double conv_sq_dist;
    double ncc_epsilon;
    uint32_t index_activation_threshold;
    uint32_t max_iters;
    uint64_t seed;    /* k-means++ seed when no init seeds are given */
    uint32_t threads; /* accepted for API parity; the GPU grid replaces it */
    int32_t device;   /* CUDA device ordinal */
} sskm_run_config;

/* IterationStats, engine.hpp:43-57, followed by GPU extras. `dot_products`
 * counts exactly what the reference's assign would have evaluated
 * (engine.cpp:253-306) so the reference's accounting invariants hold;
 * `gpu_dot_products` is what the kernels evaluated: full (document, centroid)
 * dots — exact fp64 ones (bound-screen candidates and own-cluster dots, exact
 * tile scans) and the fp32 screens' dots — not the bound screen's partial sums
 * over high centroid entries. */
typedef struct {
    uint32_t iteration;
    uint32_t n_unchanged_centroids;
    uint64_t n_reassigned;
    uint64_t dot_products;
    uint64_t index_queries;
    uint64_t candidates_total;
    double wall_seconds;
    double index_build_seconds;
    double max_sq_drift;
    double objective;
    int32_t index_active;
    int32_t n_repaired;
    /* --- GPU extras --- */
    uint64_t gpu_dot_products;
    uint64_t n_moved;         /* documents whose cluster changed since the last update */
    uint32_t n_changed;       /* centroids scanned by the NCC pass (unchanged flag clear) */
    uint32_t n_recomputed;    /* centroid columns rewritten by the update */
    uint64_t n_rescan;        /* NCC documents that needed the unchanged-centroid pass */
    uint64_t n_exact;         /* documents the screen handed to the exact fp64 tile scan */
    double update_ms;         /* device time of compute_centroids + detect_unchanged */
    double assign_ms;         /* device time of the assignment step */
    double assign_kernel_ms;  /* = assign_ms (a separate event pair was dropped: two launches on the host's path) */
    double screen_ms;         /* device time of the screen kernel launches only (bound or postings screen) */
    uint32_t screen_launches; /* screen launches in this assign (one per cluster tile) */
    uint32_t second_pass_docs; /* hash screens: documents the first pass left that a second pass (lower theta, larger tables) screened */
    double centroid_density;  /* nonzero fraction of the centroid tile last indexed (screen choice) */
    /* bound screen (the default screen after the seed assignment) */
    uint64_t bound_docs;       /* documents the bound screen resolved (summed over its passes) */
    uint64_t bound_pairs;      /* high (cluster, value) pairs accumulated */
    uint64_t bound_candidates; /* exact fp64 candidate dots */
    uint64_t bound_doc_nnz;    /* document nonzeros read by the bound-screen launches (all tiles) */
    uint64_t bound_cand_nnz;   /* document nonzeros of the candidate dots (= centroid values gathered) */
    double bound_theta;        /* high/low split of the centroid weights used by the last pass */
    uint64_t bound_visits;     /* documents visited by the bound-screen launches (all tiles) */
    uint64_t bound_own_dots;   /* exact own-cluster dots computed inside the screen (the rest were cached) */
    uint64_t skip_docs;        /* documents the drift bound kept in their cluster without a screen */
    uint64_t bound_own_nnz;    /* document nonzeros of those own dots (= own-column weights gathered from C^T) */
    uint64_t reserved2;
    double skip_ms;            /* CUDA-event time of the drift-bound pass */
} sskm_iteration_stats;

typedef struct sskm_ctx sskm_ctx;

const char* sskm_last_error(void);

/* Validation exactly as RunConfig::validate (engine.cpp:47-64). */
int sskm_validate(const sskm_run_config* cfg, uint64_t n_docs);

/* Context on one device. */
int sskm_open(int32_t device, sskm_ctx** out);
int sskm_close(sskm_ctx* ctx);

/* Copies a caller-owned CSR corpus (int64 indptr[n+1], int32 indices sorted
 * strictly ascending within a row, fp32 values) to the device. Replaces
 * building sskm::CorpusMatrix (corpus.hpp:26-32). For a document shard of a
 * multi-GPU run, doc_offset is the global id of row 0 and n_docs_total the
 * global corpus size (both 0 / n_docs for a single GPU). */
int sskm_upload_csr(sskm_ctx* ctx, int64_t n_docs, uint32_t dims, const int64_t* indptr,
                    const int32_t* indices, const float* values, int64_t doc_offset,
                    int64_t n_docs_total);

/* Config for the following calls; validates like RunConfig::validate. */
int sskm_configure(sskm_ctx* ctx, const sskm_run_config* cfg);

/* BASELINE init: centroid j = document seeds[j] (global ids), then the
 * nearest-seed full-scan assignment with ties to the lowest seed — the state
 * seed_kmeanspp (engine.hpp:74, engine.cpp:82-97) leaves for those seeds. */
int sskm_init_from_seeds(sskm_ctx* ctx, const uint32_t* seeds);

/* k-means++ seeding, seed_kmeanspp (engine.hpp:74; engine.cpp:66-130), with the
 * pinned mt19937_64 draws (random.hpp:11-19); writes the k chosen documents. */
int sskm_init_kmeanspp(sskm_ctx* ctx, uint64_t seed, uint32_t* seeds_out);

/* compute_centroids (engine.hpp:93) + detect_unchanged (engine.hpp:106) + the
 * repaired-forces-changed rule (engine.cpp:371-376): one iteration's update. */
int sskm_update(sskm_ctx* ctx, sskm_iteration_stats* st);

/* assign (engine.hpp:124) for the current iteration (full scan on iteration 1
 * or in baseline mode, exact NCC otherwise) + objective (engine.cpp:403-405). */
int sskm_assign(sskm_ctx* ctx, sskm_iteration_stats* st);

/* One Lloyd iteration = sskm_update + sskm_assign (run() loop body, engine.cpp:357-407). */
int sskm_step(sskm_ctx* ctx, sskm_iteration_stats* st);

/* n Lloyd iterations back to back, whatever the stop rules say (fixed-length
 * runs: benchmarks, the reference CLI's bench with a fixed iteration count);
 * stats has room for n entries (or is NULL). */
int sskm_step_n(sskm_ctx* ctx, uint32_t n, sskm_iteration_stats* stats);

/* run() loop (engine.cpp:357-424) from the current state: iterations until no
 * reassignment, drift < conv_sq_dist (iteration > 1), or max_iters. */
int sskm_run(sskm_ctx* ctx, sskm_iteration_stats* stats, uint32_t stats_cap, uint32_t* n_iters,
             int32_t* stop_reason);

/* State readback / teacher forcing (ClusteringState, engine.hpp:110-117). */
int sskm_get_state(sskm_ctx* ctx, uint32_t* assignments, double* sims, uint8_t* unchanged);
int sskm_set_state(sskm_ctx* ctx, const uint32_t* assignments, const double* sims,
                   uint32_t iteration);
/* Centroids as Cᵀ, d rows × k columns, row-major fp32. */
int sskm_get_centroids(sskm_ctx* ctx, float* ct);
int sskm_set_centroids(sskm_ctx* ctx, const float* ct);
/* Slices of Cᵀ for large-k checks (the dense d×k copy is 26 GB at config 4):
 * rows[0..n_rows) of Cᵀ → out[n_rows][k]; columns cols[0..n_cols) → out[d][n_cols]. */
int sskm_get_centroid_rows(sskm_ctx* ctx, uint32_t n_rows, const uint32_t* rows, float* out);
int sskm_get_centroid_cols(sskm_ctx* ctx, uint32_t n_cols, const uint32_t* cols, float* out);
/* Teacher forcing of the NCC flags (unchanged[j] = 1: cluster j skipped by the
 * changed-list scan); extension, no reference counterpart. */
int sskm_set_unchanged(sskm_ctx* ctx, const uint8_t* unchanged);
int sskm_get_repaired(sskm_ctx* ctx, uint32_t* repaired, uint32_t* n_repaired);
int sskm_get_iteration(sskm_ctx* ctx, uint32_t* iteration);

/* Multi-device context (SURVEY §8b sskm_cuda_open(n_dev, devs)): one host
 * thread drives the listed GPUs; documents are sharded in contiguous equal
 * ranges, centroids and the exact integer cluster sums replicated. Each
 * iteration every device applies every shard's moved rows to its own sums,
 * reading the peers' shards over NVLink (peer access): no gather, no
 * collective library. Assignments, sims and centroids are bitwise those of a
 * single device. The calls mirror the single-device ones above. */
typedef struct sskm_multi sskm_multi;
int sskm_multi_open(int32_t n_devices, const int32_t* devices, sskm_multi** out);
int sskm_multi_close(sskm_multi* ctx);
int sskm_multi_upload_csr(sskm_multi* ctx, int64_t n_docs, uint32_t dims, const int64_t* indptr,
                          const int32_t* indices, const float* values);
int sskm_multi_configure(sskm_multi* ctx, const sskm_run_config* cfg);
int sskm_multi_init_from_seeds(sskm_multi* ctx, const uint32_t* seeds);
int sskm_multi_step(sskm_multi* ctx, sskm_iteration_stats* st);
int sskm_multi_run(sskm_multi* ctx, sskm_iteration_stats* stats, uint32_t stats_cap, uint32_t* n_iters,
                   int32_t* stop_reason);
int sskm_multi_get_state(sskm_multi* ctx, uint32_t* assignments, double* sims);
int sskm_multi_get_centroids(sskm_multi* ctx, float* ct);
int sskm_multi_launch_count(sskm_multi* ctx, uint64_t* n);
/* sskm::run (engine.hpp:148) over several devices, as sskm_cluster_csr below;
 * needs the seeds (k-means++ seeding is single-device). */
int sskm_cluster_csr_multi(const sskm_run_config* cfg, int32_t n_devices, const int32_t* devices, int64_t n_docs,
                           uint32_t dims, const int64_t* indptr, const int32_t* indices, const float* values,
                           const uint32_t* seeds, uint32_t* assignments, double* sims, float* ct,
                           sskm_iteration_stats* stats, uint32_t stats_cap, uint32_t* n_iters,
                           int32_t* stop_reason, double* objective);

/* Test hook: rebuilds the bound screen's high postings from the current
 * centroids and compares them with the lists kept and maintained in place
 * across iterations; bad_rows = differing rows, -1 when none are kept. */
int sskm_debug_check_postings(sskm_ctx* ctx, int64_t* bad_rows);

/* Device timing on the context's stream (CUDA events; 256 slots) and the
 * number of kernels this context has launched — the bench's live evidence. */
int sskm_timer_record(sskm_ctx* ctx, int32_t slot);
int sskm_timer_elapsed(sskm_ctx* ctx, int32_t a, int32_t b, double* ms);
int sskm_launch_count(sskm_ctx* ctx, uint64_t* n);
int sskm_synchronize(sskm_ctx* ctx);
/* Σ over document nonzeros of the number of centroids with a nonzero weight on
 * that term, for the current centroids: the (cluster, value) pairs one
 * postings-screen assign streams (the kernel's algorithmic work). */
int sskm_postings_work(sskm_ctx* ctx, uint64_t* pairs);

/* One-shot drop-in for sskm::run(const CorpusMatrix&, const RunConfig&)
 * (engine.hpp:148): upload, seed (given seeds, or k-means++ when seeds is
 * NULL), iterate, download. Any output pointer may be NULL. */
int sskm_cluster_csr(const sskm_run_config* cfg, int64_t n_docs, uint32_t dims,
                     const int64_t* indptr, const int32_t* indices, const float* values,
                     const uint32_t* seeds, uint32_t* assignments, double* sims, float* ct,
                     sskm_iteration_stats* stats, uint32_t stats_cap, uint32_t* n_iters,
                     int32_t* stop_reason, double* objective);

/* sskm_cluster_csr keeps one engine per device between calls (its HBM
 * buffers are reused); this frees them. */
int sskm_release_cache(void);

/* ---- multi-GPU document sharding (one context per GPU / process) ----------
 * Documents are sharded in contiguous ranges; centroids and the fixed-point
 * cluster sums are replicated. An iteration's update exchanges only the rows
 * of documents that moved (delta path). The host driver moves the bytes with
 * its collective library (NCCL via torch.distributed), in rank order. */

/* Local cluster sizes (int64[k]) for the global empty-cluster check. */
int sskm_local_counts(sskm_ctx* ctx, int64_t* counts);
/* The first m local documents in the reference's repair-donor order (lowest
 * cached sim, then lowest index; engine.cpp:156-161): their sims, global ids
 * and current clusters (host arrays). The driver merges all ranks' lists and
 * replays the sequential repair rule identically on every rank. */
int sskm_local_candidates(sskm_ctx* ctx, int64_t m, double* sims, int64_t* gids, uint32_t* clusters,
                          int64_t* m_out);
/* Reassign a local document (repair move, engine.cpp:162-165). */
int sskm_move_doc(sskm_ctx* ctx, int64_t global_doc, uint32_t cluster);
/* Moved documents of this shard: count and total nonzeros (device-side). */
int sskm_moved_prepare(sskm_ctx* ctx, int64_t* n_moved, int64_t* nnz_moved);
/* Packs them into caller-owned DEVICE buffers: old/new cluster per document,
 * row lengths, and the rows' indices and values back to back. */
int sskm_moved_pack(sskm_ctx* ctx, uint32_t* old_c, uint32_t* new_c, int32_t* lens, int32_t* idx, float* val);
/* Seed init from the k seed rows gathered across shards (host CSR, k rows). */
int sskm_init_from_rows(sskm_ctx* ctx, const int64_t* row_ptr, const int32_t* idx, const float* val);
/* Applies gathered moved rows (DEVICE pointers on this context's GPU; rows
 * from all ranks, any order) to the
 * replicated sums, then finishes the update exactly like sskm_update. */
int sskm_update_apply(sskm_ctx* ctx, int64_t n_moved, const uint32_t* old_c, const uint32_t* new_c,
                      const int64_t* row_ptr, const int32_t* idx, const float* val,
                      const uint32_t* repaired, uint32_t n_repaired, sskm_iteration_stats* st);
/* Local partials for the assign step's scalars (sums over the shard). */
int sskm_local_sims_sum(sskm_ctx* ctx, double* sum);

/* GPU TF-IDF ingestion: vectorize_corpus (corpus.hpp:60-88, corpus.cpp:101-134;
 * Python binding bindings.cpp:53-63), bit-identical to the reference.
 * Documents are one byte array `text` with n_docs + 1 nondecreasing offsets
 * (the caller keeps the ids); stop words likewise (n_stop strings). Errors as
 * the reference: SSKM_ERUNTIME "empty corpus" / "empty vocabulary",
 * SSKM_EINVAL "max_df_ratio must be in (0, 1]". The result handle holds host
 * copies: the CSR rows (fp64 values, int32 dims ascending), the input document
 * index of each row, the dropped documents in the reference's order (stop-word
 * documents first, then rows that vectorised to zero), doc_freq by dim,
 * Vocabulary::n_docs and the vocabulary strings in dim order. */
typedef struct sskm_vec sskm_vec;
int sskm_vectorize(int32_t device, int64_t n_docs, const char* text, const int64_t* text_offsets, int64_t n_stop,
                   const char* stop_text, const int64_t* stop_offsets, double max_df_ratio, sskm_vec** out);
int sskm_vec_sizes(const sskm_vec* v, int64_t* n_rows, int64_t* nnz, uint32_t* dims, uint32_t* n_docs_vocab,
                   int64_t* n_dropped, int64_t* vocab_bytes);
/* Any output pointer may be NULL (skipped). vocab_offsets has dims + 1 entries. */
int sskm_vec_export(const sskm_vec* v, int64_t* indptr, int32_t* indices, double* values, int64_t* kept_docs,
                    int64_t* dropped_docs, uint32_t* doc_freq, char* vocab_text, int64_t* vocab_offsets);
/* Device time of the pipeline (upload to the last kernel), kernels launched,
 * tokens, rows that needed Brent's cycle search in normalize. */
int sskm_vec_stats(const sskm_vec* v, double* gpu_ms, uint64_t* launches, uint64_t* n_tokens, uint64_t* brent_rows);
int sskm_vec_free(sskm_vec* v);
/* normalize (sparse_vector.hpp:60-63, sparse_vector.cpp:158-209) of every row
 * of a host CSR on the GPU, bit-identical to the reference (iterated unit step,
 * period-2 rule, Brent's cycle search). Outputs sized like the inputs; rows can
 * only lose entries whose quotient underflows. */
int sskm_normalize_csr(int32_t device, int64_t n_rows, const int64_t* indptr, const int32_t* indices,
                       const double* values, int64_t* out_indptr, int32_t* out_indices, double* out_values);

#ifdef __cplusplus
}
#endif
#endif /* SSKM_B200_H */
