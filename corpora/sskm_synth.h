/* Seeded synthetic TF-IDF corpus generator for the BASELINE configs
 * (paper_2108_00895_b200/csrc/synth.cpp; generator pinned in DESIGN.md).
 * Benchmark/test input only; not part of the reference's hot-path boundary. */
#ifndef SSKM_SYNTH_H
#define SSKM_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
const char* sskm_synth_last_error(void);
void* sskm_synth_generate(int64_t n_docs, uint32_t d, uint32_t k_true, double mean_len, double sigma,
                          double zipf_s, uint64_t seed, int threads);
void sskm_synth_sizes(void* h, int64_t* n, int64_t* nnz, uint32_t* d, int64_t* dropped);
void sskm_synth_export(void* h, int64_t* indptr, int32_t* idx, float* val);
void sskm_synth_free(void* h);
#ifdef __cplusplus
}
#endif
#endif
