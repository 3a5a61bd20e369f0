/* Corpus IO (paper_2108_00895_b200/csrc/io.cpp): the reference's text matrix
 * format (write_matrix / load_matrix, corpus.cpp:182-272; same checks and
 * messages) and a binary CSR format. Host code, not on the hot path. */
#ifndef SSKM_IO_H
#define SSKM_IO_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
const char* sskm_io_last_error(void);
void* sskm_io_load_matrix(const char* path, double norm_tol, int threads);
void sskm_io_sizes(void* h, int64_t* n, uint32_t* dims, int64_t* nnz, int64_t* ids_bytes);
void sskm_io_export(void* h, int64_t* indptr, int32_t* idx, float* values_f32, double* values_f64, char* ids);
void sskm_io_free(void* h);
int sskm_io_write_matrix(const char* path, int64_t n, uint32_t dims, const int64_t* indptr, const int32_t* idx,
                         const float* val, const char* ids_joined);
int sskm_io_save_csr(const char* path, int64_t n, uint32_t dims, const int64_t* indptr, const int32_t* idx,
                     const float* val);
int sskm_io_csr_header(const char* path, int64_t* n, uint32_t* dims, int64_t* nnz);
int sskm_io_csr_read(const char* path, int64_t* indptr, int32_t* idx, float* val);
#ifdef __cplusplus
}
#endif
#endif
