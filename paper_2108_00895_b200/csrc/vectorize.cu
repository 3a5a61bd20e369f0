// GPU TF-IDF vectorisation: the reference's ingestion pipeline
// vectorize_corpus (corpus.cpp:101-134) — tokenize (:16-30), build_vocabulary
// (:32-64), tfidf (:66-84), vectorize/normalize (:86-91; sparse_vector.cpp:
// 119-209) — on the device, bit for bit.
//
// Layout: the documents' texts are one byte array with int64 offsets (the host
// keeps the ids). Every per-byte, per-token, per-term and per-nonzero step runs
// on the GPU:
//   1. byte classes → token start/end flags (a document boundary ends a token),
//      compacted into token extents;
//   2. per token: its document (binary search) and a 64-bit hash of its
//      lowercased bytes; a stable radix sort by hash groups the occurrences of
//      a term in corpus order, so a group's head is the term's first
//      occurrence; every occurrence is compared byte for byte with its head
//      (a 64-bit collision between different strings fails loudly);
//   3. per term: document frequency (document changes inside the group), stop
//      word test (sorted stop-word hashes + byte compare); documents holding a
//      non-stop token are kept, the rest dropped before the vocabulary
//      (corpus.cpp:106-118); terms pass the max-df test on the kept count in
//      fp64 exactly as :57; dims in first-occurrence order = a sort of the
//      surviving heads' token positions;
//   4. per (kept document, dim): a radix sort of packed keys and a run-length
//      encode give tf in ascending dim within each document; w = tf·idf,
//      zero weights dropped (:77-78), empty rows dropped (:124-129);
//   5. normalize per row (one thread per row, sequential fp64 in entry order
//      with explicit _rn intrinsics, no FMA contraction): the reference's
//      iterated unit step to its fixpoint or period-2 cycle, and Brent's cycle
//      search for the rare long orbits (a second kernel over those rows).
// The idf table ln(N/df) is vocabulary-sized; it is evaluated with the host's
// libm (the reference's own std::log), so weights match the reference bit for
// bit — CUDA's log() is not correctly rounded (≤ 1 ulp).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "../../include/sskm_b200.h"
#include "common.cuh"

namespace sskm_b200 {
void set_last_error(const char* msg);  // engine.cu (sskm_last_error)

namespace vec {

template <typename T>
struct Buf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        free();
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    Buf() = default;
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    ~Buf() { free(); }
};

// C-locale isalnum || byte >= 0x80 (corpus.cpp:20)
__host__ __device__ __forceinline__ bool word_byte(uint8_t c) {
    return (c >= '0' && c <= '9') || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c >= 0x80;
}
__host__ __device__ __forceinline__ uint8_t lower(uint8_t c) { return (c >= 'A' && c <= 'Z') ? c + 32 : c; }

// FNV-1a over the bytes, then a SplitMix64 finaliser (the sort key)
__host__ __device__ __forceinline__ uint64_t hash_bytes(const uint8_t* s, int64_t n, bool fold) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int64_t i = 0; i < n; ++i) {
        h ^= fold ? lower(s[i]) : s[i];
        h *= 0x100000001b3ull;
    }
    h ^= static_cast<uint64_t>(n) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 30;
    h *= 0xbf58476d1ce4e5b9ull;
    h ^= h >> 27;
    h *= 0x94d049bb133111ebull;
    h ^= h >> 31;
    return h;
}

__global__ void mark_bounds_kernel(const int64_t* __restrict__ offs, int64_t n_docs, uint8_t* __restrict__ bnd) {
    for (int64_t d = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; d <= n_docs;
         d += static_cast<int64_t>(gridDim.x) * blockDim.x)
        bnd[offs[d]] = 1;
}

// Token starts (bit 0) and ends (bit 1) per byte: a token is a maximal run of
// word bytes inside one document.
__global__ void token_flags_kernel(const uint8_t* __restrict__ text, int64_t T, const uint8_t* __restrict__ bnd,
                                   uint8_t* __restrict__ st, uint8_t* __restrict__ en) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool w = word_byte(text[i]);
        const bool prev_w = i > 0 && !bnd[i] && word_byte(text[i - 1]);
        const bool next_w = i + 1 < T && !bnd[i + 1] && word_byte(text[i + 1]);
        st[i] = w && !prev_w;
        en[i] = w && !next_w;
    }
}

// Per token: document (last offset <= start) and hash of the lowercased bytes.
__global__ void token_hash_kernel(const uint8_t* __restrict__ text, const int64_t* __restrict__ tb,
                                  const int64_t* __restrict__ te, int64_t M, const int64_t* __restrict__ offs,
                                  int64_t n_docs, uint64_t* __restrict__ key, uint32_t* __restrict__ tid,
                                  uint32_t* __restrict__ tdoc) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < M;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = tb[j];
        int64_t lo = 0, hi = n_docs;  // largest d with offs[d] <= b (and offs[d+1] > b)
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (offs[mid] <= b) lo = mid;
            else hi = mid;
        }
        tdoc[j] = static_cast<uint32_t>(lo);
        key[j] = hash_bytes(text + b, te[j] - b + 1, true);
        tid[j] = static_cast<uint32_t>(j);
    }
}

__device__ __forceinline__ bool same_token(const uint8_t* text, int64_t b1, int64_t n1, int64_t b2, int64_t n2) {
    if (n1 != n2) return false;
    for (int64_t i = 0; i < n1; ++i)
        if (lower(text[b1 + i]) != lower(text[b2 + i])) return false;
    return true;
}

// Group heads over the hash-sorted occurrences.
__global__ void head_kernel(const uint64_t* __restrict__ key, int64_t M, uint32_t* __restrict__ head) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < M;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        head[j] = (j == 0 || key[j] != key[j - 1]) ? 1u : 0u;
}

__global__ void dec_kernel(uint32_t* __restrict__ v, int64_t n) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[j] -= 1u;
}

// gid = inclusive scan of head − 1. Per occurrence: byte compare with the
// group's head occurrence; df += 1 at the head and at every document change.
__global__ void group_stats_kernel(const uint8_t* __restrict__ text, const int64_t* __restrict__ tb,
                                   const int64_t* __restrict__ te, const uint32_t* __restrict__ tid,
                                   const uint32_t* __restrict__ tdoc, const uint32_t* __restrict__ gid, int64_t M,
                                   const uint32_t* __restrict__ ghead_pos, uint32_t* __restrict__ df,
                                   unsigned long long* __restrict__ collision) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < M;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t g = gid[j];
        const uint32_t h = ghead_pos[g];  // sorted position of the head
        const uint32_t t = tid[j], t0 = tid[h];
        if (static_cast<uint32_t>(j) != h &&
            !same_token(text, tb[t], te[t] - tb[t] + 1, tb[t0], te[t0] - tb[t0] + 1))
            atomicOr(collision, 1ull);
        if (static_cast<uint32_t>(j) == h || tdoc[t] != tdoc[tid[j - 1]]) atomicAdd(df + g, 1u);
    }
}

__global__ void head_pos_kernel(const uint32_t* __restrict__ head, const uint32_t* __restrict__ gid, int64_t M,
                                uint32_t* __restrict__ ghead_pos) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < M;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (head[j]) ghead_pos[gid[j]] = static_cast<uint32_t>(j);
}

// Stop-word test per group (exact string equality with a stop word: the hash
// of the raw stop word equals the hash of the lowercased token, then bytes).
__global__ void stop_kernel(const uint8_t* __restrict__ text, const int64_t* __restrict__ tb,
                            const int64_t* __restrict__ te, const uint32_t* __restrict__ tid,
                            const uint64_t* __restrict__ key, const uint32_t* __restrict__ ghead_pos, uint32_t G,
                            const uint64_t* __restrict__ skey, const uint8_t* __restrict__ stext,
                            const int64_t* __restrict__ soff, const uint32_t* __restrict__ sidx, int64_t S,
                            uint8_t* __restrict__ is_stop) {
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < G;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t h = ghead_pos[g];
        const uint64_t k = key[h];
        int64_t lo = 0, hi = S;  // first stop key >= k
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (skey[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        bool stop = false;
        const uint32_t t = tid[h];
        const int64_t b = tb[t], n = te[t] - b + 1;
        for (int64_t q = lo; q < S && skey[q] == k && !stop; ++q) {
            const uint32_t w = sidx[q];
            const int64_t sb = soff[w], sn = soff[w + 1] - sb;
            if (sn != n) continue;
            bool eq = true;
            for (int64_t i = 0; i < n && eq; ++i) eq = lower(text[b + i]) == stext[sb + i];
            stop = eq;
        }
        is_stop[g] = stop ? 1 : 0;
    }
}

// A document is kept when one of its tokens is not a stop word (:106-113).
__global__ void doc_keep_kernel(const uint32_t* __restrict__ tid, const uint32_t* __restrict__ tdoc,
                                const uint32_t* __restrict__ gid, const uint8_t* __restrict__ is_stop, int64_t M,
                                uint32_t* __restrict__ keep) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < M;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (!is_stop[gid[j]]) keep[tdoc[tid[j]]] = 1u;
}

// Vocabulary membership (:55-58): not a stop word and df/N <= max_df in fp64.
// Emits the surviving groups' first-occurrence positions for the dim sort.
__global__ void vocab_select_kernel(const uint32_t* __restrict__ tid, const uint32_t* __restrict__ ghead_pos,
                                    const uint8_t* __restrict__ is_stop, const uint32_t* __restrict__ df, uint32_t G,
                                    double n_docs, double max_df, uint32_t* __restrict__ first,
                                    uint32_t* __restrict__ gsel, unsigned long long* __restrict__ n_sel) {
    for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < G;
         g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (is_stop[g]) continue;
        if (__ddiv_rn(static_cast<double>(df[g]), n_docs) > max_df) continue;
        const unsigned long long pos = atomicAdd(n_sel, 1ull);
        first[pos] = tid[ghead_pos[g]];
        gsel[pos] = static_cast<uint32_t>(g);
    }
}

__global__ void dim_assign_kernel(const uint32_t* __restrict__ gsorted, uint32_t V, uint32_t* __restrict__ gdim) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < V;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        gdim[gsorted[r]] = static_cast<uint32_t>(r);
}

// Per occurrence of a vocabulary term in a kept document: key = kept row ·
// 2^dim_bits + dim (sorting it orders rows, then dims).
__global__ void pair_keys_kernel(const uint32_t* __restrict__ tid, const uint32_t* __restrict__ tdoc,
                                 const uint32_t* __restrict__ gid, const uint32_t* __restrict__ gdim,
                                 const uint32_t* __restrict__ krow, int64_t M, int dim_bits,
                                 uint64_t* __restrict__ out, unsigned long long* __restrict__ n_out) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < M;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t dm = gdim[gid[j]];
        if (dm == kNone) continue;
        const uint32_t r = krow[tdoc[tid[j]]];  // kept (every vocabulary term lies in a kept document)
        const unsigned long long pos = atomicAdd(n_out, 1ull);
        out[pos] = (static_cast<uint64_t>(r) << dim_bits) | dm;
    }
}

// tf·idf per (row, dim) run; zero weights dropped (:77-78); row counts.
__global__ void weights_kernel(const uint64_t* __restrict__ ukey, const uint32_t* __restrict__ cnt, int64_t U,
                               int dim_bits, const double* __restrict__ idf, uint32_t* __restrict__ rdim,
                               double* __restrict__ rw, uint32_t* __restrict__ row_of, uint32_t* __restrict__ rcnt) {
    const uint64_t mask = (1ull << dim_bits) - 1ull;
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < U;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t dm = static_cast<uint32_t>(ukey[u] & mask);
        const uint32_t r = static_cast<uint32_t>(ukey[u] >> dim_bits);
        const double w = __dmul_rn(static_cast<double>(cnt[u]), idf[dm]);
        rdim[u] = dm;
        rw[u] = w;
        row_of[u] = r;
        if (w != 0.0) atomicAdd(rcnt + r, 1u);
    }
}

// Surviving (nonzero-weight) entries to their CSR positions (an exclusive scan
// of the nonzero flags over the row-major runs).
__global__ void nz_flag_kernel(const double* __restrict__ rw, int64_t U, uint32_t* __restrict__ f) {
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < U;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x)
        f[u] = rw[u] != 0.0;
}

__global__ void scatter_entries_kernel(const uint32_t* __restrict__ rdim, const double* __restrict__ rw,
                                       const uint64_t* __restrict__ pos, int64_t U, uint32_t* __restrict__ odim,
                                       double* __restrict__ ow) {
    for (int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; u < U;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (rw[u] != 0.0) {
            odim[pos[u]] = rdim[u];
            ow[pos[u]] = rw[u];
        }
}

__global__ void flag_pos_kernel(const uint32_t* __restrict__ c, int64_t n, uint8_t* __restrict__ f, int invert) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        f[i] = (c[i] != 0) != (invert != 0);
}

// ---------------------------------------------------------------- normalize --
// unit_step (sparse_vector.cpp:122-150): out = in / ‖in‖ with zero quotients
// dropped, after exact power-of-two rescales while the squared sum under- or
// overflows; an exact unit norm returns the input. Returns the output length,
// or -1 for "cannot normalize zero vector".
__device__ int64_t unit_step(const uint32_t* id, const double* iw, int64_t n, uint32_t* od, double* ow) {
    // the rescale loop works on (od, ow) once it has rescaled
    const uint32_t* cd = id;
    const double* cw = iw;
    for (;;) {
        double s = 0.0;
        for (int64_t q = 0; q < n; ++q) s = __dadd_rn(s, __dmul_rn(cw[q], cw[q]));
        const double nrm = __dsqrt_rn(s);
        if (nrm == 0.0 || isinf(nrm)) {
            const double scale = nrm == 0.0 ? 0x1p538 : 0x1p-538;
            int64_t m = 0;
            for (int64_t q = 0; q < n; ++q) {
                const double w = __dmul_rn(cw[q], scale);
                const uint32_t dd = cd[q];
                if (w != 0.0) {
                    od[m] = dd;
                    ow[m] = w;
                    ++m;
                }
            }
            if (m == 0) return -1;
            cd = od;
            cw = ow;
            n = m;
            continue;
        }
        if (nrm == 1.0) {
            if (cw != ow)
                for (int64_t q = 0; q < n; ++q) {
                    od[q] = cd[q];
                    ow[q] = cw[q];
                }
            return n;
        }
        int64_t m = 0;
        for (int64_t q = 0; q < n; ++q) {
            const double w = __ddiv_rn(cw[q], nrm);
            const uint32_t dd = cd[q];
            if (w != 0.0) {
                od[m] = dd;
                ow[m] = w;
                ++m;
            }
        }
        return m;
    }
}

__device__ __forceinline__ bool vec_eq(const uint32_t* ad, const double* aw, int64_t an, const uint32_t* bd,
                                       const double* bw, int64_t bn) {
    if (an != bn) return false;
    for (int64_t q = 0; q < an; ++q)
        if (ad[q] != bd[q] || aw[q] != bw[q]) return false;
    return true;
}

// lex_less (sparse_vector.cpp:112-117)
__device__ __forceinline__ bool lex_less(const double* aw, int64_t an, const double* bw, int64_t bn) {
    for (int64_t q = 0; q < an && q < bn; ++q)
        if (aw[q] != bw[q]) return aw[q] < bw[q];
    return an < bn;
}

__device__ __forceinline__ void vcopy(uint32_t* od, double* ow, const uint32_t* id, const double* iw, int64_t n) {
    for (int64_t q = 0; q < n; ++q) {
        od[q] = id[q];
        ow[q] = iw[q];
    }
}

// normalize (sparse_vector.cpp:158-183): one thread per row, the row's own
// slots hold `cur`; scratch A/B (same offsets) hold prev/next. Rows still
// moving after 8 passes go to the Brent kernel (flag 1). Output length in
// olen (rows may lose entries whose quotient underflows).
__global__ void normalize_kernel(const int64_t* __restrict__ rptr, int64_t R, uint32_t* dim, double* w,
                                 uint32_t* ad, double* aw, uint32_t* bd, double* bw, int64_t* __restrict__ olen,
                                 uint8_t* __restrict__ brent, unsigned long long* __restrict__ err) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < R;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t o = rptr[r];
        const int64_t n0 = rptr[r + 1] - o;
        brent[r] = 0;
        if (n0 == 1) {  // sqrt(w·w) may miss |w| by an ulp: the exact unit vector is ±1
            w[o] = w[o] > 0.0 ? 1.0 : -1.0;
            olen[r] = 1;
            continue;
        }
        uint32_t* cd = dim + o;
        double* cw = w + o;
        uint32_t* pd = ad + o;
        double* pw = aw + o;
        uint32_t* nd = bd + o;
        double* nw = bw + o;
        int64_t cn = n0, pn = -1;
        int64_t res = -2;  // -2: undecided
        // the three buffers rotate; `cur` ends in whichever holds it
        for (int pass = 0; pass < 8; ++pass) {
            const int64_t nn = unit_step(cd, cw, cn, nd, nw);
            if (nn < 0) {
                atomicOr(err, 1ull);
                res = 0;
                break;
            }
            if (vec_eq(nd, nw, nn, cd, cw, cn)) {  // fixpoint
                cd = nd;
                cw = nw;
                cn = nn;
                res = 1;
                break;
            }
            if (pn >= 0 && vec_eq(nd, nw, nn, pd, pw, pn)) {  // period-2: the lexicographically smaller
                if (lex_less(cw, cn, nw, nn)) { /* cur stays */
                } else {
                    cd = nd;
                    cw = nw;
                    cn = nn;
                }
                res = 1;
                break;
            }
            // prev = cur; cur = next (the old prev buffer becomes next's)
            uint32_t* td = pd;
            double* tw = pw;
            pd = cd;
            pw = cw;
            pn = cn;
            cd = nd;
            cw = nw;
            cn = nn;
            nd = td;
            nw = tw;
        }
        if (res == -2) brent[r] = 1;  // cur carried to the Brent kernel
        // the result (or Brent's start) into the row's own slots
        if (cd != dim + o) {
            // the row's own slots may hold prev (or next): copy cur over them
            vcopy(dim + o, w + o, cd, cw, cn);
        }
        olen[r] = res == 0 ? 0 : cn;
    }
}

// Brent's cycle search (sparse_vector.cpp:184-208) for rows whose orbit did not
// settle in 8 passes; one thread per such row, five row-sized buffers.
__global__ void brent_kernel(const uint32_t* __restrict__ rows, int64_t nr, const int64_t* __restrict__ rptr,
                             uint32_t* dim, double* w, const int64_t* __restrict__ soff, uint32_t* sd, double* sw,
                             int64_t* __restrict__ olen, unsigned long long* __restrict__ err) {
    for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nr;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t r = rows[q];
        const int64_t o = rptr[r], n0 = olen[r], L = rptr[r + 1] - o;
        uint32_t* bufd[5];
        double* bufw[5];
        for (int b = 0; b < 5; ++b) {
            bufd[b] = sd + soff[q] * 5 + b * L;
            bufw[b] = sw + soff[q] * 5 + b * L;
        }
        // 0 tortoise, 1 hare, 2 best, 3 walk, 4 temp
        int T = 0, H = 1, B = 2, W = 3, X = 4;
        int64_t tn = n0, hn, bn, wn;
        vcopy(bufd[T], bufw[T], dim + o, w + o, n0);
        hn = unit_step(bufd[T], bufw[T], tn, bufd[H], bufw[H]);
        if (hn < 0) {
            atomicOr(err, 1ull);
            olen[r] = 0;
            continue;
        }
        uint64_t power = 1, lam = 1;
        bool bad = false;
        while (!vec_eq(bufd[T], bufw[T], tn, bufd[H], bufw[H], hn)) {
            if (power == lam) {
                vcopy(bufd[T], bufw[T], bufd[H], bufw[H], hn);
                tn = hn;
                power *= 2;
                lam = 0;
            }
            const int64_t xn = unit_step(bufd[H], bufw[H], hn, bufd[X], bufw[X]);
            if (xn < 0) {
                bad = true;
                break;
            }
            const int t = H;
            H = X;
            X = t;
            hn = xn;
            ++lam;
        }
        if (bad) {
            atomicOr(err, 1ull);
            olen[r] = 0;
            continue;
        }
        vcopy(bufd[B], bufw[B], bufd[H], bufw[H], hn);
        bn = hn;
        wn = unit_step(bufd[H], bufw[H], hn, bufd[W], bufw[W]);
        for (uint64_t i = 1; i < lam && wn >= 0; ++i) {
            if (lex_less(bufw[W], wn, bufw[B], bn)) {
                vcopy(bufd[B], bufw[B], bufd[W], bufw[W], wn);
                bn = wn;
            }
            const int64_t xn = unit_step(bufd[W], bufw[W], wn, bufd[X], bufw[X]);
            const int t = W;
            W = X;
            X = t;
            wn = xn;
        }
        if (wn < 0) {
            atomicOr(err, 1ull);
            olen[r] = 0;
            continue;
        }
        vcopy(dim + o, w + o, bufd[B], bufw[B], bn);
        olen[r] = bn;
    }
}

__global__ void shrink_rows_kernel(const int64_t* __restrict__ rptr, const int64_t* __restrict__ nptr, int64_t R,
                                   const uint32_t* __restrict__ dim, const double* __restrict__ w,
                                   int32_t* __restrict__ od, double* __restrict__ ow) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < R;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = rptr[r], o = nptr[r], n = nptr[r + 1] - o;
        for (int64_t q = 0; q < n; ++q) {
            od[o + q] = static_cast<int32_t>(dim[s + q]);
            ow[o + q] = w[s + q];
        }
    }
}

// vocabulary strings in dim order (lowercased first occurrences)
__global__ void vocab_len_kernel(const uint32_t* __restrict__ gsorted, uint32_t V, const uint32_t* __restrict__ tid,
                                 const uint32_t* __restrict__ ghead_pos, const int64_t* __restrict__ tb,
                                 const int64_t* __restrict__ te, int64_t* __restrict__ vlen) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < V;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t t = tid[ghead_pos[gsorted[r]]];
        vlen[r] = te[t] - tb[t] + 1;
    }
}

__global__ void vocab_copy_kernel(const uint32_t* __restrict__ gsorted, uint32_t V, const uint32_t* __restrict__ tid,
                                  const uint32_t* __restrict__ ghead_pos, const int64_t* __restrict__ tb,
                                  const uint8_t* __restrict__ text, const int64_t* __restrict__ voff,
                                  uint8_t* __restrict__ out) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < V;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t t = tid[ghead_pos[gsorted[r]]];
        const int64_t b = tb[t], n = voff[r + 1] - voff[r];
        for (int64_t i = 0; i < n; ++i) out[voff[r] + i] = lower(text[b + i]);
    }
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ at, int64_t n,
                                  uint32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = src[at[i]];
}

}  // namespace vec
}  // namespace sskm_b200

// ----------------------------------------------------------------- host side --
struct sskm_vec {
    // results (host copies; the device work is done when sskm_vectorize returns)
    std::vector<int64_t> indptr;
    std::vector<int32_t> idx;
    std::vector<double> val;
    std::vector<int64_t> kept_docs;     // input document index of each row
    std::vector<int64_t> dropped_docs;  // the reference's order: pre-pass drops, then empty rows
    std::vector<uint32_t> doc_freq;     // by dim
    std::vector<int64_t> vocab_off;     // V + 1
    std::vector<char> vocab_text;
    uint32_t n_docs_vocab = 0;          // Vocabulary::n_docs
    double gpu_ms = 0.0;
    uint64_t launches = 0;
    uint64_t n_tokens = 0;
    uint64_t brent_rows = 0;
};

namespace {
using namespace sskm_b200;
using namespace sskm_b200::vec;

struct Launcher {
    int sms = 148;
    unsigned grid(int64_t work, int block = 256) const {
        const int64_t g = (work + block - 1) / block;
        return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g, static_cast<int64_t>(sms) * 16)));
    }
};

template <typename T>
void d2h(std::vector<T>& out, const T* p, size_t n, cudaStream_t s) {
    out.resize(n);
    if (n) CK(cudaMemcpyAsync(out.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

uint64_t d2h1(const unsigned long long* p, cudaStream_t s) {
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
}


template <typename T>
struct Widen {
    __host__ __device__ T operator()(uint32_t v) const { return static_cast<T>(v); }
};

template <typename F>
size_t cub_tmp(Buf<unsigned char>& tmp, F&& f) {
    size_t need = 0;
    CK(f(static_cast<void*>(nullptr), need));
    if (need > tmp.n) tmp.alloc(need + need / 4);
    need = tmp.n;
    CK(f(static_cast<void*>(tmp.p), need));
    return need;
}

// normalize (sparse_vector.cpp:158-209) of every row of a CSR held on the
// device, in place; olen[r] = the row's new length (entries whose quotient
// underflows vanish). Returns the number of rows that needed Brent's search.
uint64_t normalize_rows(const Launcher& L, cudaStream_t s, Buf<unsigned char>& tmp, unsigned long long* ctr,
                        unsigned long long* err, const int64_t* rptr, int64_t Rn, uint64_t nnz, uint32_t* dim,
                        double* w, int64_t* olen, uint64_t* launches) {
    Buf<uint32_t> ad, bd;
    Buf<double> aw, bw;
    Buf<uint8_t> brent;
    ad.alloc(nnz);
    bd.alloc(nnz);
    aw.alloc(nnz);
    bw.alloc(nnz);
    brent.alloc(Rn);
    normalize_kernel<<<L.grid(Rn, 128), 128, 0, s>>>(rptr, Rn, dim, w, ad.p, aw.p, bd.p, bw.p, olen, brent.p, err);
    CK_LAUNCH();
    ++*launches;
    ad.free();
    bd.free();
    aw.free();
    bw.free();
    Buf<uint32_t> brows;
    brows.alloc(Rn);
    CK(cudaMemsetAsync(ctr, 0, 8, s));
    thrust::counting_iterator<uint32_t> it(0);
    cub_tmp(tmp, [&](void* t, size_t& n) {
        return cub::DeviceSelect::Flagged(t, n, it, brent.p, brows.p, ctr, static_cast<int>(Rn), s);
    });
    ++*launches;
    const int64_t nb = static_cast<int64_t>(d2h1(ctr, s));
    if (nb) {
        // five row-sized buffers per such row
        std::vector<uint32_t> hb(nb);
        CK(cudaMemcpy(hb.data(), brows.p, 4 * nb, cudaMemcpyDeviceToHost));
        std::vector<int64_t> hp(Rn + 1);
        CK(cudaMemcpy(hp.data(), rptr, 8 * (Rn + 1), cudaMemcpyDeviceToHost));
        std::vector<int64_t> so(nb + 1, 0);
        for (int64_t q = 0; q < nb; ++q) so[q + 1] = so[q] + (hp[hb[q] + 1] - hp[hb[q]]);
        Buf<int64_t> d_so;
        Buf<uint32_t> sd;
        Buf<double> sw;
        d_so.alloc(nb + 1);
        sd.alloc(5 * so[nb]);
        sw.alloc(5 * so[nb]);
        CK(cudaMemcpyAsync(d_so.p, so.data(), 8 * (nb + 1), cudaMemcpyHostToDevice, s));
        brent_kernel<<<L.grid(nb, 64), 64, 0, s>>>(brows.p, nb, rptr, dim, w, d_so.p, sd.p, sw.p, olen, err);
        CK_LAUNCH();
        ++*launches;
        CK(cudaStreamSynchronize(s));
    }
    return static_cast<uint64_t>(nb);
}

void vectorize(int device, int64_t n_docs, const char* text, const int64_t* offs, int64_t n_stop,
               const char* stop_text, const int64_t* stop_offs, double max_df, sskm_vec* R) {
    // corpus.cpp:102: an empty corpus is a runtime_error
    if (n_docs <= 0) throw std::runtime_error("empty corpus");
    if (!offs || offs[0] != 0) throw std::invalid_argument("text offsets must start at 0");
    for (int64_t d = 0; d < n_docs; ++d)
        if (offs[d + 1] < offs[d]) throw std::invalid_argument("text offsets must be nondecreasing");
    if (n_docs >= (1ll << 31)) throw std::invalid_argument("too many documents");
    if (n_stop < 0 || (n_stop > 0 && (!stop_offs || stop_offs[0] != 0))) throw std::invalid_argument("bad stop words");
    const int64_t T = offs[n_docs];
    if (T > 0 && !text) throw std::invalid_argument("null text");
    int n_dev = 0;
    CK(cudaGetDeviceCount(&n_dev));
    if (device < 0 || device >= n_dev) throw std::invalid_argument("invalid CUDA device ordinal");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError("sskm_b200 requires an sm_100 (B200) device");
    Launcher L;
    L.sms = prop.multiProcessorCount;
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{s};
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    struct EvGuard {
        cudaEvent_t a, b;
        ~EvGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } eg{e0, e1};
    auto launched = [&]() {
        CK_LAUNCH();
        ++R->launches;
    };
    Buf<unsigned char> tmp;
    Buf<unsigned long long> cnt;
    cnt.alloc(8);
    CK(cudaMemsetAsync(cnt.p, 0, 64, s));
    CK(cudaEventRecord(e0, s));

    // ---- 1. bytes → token extents
    Buf<uint8_t> d_text;
    Buf<int64_t> d_off, tb, te;
    d_text.alloc(T + 1);
    d_off.alloc(n_docs + 1);
    if (T) CK(cudaMemcpyAsync(d_text.p, text, T, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(d_off.p, offs, (n_docs + 1) * 8, cudaMemcpyHostToDevice, s));
    int64_t M = 0;
    {
        Buf<uint8_t> bnd, fs, fe;
        bnd.alloc(T + 1);
        fs.alloc(T + 1);
        fe.alloc(T + 1);
        CK(cudaMemsetAsync(bnd.p, 0, T + 1, s));
        mark_bounds_kernel<<<L.grid(n_docs + 1), 256, 0, s>>>(d_off.p, n_docs, bnd.p);
        launched();
        if (T) {
            token_flags_kernel<<<L.grid(T), 256, 0, s>>>(d_text.p, T, bnd.p, fs.p, fe.p);
            launched();
        }
        tb.alloc(T / 2 + 1);
        te.alloc(T / 2 + 1);
        thrust::counting_iterator<int64_t> it(0);
        if (T) {
            cub_tmp(tmp, [&](void* t, size_t& n) {
                return cub::DeviceSelect::Flagged(t, n, it, fs.p, tb.p, cnt.p, T, s);
            });
            cub_tmp(tmp, [&](void* t, size_t& n) {
                return cub::DeviceSelect::Flagged(t, n, it, fe.p, te.p, cnt.p + 1, T, s);
            });
            R->launches += 2;
        }
        M = static_cast<int64_t>(d2h1(cnt.p, s));
    }
    if (M >= (1ll << 32) - 1) throw std::invalid_argument("too many tokens (2^32)");
    R->n_tokens = static_cast<uint64_t>(M);

    // ---- 2. per token: document and hash; stable sort by hash (corpus order
    // inside each group: the head is the first occurrence)
    Buf<uint64_t> key_s;
    Buf<uint32_t> tid_s, tdoc;
    key_s.alloc(M);
    tid_s.alloc(M);
    tdoc.alloc(M);
    if (M) {
        Buf<uint64_t> key;
        Buf<uint32_t> tid;
        key.alloc(M);
        tid.alloc(M);
        token_hash_kernel<<<L.grid(M), 256, 0, s>>>(d_text.p, tb.p, te.p, M, d_off.p, n_docs, key.p, tid.p, tdoc.p);
        launched();
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceRadixSort::SortPairs(t, n, key.p, key_s.p, tid.p, tid_s.p, static_cast<int>(M), 0, 64, s);
        });
        ++R->launches;
    }

    // ---- 3. groups = distinct terms
    Buf<uint32_t> gid, head;
    gid.alloc(M);
    head.alloc(M);
    uint32_t G = 0;
    if (M) {
        head_kernel<<<L.grid(M), 256, 0, s>>>(key_s.p, M, head.p);
        launched();
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceScan::InclusiveSum(t, n, head.p, gid.p, static_cast<int>(M), s);
        });
        ++R->launches;
        CK(cudaMemcpyAsync(&G, gid.p + M - 1, 4, cudaMemcpyDeviceToHost, s));
        dec_kernel<<<L.grid(M), 256, 0, s>>>(gid.p, M);
        launched();
        CK(cudaStreamSynchronize(s));
    }
    Buf<uint32_t> ghead, df;
    Buf<uint8_t> is_stop;
    ghead.alloc(G);
    df.alloc(G);
    is_stop.alloc(G);
    if (G) {
        head_pos_kernel<<<L.grid(M), 256, 0, s>>>(head.p, gid.p, M, ghead.p);
        launched();
        CK(cudaMemsetAsync(df.p, 0, 4ull * G, s));
        group_stats_kernel<<<L.grid(M), 256, 0, s>>>(d_text.p, tb.p, te.p, tid_s.p, tdoc.p, gid.p, M, ghead.p, df.p,
                                                    cnt.p + 2);
        launched();
        // stop words: raw-byte hashes, sorted on the host (a handful of strings)
        std::vector<std::pair<uint64_t, uint32_t>> sk;
        for (int64_t w = 0; w < n_stop; ++w)
            sk.emplace_back(hash_bytes(reinterpret_cast<const uint8_t*>(stop_text) + stop_offs[w],
                                       stop_offs[w + 1] - stop_offs[w], false),
                            static_cast<uint32_t>(w));
        std::sort(sk.begin(), sk.end());
        std::vector<uint64_t> skey(sk.size());
        std::vector<uint32_t> sidx(sk.size());
        for (size_t q = 0; q < sk.size(); ++q) {
            skey[q] = sk[q].first;
            sidx[q] = sk[q].second;
        }
        const int64_t SB = n_stop ? stop_offs[n_stop] : 0;
        Buf<uint64_t> d_skey;
        Buf<uint32_t> d_sidx;
        Buf<uint8_t> d_stext;
        Buf<int64_t> d_soff;
        d_skey.alloc(sk.size());
        d_sidx.alloc(sk.size());
        d_stext.alloc(SB + 1);
        d_soff.alloc(n_stop + 1);
        if (n_stop) {
            CK(cudaMemcpyAsync(d_skey.p, skey.data(), 8 * skey.size(), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(d_sidx.p, sidx.data(), 4 * sidx.size(), cudaMemcpyHostToDevice, s));
            if (SB) CK(cudaMemcpyAsync(d_stext.p, stop_text, SB, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(d_soff.p, stop_offs, 8 * (n_stop + 1), cudaMemcpyHostToDevice, s));
        }
        stop_kernel<<<L.grid(G), 256, 0, s>>>(d_text.p, tb.p, te.p, tid_s.p, key_s.p, ghead.p, G, d_skey.p,
                                              d_stext.p, d_soff.p, d_sidx.p, n_stop, is_stop.p);
        launched();
        CK(cudaStreamSynchronize(s));  // the stop-word buffers go out of scope
    }
    if (M && d2h1(cnt.p + 2, s))
        throw std::runtime_error("vectorize: 64-bit term hash collision between different terms");

    // kept documents (a non-stop token) and their row numbers
    head.free();
    Buf<uint32_t> keep, krow;
    keep.alloc(n_docs + 1);
    krow.alloc(n_docs + 1);
    CK(cudaMemsetAsync(keep.p, 0, 4ull * (n_docs + 1), s));
    if (M) {
        doc_keep_kernel<<<L.grid(M), 256, 0, s>>>(tid_s.p, tdoc.p, gid.p, is_stop.p, M, keep.p);
        launched();
    }
    cub_tmp(tmp, [&](void* t, size_t& n) {
        return cub::DeviceScan::ExclusiveSum(t, n, keep.p, krow.p, static_cast<int>(n_docs + 1), s);
    });
    ++R->launches;
    uint32_t N = 0;  // krow[n_docs] = kept documents
    CK(cudaMemcpyAsync(&N, krow.p + n_docs, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // :114-115: nothing left after the pre-pass
    if (N == 0) throw std::runtime_error("empty corpus");
    // build_vocabulary (:34-37)
    if (!(max_df > 0.0 && max_df <= 1.0)) throw std::invalid_argument("max_df_ratio must be in (0, 1]");
    R->n_docs_vocab = N;

    // ---- vocabulary: dims in first-occurrence order
    Buf<uint32_t> first, gsel, first_s, gsorted, gdim;
    first.alloc(G);
    gsel.alloc(G);
    first_s.alloc(G);
    gsorted.alloc(G);
    gdim.alloc(G);
    CK(cudaMemsetAsync(cnt.p + 3, 0, 8, s));
    if (G) {
        vocab_select_kernel<<<L.grid(G), 256, 0, s>>>(tid_s.p, ghead.p, is_stop.p, df.p, G, static_cast<double>(N),
                                                      max_df, first.p, gsel.p, cnt.p + 3);
        launched();
    }
    const uint32_t V = static_cast<uint32_t>(d2h1(cnt.p + 3, s));
    if (V == 0) throw std::runtime_error("empty vocabulary");
    int first_bits = 1;
    while (first_bits < 32 && (1ull << first_bits) < static_cast<uint64_t>(M)) ++first_bits;
    cub_tmp(tmp, [&](void* t, size_t& n) {
        return cub::DeviceRadixSort::SortPairs(t, n, first.p, first_s.p, gsel.p, gsorted.p, static_cast<int>(V), 0,
                                               first_bits, s);
    });
    ++R->launches;
    CK(cudaMemsetAsync(gdim.p, 0xFF, 4ull * G, s));
    dim_assign_kernel<<<L.grid(V), 256, 0, s>>>(gsorted.p, V, gdim.p);
    launched();
    // doc frequencies by dim → the idf table (host libm: the reference's std::log)
    {
        Buf<uint32_t> dfd;
        dfd.alloc(V);
        gather_u32_kernel<<<L.grid(V), 256, 0, s>>>(df.p, gsorted.p, V, dfd.p);
        launched();
        d2h(R->doc_freq, dfd.p, V, s);
        CK(cudaStreamSynchronize(s));
    }
    std::vector<double> idf(V);
    for (uint32_t v = 0; v < V; ++v)
        idf[v] = std::log(static_cast<double>(N) / static_cast<double>(R->doc_freq[v]));  // corpus.cpp:74-75
    Buf<double> d_idf;
    d_idf.alloc(V);
    CK(cudaMemcpyAsync(d_idf.p, idf.data(), 8ull * V, cudaMemcpyHostToDevice, s));
    // vocabulary strings
    {
        Buf<int64_t> vlen, voff;
        vlen.alloc(V + 1);
        voff.alloc(V + 1);
        vocab_len_kernel<<<L.grid(V), 256, 0, s>>>(gsorted.p, V, tid_s.p, ghead.p, tb.p, te.p, vlen.p);
        launched();
        CK(cudaMemsetAsync(vlen.p + V, 0, 8, s));
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceScan::ExclusiveSum(t, n, vlen.p, voff.p, static_cast<int>(V + 1), s);
        });
        ++R->launches;
        d2h(R->vocab_off, voff.p, V + 1, s);
        CK(cudaStreamSynchronize(s));
        Buf<uint8_t> vt;
        vt.alloc(R->vocab_off[V] + 1);
        vocab_copy_kernel<<<L.grid(V), 256, 0, s>>>(gsorted.p, V, tid_s.p, ghead.p, tb.p, d_text.p, voff.p, vt.p);
        launched();
        R->vocab_text.resize(R->vocab_off[V]);
        if (R->vocab_off[V])
            CK(cudaMemcpyAsync(R->vocab_text.data(), vt.p, R->vocab_off[V], cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }

    // ---- 4. tf per (kept row, dim): sort packed keys, run-length encode
    int dim_bits = 1;
    while ((1ull << dim_bits) < V) ++dim_bits;
    int row_bits = 1;
    while ((1ull << row_bits) < N) ++row_bits;
    if (dim_bits + row_bits > 64) throw std::runtime_error("vectorize: key overflow");
    Buf<uint64_t> pk, pk_s, ukey;
    Buf<uint32_t> runs;
    pk.alloc(M);
    pk_s.alloc(M);
    CK(cudaMemsetAsync(cnt.p + 4, 0, 16, s));
    if (M) {
        pair_keys_kernel<<<L.grid(M), 256, 0, s>>>(tid_s.p, tdoc.p, gid.p, gdim.p, krow.p, M, dim_bits, pk.p,
                                                   cnt.p + 4);
        launched();
    }
    const int64_t P = static_cast<int64_t>(d2h1(cnt.p + 4, s));
    // the token arrays are done
    key_s.free();
    gid.free();
    cub_tmp(tmp, [&](void* t, size_t& n) {
        return cub::DeviceRadixSort::SortKeys(t, n, pk.p, pk_s.p, static_cast<int>(P), 0, dim_bits + row_bits, s);
    });
    ++R->launches;
    pk.free();
    ukey.alloc(P);
    runs.alloc(P);
    cub_tmp(tmp, [&](void* t, size_t& n) {
        return cub::DeviceRunLengthEncode::Encode(t, n, pk_s.p, ukey.p, runs.p, cnt.p + 5, static_cast<int>(P), s);
    });
    ++R->launches;
    const int64_t U = static_cast<int64_t>(d2h1(cnt.p + 5, s));
    pk_s.free();
    Buf<uint32_t> rdim, row_of, rcnt, nzf;
    Buf<double> rw;
    rdim.alloc(U);
    row_of.alloc(U);
    rw.alloc(U);
    rcnt.alloc(N + 1);
    CK(cudaMemsetAsync(rcnt.p, 0, 4ull * (N + 1), s));
    if (U) {
        weights_kernel<<<L.grid(U), 256, 0, s>>>(ukey.p, runs.p, U, dim_bits, d_idf.p, rdim.p, rw.p, row_of.p,
                                                 rcnt.p);
        launched();
    }
    // nonzero entries to CSR positions (rows with no entries simply vanish)
    Buf<uint64_t> epos;
    Buf<uint32_t> odim;
    Buf<double> ow;
    epos.alloc(U + 1);
    nzf.alloc(U + 1);
    CK(cudaMemsetAsync(nzf.p + U, 0, 4, s));
    if (U) {
        nz_flag_kernel<<<L.grid(U), 256, 0, s>>>(rw.p, U, nzf.p);
        launched();
    }
    {
        thrust::transform_iterator<Widen<uint64_t>, const uint32_t*> nz64(nzf.p, Widen<uint64_t>());
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceScan::ExclusiveSum(t, n, nz64, epos.p, static_cast<int>(U + 1), s);
        });
        ++R->launches;
    }
    uint64_t nnz = 0;
    CK(cudaMemcpyAsync(&nnz, epos.p + U, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    odim.alloc(nnz);
    ow.alloc(nnz);
    if (U) {
        scatter_entries_kernel<<<L.grid(U), 256, 0, s>>>(rdim.p, rw.p, epos.p, U, odim.p, ow.p);
        launched();
    }
    rdim.free();
    rw.free();
    row_of.free();
    ukey.free();
    runs.free();
    // rows with entries (:124-129 drop the others)
    Buf<uint8_t> rflag;
    Buf<uint32_t> rows, rlen;
    rflag.alloc(N);
    rows.alloc(N);
    flag_pos_kernel<<<L.grid(N), 256, 0, s>>>(rcnt.p, N, rflag.p, 0);
    launched();
    {
        thrust::counting_iterator<uint32_t> it(0);
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceSelect::Flagged(t, n, it, rflag.p, rows.p, cnt.p + 6, static_cast<int>(N), s);
        });
        ++R->launches;
    }
    const int64_t Rn = static_cast<int64_t>(d2h1(cnt.p + 6, s));
    // :133: every row vectorised to zero
    if (Rn == 0) throw std::runtime_error("empty corpus");
    rlen.alloc(Rn + 1);
    gather_u32_kernel<<<L.grid(Rn), 256, 0, s>>>(rcnt.p, rows.p, Rn, rlen.p);
    launched();
    CK(cudaMemsetAsync(rlen.p + Rn, 0, 4, s));
    Buf<int64_t> rptr;
    rptr.alloc(Rn + 1);
    {
        thrust::transform_iterator<Widen<int64_t>, const uint32_t*> l64(rlen.p, Widen<int64_t>());
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceScan::ExclusiveSum(t, n, l64, rptr.p, static_cast<int>(Rn + 1), s);
        });
        ++R->launches;
    }

    // ---- 5. normalize each row
    Buf<int64_t> olen;
    olen.alloc(Rn + 1);
    R->brent_rows = normalize_rows(L, s, tmp, cnt.p + 6, cnt.p + 7, rptr.p, Rn, nnz, odim.p, ow.p, olen.p,
                                   &R->launches);
    if (d2h1(cnt.p + 7, s)) throw std::invalid_argument("cannot normalize zero vector");
    // final CSR (rows may have lost entries whose quotient underflowed)
    Buf<int64_t> nptr;
    Buf<int32_t> fidx;
    Buf<double> fval;
    nptr.alloc(Rn + 1);
    CK(cudaMemsetAsync(olen.p + Rn, 0, 8, s));
    cub_tmp(tmp, [&](void* t, size_t& n) {
        return cub::DeviceScan::ExclusiveSum(t, n, olen.p, nptr.p, static_cast<int>(Rn + 1), s);
    });
    ++R->launches;
    int64_t fnnz = 0;
    CK(cudaMemcpyAsync(&fnnz, nptr.p + Rn, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fidx.alloc(fnnz);
    fval.alloc(fnnz);
    shrink_rows_kernel<<<L.grid(Rn), 256, 0, s>>>(rptr.p, nptr.p, Rn, odim.p, ow.p, fidx.p, fval.p);
    launched();
    CK(cudaEventRecord(e1, s));
    d2h(R->indptr, nptr.p, Rn + 1, s);
    d2h(R->idx, fidx.p, fnnz, s);
    d2h(R->val, fval.p, fnnz, s);
    // row bookkeeping: kept docs (row -> input document), dropped docs
    std::vector<uint32_t> hkeep, hrows;
    d2h(hkeep, keep.p, n_docs, s);
    d2h(hrows, rows.p, Rn, s);
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    R->gpu_ms = ms;
    std::vector<int64_t> kept_doc;
    kept_doc.reserve(N);
    for (int64_t d = 0; d < n_docs; ++d) {
        if (hkeep[d]) kept_doc.push_back(d);
        else R->dropped_docs.push_back(d);  // pre-pass drops first (:116), in input order
    }
    R->kept_docs.resize(Rn);
    size_t q = 0;
    for (uint32_t r = 0; r < N; ++r) {
        if (q < hrows.size() && hrows[q] == r) {
            R->kept_docs[q++] = kept_doc[r];
        } else {
            R->dropped_docs.push_back(kept_doc[r]);  // then rows that vectorised to zero (:127)
        }
    }
}

}  // namespace

extern "C" {

int sskm_vectorize(int32_t device, int64_t n_docs, const char* text, const int64_t* text_offsets, int64_t n_stop,
                   const char* stop_text, const int64_t* stop_offsets, double max_df_ratio, sskm_vec** out) {
    try {
        if (!out) throw std::invalid_argument("null output handle");
        *out = nullptr;
        std::unique_ptr<sskm_vec> r(new sskm_vec());
        vectorize(device, n_docs, text, text_offsets, n_stop, stop_text, stop_offsets, max_df_ratio, r.get());
        *out = r.release();
        return SSKM_OK;
    } catch (const std::invalid_argument& e) {
        sskm_b200::set_last_error(e.what());
        return SSKM_EINVAL;
    } catch (const std::exception& e) {
        sskm_b200::set_last_error(e.what());
        return SSKM_ERUNTIME;
    }
}

int sskm_vec_sizes(const sskm_vec* v, int64_t* n_rows, int64_t* nnz, uint32_t* dims, uint32_t* n_docs_vocab,
                   int64_t* n_dropped, int64_t* vocab_bytes) {
    if (!v) {
        sskm_b200::set_last_error("null vectorize handle");
        return SSKM_EINVAL;
    }
    *n_rows = static_cast<int64_t>(v->indptr.size()) - 1;
    *nnz = static_cast<int64_t>(v->idx.size());
    *dims = static_cast<uint32_t>(v->doc_freq.size());
    *n_docs_vocab = v->n_docs_vocab;
    *n_dropped = static_cast<int64_t>(v->dropped_docs.size());
    *vocab_bytes = static_cast<int64_t>(v->vocab_text.size());
    return SSKM_OK;
}

int sskm_vec_export(const sskm_vec* v, int64_t* indptr, int32_t* indices, double* values, int64_t* kept_docs,
                    int64_t* dropped_docs, uint32_t* doc_freq, char* vocab_text, int64_t* vocab_offsets) {
    if (!v) {
        sskm_b200::set_last_error("null vectorize handle");
        return SSKM_EINVAL;
    }
    auto cp = [](auto* dst, const auto& src) {
        if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
    };
    cp(indptr, v->indptr);
    cp(indices, v->idx);
    cp(values, v->val);
    cp(kept_docs, v->kept_docs);
    cp(dropped_docs, v->dropped_docs);
    cp(doc_freq, v->doc_freq);
    cp(vocab_text, v->vocab_text);
    cp(vocab_offsets, v->vocab_off);
    return SSKM_OK;
}

int sskm_vec_stats(const sskm_vec* v, double* gpu_ms, uint64_t* launches, uint64_t* n_tokens, uint64_t* brent_rows) {
    if (!v) {
        sskm_b200::set_last_error("null vectorize handle");
        return SSKM_EINVAL;
    }
    *gpu_ms = v->gpu_ms;
    *launches = v->launches;
    *n_tokens = v->n_tokens;
    *brent_rows = v->brent_rows;
    return SSKM_OK;
}

int sskm_normalize_csr(int32_t device, int64_t n_rows, const int64_t* indptr, const int32_t* indices,
                       const double* values, int64_t* out_indptr, int32_t* out_indices, double* out_values) {
    try {
        if (n_rows < 0 || !indptr || indptr[0] != 0) throw std::invalid_argument("malformed CSR");
        const int64_t nnz = indptr[n_rows];
        for (int64_t r = 0; r < n_rows; ++r) {
            if (indptr[r + 1] < indptr[r]) throw std::invalid_argument("malformed CSR");
            if (indptr[r + 1] == indptr[r]) throw std::invalid_argument("cannot normalize zero vector");
        }
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw CudaError("sskm_b200 requires an sm_100 (B200) device");
        Launcher L;
        L.sms = prop.multiProcessorCount;
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{s};
        Buf<unsigned char> tmp;
        Buf<unsigned long long> cnt;
        Buf<int64_t> rptr, olen, nptr;
        Buf<uint32_t> dim;
        Buf<double> w;
        Buf<int32_t> fidx;
        Buf<double> fval;
        cnt.alloc(2);
        rptr.alloc(n_rows + 1);
        olen.alloc(n_rows + 1);
        nptr.alloc(n_rows + 1);
        dim.alloc(nnz);
        w.alloc(nnz);
        CK(cudaMemsetAsync(cnt.p, 0, 16, s));
        CK(cudaMemcpyAsync(rptr.p, indptr, 8 * (n_rows + 1), cudaMemcpyHostToDevice, s));
        if (nnz) {
            CK(cudaMemcpyAsync(dim.p, indices, 4 * nnz, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(w.p, values, 8 * nnz, cudaMemcpyHostToDevice, s));
        }
        uint64_t launches = 0;
        normalize_rows(L, s, tmp, cnt.p, cnt.p + 1, rptr.p, n_rows, nnz, dim.p, w.p, olen.p, &launches);
        if (d2h1(cnt.p + 1, s)) throw std::invalid_argument("cannot normalize zero vector");
        CK(cudaMemsetAsync(olen.p + n_rows, 0, 8, s));
        cub_tmp(tmp, [&](void* t, size_t& n) {
            return cub::DeviceScan::ExclusiveSum(t, n, olen.p, nptr.p, static_cast<int>(n_rows + 1), s);
        });
        int64_t fnnz = 0;
        CK(cudaMemcpyAsync(&fnnz, nptr.p + n_rows, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fidx.alloc(fnnz);
        fval.alloc(fnnz);
        shrink_rows_kernel<<<L.grid(n_rows), 256, 0, s>>>(rptr.p, nptr.p, n_rows, dim.p, w.p, fidx.p, fval.p);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(out_indptr, nptr.p, 8 * (n_rows + 1), cudaMemcpyDeviceToHost, s));
        if (fnnz) {
            CK(cudaMemcpyAsync(out_indices, fidx.p, 4 * fnnz, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(out_values, fval.p, 8 * fnnz, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        return SSKM_OK;
    } catch (const std::invalid_argument& e) {
        sskm_b200::set_last_error(e.what());
        return SSKM_EINVAL;
    } catch (const std::exception& e) {
        sskm_b200::set_last_error(e.what());
        return SSKM_ERUNTIME;
    }
}

int sskm_vec_free(sskm_vec* v) {
    delete v;
    return SSKM_OK;
}

}  // extern "C"
