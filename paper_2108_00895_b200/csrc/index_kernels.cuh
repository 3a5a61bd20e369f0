// The reference's Lemma-1 pruning index (prune_index.cpp) evaluated on the GPU
// for `ncc+index` accounting. The exact NCC kernels produce the assignment (the
// index only prunes what cannot win); these kernels rebuild the
// index the reference would build from the same centroids and replay its
// queries, so index_queries, candidates_total and dot_products are the
// reference's (engine.cpp:277-298).
//
// Build (MultiIndex::build, prune_index.cpp:20-90), per iteration:
//   1. each centroid's support as keys (|w| descending, term ascending) —
//      exactly the reference's (w², dim) order: w is fp32, w² exact in fp64;
//   2. per (λ, centroid) the sequential fp64 sliding window over the squared
//      weights, in the reference's add/subtract order, giving min_overlap per
//      rank and the number J of emitted ranks;
//   3. per cluster tile, postings term -> (centroid, min_overlap) per λ.
// Query (IndexQuery::compute_overlaps / collect_candidates, :133-174), warp per
// document: overlap counts over the general postings, the smallest min_overlap
// per centroid over the λ postings of the document's terms, candidates =
// {c : min_overlap(c) <= overlap(c)}.
#pragma once

#include "common.cuh"

namespace sskm_b200 {

// Support sizes of row-chunk `blockIdx.y` for 32·blockDim.x/32 columns: thread
// (column c, chunk) counts the nonzeros of CT[t][c], t in the chunk
// (coalesced: a warp reads 32 consecutive columns of one row).
__global__ void idx_support_count_kernel(const float* __restrict__ CT, uint64_t ld, uint32_t d, uint32_t k,
                                         uint32_t rows_per_chunk, uint32_t n_chunks, uint32_t* __restrict__ cnt) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t ch = blockIdx.y;
    if (c >= k) return;
    const uint32_t t0 = ch * rows_per_chunk, t1 = min(d, t0 + rows_per_chunk);
    uint32_t n = 0;
    for (uint32_t t = t0; t < t1; ++t) n += __ldg(CT + static_cast<uint64_t>(t) * ld + c) != 0.f;
    cnt[static_cast<uint64_t>(c) * n_chunks + ch] = n;  // cluster-major, chunk-minor: one scan gives offsets
}

// Keys ((~|w| bits) << 32 | t) of every nonzero, cluster-major, ascending t
// within each (cluster, chunk) — deterministic positions from the scan.
__global__ void idx_support_fill_kernel(const float* __restrict__ CT, uint64_t ld, uint32_t d, uint32_t k,
                                        uint32_t rows_per_chunk, uint32_t n_chunks, const uint64_t* __restrict__ off,
                                        uint64_t* __restrict__ keys) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t ch = blockIdx.y;
    if (c >= k) return;
    const uint32_t t0 = ch * rows_per_chunk, t1 = min(d, t0 + rows_per_chunk);
    uint64_t pos = off[static_cast<uint64_t>(c) * n_chunks + ch];
    for (uint32_t t = t0; t < t1; ++t) {
        const float w = __ldg(CT + static_cast<uint64_t>(t) * ld + c);
        if (w != 0.f) {
            const uint32_t ab = __float_as_uint(w) & 0x7FFFFFFFu;
            keys[pos++] = (static_cast<uint64_t>(~ab) << 32) | t;
        }
    }
}

__device__ __forceinline__ double key_w2(uint64_t key) {
    const double w = static_cast<double>(__uint_as_float(~static_cast<uint32_t>(key >> 32)));
    return w * w;
}

// Sliding window of MultiIndex::build (prune_index.cpp:54-88), one warp per
// (λ, centroid), same fp64 operation order: grow the tail while sum < target,
// emit min_overlap = tail - j, subtract the head. Every lane runs the same
// sequential window (no divergence); the squared weights arrive 32 at a time
// in coalesced loads and are broadcast by shuffle.
__global__ void idx_window_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ cptr, uint32_t k,
                                  const double* __restrict__ lambdas, uint32_t n_lambdas, uint64_t nnz_c,
                                  uint32_t* __restrict__ mval, uint32_t* __restrict__ jlen) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t g = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    if (g >= static_cast<uint64_t>(k) * n_lambdas) return;
    const uint32_t l = static_cast<uint32_t>(g / k), c = static_cast<uint32_t>(g % k);
    const uint64_t base = cptr[c], m = cptr[c + 1] - base;
    const double lam = lambdas[l];
    const double target = lam * lam * (1.0 - 1e-9);  // kSumSlack (prune_index.cpp:16, :58)
    const uint64_t* kk = keys + base;
    uint32_t* mv = mval + static_cast<uint64_t>(l) * nnz_c + base;
    auto load = [&](uint64_t at) { return at + lane < m ? key_w2(__ldg(kk + at + lane)) : 0.0; };
    uint64_t tail = 0, tbase = 0, hbase = 0, j = 0;
    double tb = load(0), hb = tb;
    double sum = 0.0;
    for (; j < m; ++j) {
        while (tail < m && sum < target) {
            if (tail - tbase == kWarp) {
                tbase = tail;
                tb = load(tbase);
            }
            sum += __shfl_sync(0xFFFFFFFFu, tb, static_cast<int>(tail - tbase));
            ++tail;
        }
        if (sum < target) break;  // suffix exhausted
        if (j - hbase == kWarp) {
            hbase = j;
            hb = load(hbase);
        }
        if (static_cast<uint64_t>(lane) == j - hbase) mv[j] = static_cast<uint32_t>(tail - j);
        sum -= __shfl_sync(0xFFFFFFFFu, hb, static_cast<int>(j - hbase));
    }
    if (lane == 0) jlen[static_cast<uint64_t>(l) * k + c] = static_cast<uint32_t>(j);
}

// λ postings of the cluster tile [c0, c0 + kt): per term, the (local cluster,
// min_overlap) pairs of ranks < J. Warp per cluster; count then fill.
__global__ void idx_lam_count_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ cptr,
                                     const uint32_t* __restrict__ jlen_l, uint32_t c0, uint32_t kt,
                                     uint32_t* __restrict__ cnt) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    if (w >= kt) return;
    const uint32_t c = c0 + w;
    const uint64_t base = cptr[c];
    const uint32_t J = jlen_l[c];
    for (uint32_t j = lane; j < J; j += kWarp) atomicAdd(cnt + static_cast<uint32_t>(keys[base + j]), 1u);
}

__global__ void idx_lam_fill_kernel(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ cptr,
                                    const uint32_t* __restrict__ jlen_l, const uint32_t* __restrict__ mval_l,
                                    uint32_t c0, uint32_t kt, const uint32_t* __restrict__ lptr,
                                    uint32_t* __restrict__ fill, uint2* __restrict__ ent) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    if (w >= kt) return;
    const uint32_t c = c0 + w;
    const uint64_t base = cptr[c];
    const uint32_t J = jlen_l[c];
    for (uint32_t j = lane; j < J; j += kWarp) {
        const uint32_t t = static_cast<uint32_t>(keys[base + j]);
        const uint32_t slot = atomicAdd(fill + t, 1u);  // order inside a list is irrelevant (a min)
        ent[lptr[t] + slot] = make_uint2(w, mval_l[base + j]);
    }
}

struct IndexSelArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const float* CT;
    uint64_t ld_ct;
    int64_t n;
    const uint32_t* a_start;
    const double* sims_start;
    const uint8_t* unchanged;
    const uint8_t* rescan;     // per document: the unchanged list was rescanned
    const double* lambdas;
    uint32_t n_lambdas;
    uint64_t n_changed, n_unchanged;
    uint8_t* sel;              // chosen λ index, or 0xFF (no query)
    unsigned long long* counters;  // [0] queries, [1] NCC dots of the queried documents minus their refreshes
};

// select_threshold (prune_index.cpp:92-102) on the assign's baseline: the
// cached similarity, or the refreshed exact dot with the own centroid
// (engine.cpp:268-273, 279).
__global__ void __launch_bounds__(256) idx_select_kernel(IndexSelArgs p) {
    __shared__ __align__(16) double fold[256];
    double* wsm = fold + (threadIdx.x & ~(kWarp - 1));
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    unsigned long long q = 0, sub = 0;
    for (uint64_t i = gw; i < static_cast<uint64_t>(p.n); i += nw) {
        const uint32_t old_a = p.a_start[i];
        const bool own_changed = p.unchanged[old_a] == 0;
        const double best = own_changed ? doc_col_dot_sm(p.idx, p.val, p.indptr[i], p.indptr[i + 1], p.CT, p.ld_ct,
                                                         old_a, lane, wsm)
                                        : p.sims_start[i];
        uint32_t s = 0xFFu;
        for (uint32_t l = 0; l < p.n_lambdas; ++l) {
            if (p.lambdas[l] <= best) s = l;
            else break;
        }
        if (lane == 0) {
            p.sel[i] = static_cast<uint8_t>(s);
            if (s != 0xFFu) {
                ++q;
                // what the NCC accounting charged this document, minus the refresh
                // the index path charges too
                sub += p.n_changed + (p.rescan[i] ? p.n_unchanged : 0ull) - (own_changed ? 1ull : 0ull);
            }
        }
    }
    if (lane == 0) {
        if (q) atomicAdd(p.counters + 0, q);
        if (sub) atomicAdd(p.counters + 1, sub);
    }
}

__global__ void idx_compact_kernel(const uint8_t* __restrict__ sel, int64_t n, uint32_t l, uint32_t* __restrict__ list,
                                   unsigned long long* n_list) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool take = sel[i] == l;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, take);
        if (m == 0) continue;
        const int lane = threadIdx.x & (kWarp - 1);
        unsigned long long base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(n_list, static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
        if (take) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<uint32_t>(i);
    }
}

struct IndexQueryArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const uint32_t* gptr;      // general postings of the tile: term -> pairs (.x = local cluster)
    const uint2* gpairs;
    const uint32_t* lptr;      // λ postings of the tile: term -> (local cluster, min_overlap)
    const uint2* lent;
    uint32_t c0, kt;
    const uint32_t* list;      // documents querying this λ
    int64_t n_list;
    const uint32_t* a_start;
    const uint8_t* unchanged;
    const uint8_t* rescan;
    unsigned long long* counters;  // [2] candidates, [3] dots the index path evaluates (beyond the refresh)
};

// One warp per document: overlap counts and the smallest min_overlap per
// centroid of the tile in shared memory, then the candidate scan.
template <int KT>
__global__ void __launch_bounds__(256) idx_query_kernel(IndexQueryArgs p) {
    extern __shared__ uint32_t smem_q[];
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    uint32_t* cnt = smem_q + static_cast<size_t>(warp) * 2 * KT;
    uint32_t* mm = cnt + KT;
    unsigned long long cands = 0, dots = 0;
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * nwarps + warp; w < p.n_list;
         w += static_cast<int64_t>(gridDim.x) * nwarps) {
        const int64_t i = p.list[w];
        const int64_t beg = p.indptr[i], end = p.indptr[i + 1];
        for (int c = lane; c < KT; c += kWarp) {
            cnt[c] = 0u;
            mm[c] = 0xFFFFFFFFu;
        }
        __syncwarp();
        for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
            const int64_t e = e0 + lane;
            uint32_t gb = 0, ge = 0, lb = 0, le = 0;
            if (e < end) {
                const int32_t t = __ldg(p.idx + e);
                gb = __ldg(p.gptr + t);
                ge = __ldg(p.gptr + t + 1);
                lb = __ldg(p.lptr + t);
                le = __ldg(p.lptr + t + 1);
            }
            const int n = static_cast<int>(imin64(kWarp, end - e0));
            for (int j = 0; j < n; ++j) {
                const uint32_t qb = __shfl_sync(0xFFFFFFFFu, gb, j), qe = __shfl_sync(0xFFFFFFFFu, ge, j);
                for (uint32_t q = qb + lane; q < qe; q += kWarp) ++cnt[__ldg(&p.gpairs[q].x)];
                const uint32_t rb = __shfl_sync(0xFFFFFFFFu, lb, j), re = __shfl_sync(0xFFFFFFFFu, le, j);
                for (uint32_t q = rb + lane; q < re; q += kWarp) {
                    const uint2 en = p.lent[q];
                    mm[en.x] = min(mm[en.x], en.y);
                }
                __syncwarp();  // a cluster occurs once per list; lists of later terms may repeat it
            }
        }
        const uint32_t old_a = p.a_start[i];
        const bool rescan = p.rescan[i] != 0;
        uint32_t nc = 0, nd = 0;
        for (uint32_t c = lane; c < p.kt; c += kWarp) {
            if (mm[c] <= cnt[c]) {
                ++nc;
                const uint32_t id = p.c0 + c;
                if (id != old_a) nd += (p.unchanged[id] == 0 || rescan) ? 1u : 0u;  // engine.cpp:287-297
            }
        }
        cands += nc;
        dots += nd;
        __syncwarp();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cands += __shfl_xor_sync(0xFFFFFFFFu, cands, off);
        dots += __shfl_xor_sync(0xFFFFFFFFu, dots, off);
    }
    if (lane == 0) {
        if (cands) atomicAdd(p.counters + 2, cands);
        if (dots) atomicAdd(p.counters + 3, dots);
    }
}

// Per-document "the unchanged list was rescanned" (engine.cpp:287-297, 303):
// own centroid changed and the changed scan did not beat the cached sim.
__global__ void idx_rescan_formula_kernel(const uint32_t* __restrict__ a_start, const double* __restrict__ sims_start,
                                          const double* __restrict__ sims, const uint8_t* __restrict__ unchanged,
                                          int64_t n, uint8_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        flag[i] = unchanged[a_start[i]] == 0 && !(sims[i] > sims_start[i]);
}

__global__ void idx_rescan_scatter_kernel(const uint32_t* __restrict__ list, int64_t n_list,
                                          uint8_t* __restrict__ flag) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n_list;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        flag[list[j]] = 1;
}

}  // namespace sskm_b200
