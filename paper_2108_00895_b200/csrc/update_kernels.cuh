// Centroid-update kernels (replace compute_centroids, engine.cpp:137-195,
// DenseAccumulator, sparse_vector.cpp:237-274, normalize, :160-209, and
// detect_unchanged / sq_euclidean, engine.cpp:197-216, sparse_vector.cpp:211-235).
//
// Cluster sums are kept resident in HBM as exact fixed-point integers
// S[t][j] = Σ_{i∈j} round(x_it · 2^K) (int64, term-major like Cᵀ). Integer
// addition is associative, so the sums are bitwise independent of document
// order, thread schedule and GPU count, and an iteration only has to apply the
// rows of documents that MOVED (S_new = S_old + Σ_in − Σ_out exactly). K is
// chosen so that N·2^K < 2^62 for unit rows (|x| ≤ 1): no overflow is
// possible. Only the columns of clusters whose membership changed are then
// renormalised (fp64) and rewritten; a cluster with unchanged membership keeps
// a bitwise-identical column, which is exactly the reference's ncc_epsilon = 0
// "unchanged" condition.
//
// The squared column norms Q_j = Σ_t S[t][j]² are kept alongside as exact
// 128-bit integers (|S| ≤ 2^62 per column norm, so Q_j < 2^124): every atomic
// S += q returns the old value s, and Q_j += q·(2s + q) telescopes to the new
// Q_j whatever the order of the atomics. A renormalisation therefore reads
// only the columns it rewrites, once.
#pragma once

#include "common.cuh"

namespace sskm_b200 {

// Cluster sizes through a per-block shared histogram (k ≤ kSmemBins): one
// global atomic per nonzero bin and block instead of one per document.
constexpr uint32_t kSmemBins = 8192;
__global__ void __launch_bounds__(1024) counts_smem_kernel(const uint32_t* __restrict__ a, int64_t n, uint32_t k,
                                                           unsigned long long* __restrict__ counts, unsigned int* bad) {
    __shared__ unsigned int h[kSmemBins];
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) h[j] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t c = a[i];
        if (c >= k) {
            atomicOr(bad, 1u);
            continue;
        }
        atomicAdd(h + c, 1u);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x)
        if (h[j]) atomicAdd(counts + j, static_cast<unsigned long long>(h[j]));
}

__global__ void counts_kernel(const uint32_t* __restrict__ a, int64_t n, uint32_t k,
                              unsigned long long* __restrict__ counts, unsigned int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t c = a[i];
        if (c >= k) {
            atomicOr(bad, 1u);
            continue;
        }
        atomicAdd(counts + c, 1ull);
    }
}

__global__ void count_empty_kernel(const unsigned long long* __restrict__ counts, uint32_t k,
                                   unsigned int* n_empty) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
        if (counts[j] == 0) atomicAdd(n_empty, 1u);
}

// Documents whose cluster differs from the cluster their row is summed into.
__global__ void moved_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_sum,
                             int64_t n, uint32_t* __restrict__ moved,
                             unsigned long long* n_moved) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (a[i] != a_sum[i]) {
            const unsigned long long pos = atomicAdd(n_moved, 1ull);
            moved[pos] = static_cast<uint32_t>(i);
        }
    }
}

__device__ __forceinline__ long long quantize(float x, int K) {
    return __double2ll_rn(ldexp(static_cast<double>(x), K));
}

// S[t·ld + c] += q; returns q·(2·old + q), the exact change of Σ S² (128-bit).
// A nonzero result marks (t, c) in the bitmap nz (ld/32 words per row): the
// column rewrite reads only marked entries, and unmarks the ones it zeroes.
__device__ __forceinline__ __int128 add_sum(long long* S, uint64_t t, uint64_t ld, uint32_t c, long long q,
                                            unsigned int* nz) {
    const long long old = static_cast<long long>(
        atomicAdd(reinterpret_cast<unsigned long long*>(S + t * ld + c), static_cast<unsigned long long>(q)));
    if (old + q != 0) {
        unsigned int* w = nz + t * (ld >> 5) + (c >> 5);
        const unsigned int bit = 1u << (c & 31u);
        if (!(*w & bit)) atomicOr(w, bit);
    }
    return static_cast<__int128>(q) * (2 * static_cast<__int128>(old) + q);
}

__device__ __forceinline__ __int128 warp_sum128(__int128 v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xFFFFFFFFu, static_cast<unsigned long long>(v), off);
        const long long hi = __shfl_xor_sync(0xFFFFFFFFu, static_cast<long long>(v >> 64), off);
        v += (static_cast<__int128>(hi) << 64) | static_cast<__int128>(lo);
    }
    return v;
}

// Q (lo, hi words) += v modulo 2^128: the low word's carry, seen in the value
// its atomic returns, goes into the high word's atomic. The final pair is exact
// in any interleaving.
__device__ __forceinline__ void atomic_add128(unsigned long long* q, __int128 v) {
    const unsigned long long lo = static_cast<unsigned long long>(v);
    const unsigned long long hi = static_cast<unsigned long long>(v >> 64);
    const unsigned long long old = atomicAdd(q, lo);
    atomicAdd(q + 1, hi + (old + lo < old ? 1ull : 0ull));
}

// Apply the rows of moved documents: warp per document, lanes over its
// nonzeros (distinct terms, so no intra-row conflicts); integer atomics only.
// The document arrays (CSR, moved list, a, a_sum) may be a PEER device's shard,
// read over NVLink (multi-device contexts: every device applies every shard's
// moved rows to its own sums, no gather); a_sum_out (the local shard only, else
// nullptr) records the cluster each row is now summed into.
__global__ void delta_local_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                   const float* __restrict__ val, const uint32_t* __restrict__ moved,
                                   const unsigned long long* n_moved_p, const uint32_t* __restrict__ a,
                                   const uint32_t* a_sum, uint32_t* a_sum_out, long long* __restrict__ S,
                                   uint64_t ld, int K, uint8_t* __restrict__ touched,
                                   unsigned long long* __restrict__ Q, unsigned int* __restrict__ nz) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    const uint64_t n_moved = *n_moved_p;
    for (uint64_t m = gw; m < n_moved; m += nw) {
        const uint32_t i = moved[m];
        const uint32_t nc = a[i], oc = a_sum[i];
        const int64_t beg = indptr[i], end = indptr[i + 1];
        __int128 dn = 0, dold = 0;
        for (int64_t e = beg + lane; e < end; e += kWarp) {
            const long long q = quantize(val[e], K);
            const uint64_t t = static_cast<uint64_t>(idx[e]);
            dn += add_sum(S, t, ld, nc, q, nz);
            if (oc != kNone) dold += add_sum(S, t, ld, oc, -q, nz);
        }
        dn = warp_sum128(dn);
        if (oc != kNone) dold = warp_sum128(dold);
        if (lane == 0) {
            atomic_add128(Q + 2ull * nc, dn);
            touched[nc] = 1;
            if (oc != kNone) {
                atomic_add128(Q + 2ull * oc, dold);
                touched[oc] = 1;
            }
            if (a_sum_out) a_sum_out[i] = nc;
        }
    }
}

// Multi-GPU: apply the packed rows gathered from every rank (delta exchange).
__global__ void delta_packed_kernel(int64_t n_moved, const uint32_t* __restrict__ old_c,
                                    const uint32_t* __restrict__ new_c,
                                    const int64_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ idx, const float* __restrict__ val,
                                    long long* __restrict__ S, uint64_t ld, int K,
                                    uint8_t* __restrict__ touched, unsigned long long* __restrict__ Q,
                                    unsigned int* __restrict__ nz) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t m = gw; m < static_cast<uint64_t>(n_moved); m += nw) {
        const uint32_t nc = new_c[m], oc = old_c[m];
        __int128 dn = 0, dold = 0;
        for (int64_t e = row_ptr[m] + lane; e < row_ptr[m + 1]; e += kWarp) {
            const long long q = quantize(val[e], K);
            const uint64_t t = static_cast<uint64_t>(idx[e]);
            dn += add_sum(S, t, ld, nc, q, nz);
            if (oc != kNone) dold += add_sum(S, t, ld, oc, -q, nz);
        }
        dn = warp_sum128(dn);
        if (oc != kNone) dold = warp_sum128(dold);
        if (lane == 0) {
            atomic_add128(Q + 2ull * nc, dn);
            touched[nc] = 1;
            if (oc != kNone) {
                atomic_add128(Q + 2ull * oc, dold);
                touched[oc] = 1;
            }
        }
    }
}

// Multi-GPU delta exchange: per moved document its (old, new) clusters and
// row length, then (after a scan) the rows themselves, packed contiguously.
__global__ void moved_meta_kernel(const uint32_t* __restrict__ moved, const unsigned long long* n_moved_p,
                                  const int64_t* __restrict__ indptr, const uint32_t* __restrict__ a,
                                  const uint32_t* __restrict__ a_sum, int64_t* __restrict__ lens,
                                  uint32_t* __restrict__ old_c, uint32_t* __restrict__ new_c) {
    const uint64_t n_moved = *n_moved_p;
    for (uint64_t m = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; m <= n_moved;
         m += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (m == n_moved) {
            lens[m] = 0;
            continue;
        }
        const uint32_t i = moved[m];
        lens[m] = indptr[i + 1] - indptr[i];
        old_c[m] = a_sum[i];
        new_c[m] = a[i];
    }
}

__global__ void row_lens_kernel(const uint32_t* __restrict__ ids, int64_t n, const int64_t* __restrict__ indptr,
                                int64_t* __restrict__ lens) {
    for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m <= n;
         m += static_cast<int64_t>(gridDim.x) * blockDim.x)
        lens[m] = m == n ? 0 : indptr[ids[m] + 1] - indptr[ids[m]];
}

__global__ void pack_rows_kernel(const uint32_t* __restrict__ moved, int64_t n_moved,
                                 const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                 const float* __restrict__ val, const int64_t* __restrict__ offs,
                                 int32_t* __restrict__ lens32, int32_t* __restrict__ idx_out,
                                 float* __restrict__ val_out) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t m = gw; m < static_cast<uint64_t>(n_moved); m += nw) {
        const uint32_t i = moved[m];
        const int64_t b = indptr[i], e = indptr[i + 1], o = offs[m];
        for (int64_t q = b + lane; q < e; q += kWarp) {
            idx_out[o + (q - b)] = idx[q];
            val_out[o + (q - b)] = val[q];
        }
        if (lane == 0) lens32[m] = static_cast<int32_t>(e - b);
    }
}

__global__ void scatter_rows_kernel(const int64_t* __restrict__ rptr, const int32_t* __restrict__ ridx,
                                    const float* __restrict__ rval, uint32_t k, float* __restrict__ CT, uint64_t ld) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const uint32_t nw = gridDim.x * blockDim.x / kWarp;
    for (uint32_t j = gw; j < k; j += nw)
        for (int64_t e = rptr[j] + lane; e < rptr[j + 1]; e += kWarp) CT[static_cast<uint64_t>(ridx[e]) * ld + j] = rval[e];
}

// Ascending compaction of {j : flag(j)} in one block (k ≤ a few 1e5).
// want = 1: keep flag != 0; want = 0: keep flag == 0.
__global__ void compact_ids_kernel(const uint8_t* __restrict__ flags, uint32_t k, int want,
                                   uint32_t* __restrict__ ids, unsigned int* n_out) {
    __shared__ unsigned int warp_sums[32];
    __shared__ unsigned int base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (uint32_t j0 = 0; j0 < k; j0 += blockDim.x) {
        const uint32_t j = j0 + threadIdx.x;
        const unsigned int f = (j < k) && ((flags[j] != 0) == (want != 0));
        const unsigned int bal = __ballot_sync(0xFFFFFFFFu, f);
        const unsigned int pre = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) warp_sums[wid] = __popc(bal);
        __syncthreads();
        unsigned int off = 0;
        for (int w = 0; w < wid; ++w) off += warp_sums[w];
        if (f) ids[base + off + pre] = j;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int tot = 0;
            for (int w = 0; w < nwarps; ++w) tot += warp_sums[w];
            base += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_out = base;
}

#ifndef SSKM_ROW_BLOCK
#define SSKM_ROW_BLOCK 128  // measured on c1 (update ms): 512 -> 0.457, 256 -> 0.437, 128 -> 0.412, 64 -> 0.422, 32 -> 0.466
#endif
constexpr int kRowBlock = SSKM_ROW_BLOCK;  // rows per partial in the column reductions

// Rewrite of the touched columns: c = S · (1/‖S‖) in fp64, stored fp32, with
// the squared drift against the previous fp32 column as fixed-order partials.
// (The reference divides by the norm and iterates to a fixpoint,
// sparse_vector.cpp:160-209; both land within one fp64 ulp, below fp32
// resolution.) The norm comes straight from the exact 128-bit Q_j.
//
// Work by 32-column groups (the bitmap's words): a warp owns group g (lane =
// column 32g + lane) over one block of kRowBlock rows. Rows are visited 32 at a
// time through their bitmap words (lane r loads row r's word), and only rows
// where some touched column of the group is marked are read: an unmarked
// (t, j) has S = 0 and Cᵀ = 0, and on the TF-IDF corpora most (row, group)
// words are empty, so most of S and Cᵀ is never read. Per (row block, column)
// the drift partial is an ascending-row fp64 sum (unmarked rows would add
// exact zeros); the partials are reduced in a fixed association below.
// In-place maintenance of the bound screen's high postings (hipost_build_kernel
// with slack) for one rewritten row t of the warp's column group g. A row's
// list is its columns in ascending order (as built; hptr.w = (sorted length <<
// 16) | capacity) followed by columns appended since. An entry that changed and
// is high, or was, is looked up by its own lane (binary search in the sorted
// part, then the short tail): it gets its new value — or 0 when it is no longer
// high (the screen adds nothing for a zero pair, and the column keeps its place,
// so the order survives); a newly high entry not in the list is appended (a full
// list raises *ovf: the host rebuilds); a new low value raises L_t. The lists
// then hold exactly the entries >= thr of the new Cᵀ (plus zero pairs), and L_t
// stays an upper bound on the row's low weights.
// `hz` is the row's L_t bits, loaded with the round's other loads.
__device__ __forceinline__ void hipost_maintain(uint4* __restrict__ hptr, uint2* __restrict__ pairs, uint32_t t,
                                                uint32_t j, bool chg, float old, float cn, float thr, uint32_t hz,
                                                unsigned int* ovf) {
    const bool oh = chg && old != 0.f && fabsf(old) >= thr;
    const bool nh = chg && cn != 0.f && fabsf(cn) >= thr;
    const bool lo = chg && !nh && cn != 0.f;
    // the largest new low weight of the row's lanes against L_t (positive floats order as their bits)
    const uint32_t lomax = __reduce_max_sync(0xFFFFFFFFu, lo ? __float_as_uint(fabsf(cn)) : 0u);
    if (lomax > hz && (threadIdx.x & (kWarp - 1)) == 0) atomicMax(&hptr[t].z, lomax);
    if (!__any_sync(0xFFFFFFFFu, oh || nh)) return;
    if (!(oh || nh)) return;
    const uint4 h = hptr[t];
    const uint32_t sorted = h.w >> 16, cap = h.w & 0xFFFFu;
    const uint2* __restrict__ row = pairs + h.x;
    // binary search in the sorted part
    uint32_t a = 0, b = sorted;
    while (a < b) {
        const uint32_t m = (a + b) >> 1;
        if (row[m].x < j) a = m + 1; else b = m;
    }
    int slot = (a < sorted && row[a].x == j) ? static_cast<int>(a) : -1;
    if (slot < 0)  // appended since the last build
        for (uint32_t q = sorted; q < min(h.y, cap); ++q)
            if (row[q].x == j) {
                slot = static_cast<int>(q);
                break;
            }
    const uint2 e = make_uint2(j, nh ? __float_as_uint(cn) : 0u);
    if (slot >= 0) {
        pairs[h.x + slot] = e;
    } else if (nh) {
        const uint32_t pos = atomicAdd(&hptr[t].y, 1u);
        if (pos < cap)
            pairs[h.x + pos] = e;
        else
            atomicOr(ovf, 1u);
    } else {
        atomicOr(ovf, 1u);  // an entry that was high is not in the list: the lists no longer describe Cᵀ
    }
}

// R = marked rows per round (loads in flight per lane: 2 per row). Measured on c1
// (update ms per iteration): R = 1 0.53 (28 registers), R = 2 0.455 (32
// registers, 64 resident warps per SM), R = 3 0.70, R = 4 0.49 (48 registers),
// R = 8 0.61 (80 registers) — in every regime, from all columns rewritten to 4%
// of them: resident warps hide this kernel's latency better than loads per warp.
template <int R>
__global__ void __launch_bounds__(128) write_groups_kernel(const long long* __restrict__ S, float* __restrict__ CT,
                                                           uint64_t ld, uint32_t d, uint32_t k,
                                                           const uint8_t* __restrict__ touched,
                                                           const unsigned long long* __restrict__ Q,
                                                           double* __restrict__ part, unsigned int* zero_flag,
                                                           unsigned int* __restrict__ nz, uint4* __restrict__ hptr,
                                                           uint2* __restrict__ pairs, float hthr,
                                                           unsigned int* hp_ovf) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t g = blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
    const uint32_t rb = blockIdx.y;
    const uint32_t j = g * kWarp + lane;
    if (g * kWarp >= k) return;
    const bool active = j < k && touched[j] != 0;
    const unsigned amask = __ballot_sync(0xFFFFFFFFu, active);
    if (amask == 0) return;
    double inv = 0.0;
    if (active) {
        const double n2 = static_cast<double>(Q[2ull * j + 1]) * 0x1p64 + static_cast<double>(Q[2ull * j]);
        const double nrm = sqrt(n2);
        if (nrm == 0.0 && rb == 0) atomicOr(zero_flag, 1u);  // normalize() of the zero vector throws
        inv = nrm == 0.0 ? 0.0 : 1.0 / nrm;
    }
    const unsigned lbit = 1u << lane;
    const uint64_t wpr = ld >> 5;
    const uint32_t t0 = rb * kRowBlock, t1 = min(d, t0 + kRowBlock);
    double dr = 0.0;
    // the bitmap words of the next 32 rows are loaded one step ahead
    unsigned wr_n = t0 + lane < t1 ? nz[static_cast<uint64_t>(t0 + lane) * wpr + g] & amask : 0u;
    for (uint32_t tb = t0; tb < t1; tb += kWarp) {
        const unsigned wr = wr_n;
        {
            const uint32_t trn = tb + kWarp + lane;
            wr_n = trn < t1 ? nz[static_cast<uint64_t>(trn) * wpr + g] & amask : 0u;
        }
        unsigned rows = __ballot_sync(0xFFFFFFFFu, wr != 0);
        // R marked rows per round: all loads of a round before its stores
        while (rows) {
            int r[R];
            unsigned w[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                r[q] = rows ? __ffs(rows) - 1 : -1;
                if (rows) rows &= rows - 1;
                w[q] = __shfl_sync(0xFFFFFFFFu, wr, r[q] < 0 ? 0 : r[q]);
            }
            long long sv[R];
            float old[R];
            uint32_t hz[R];
            bool on[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                on[q] = r[q] >= 0 && (w[q] & lbit);
                const uint64_t o = static_cast<uint64_t>(tb + r[q]) * ld + j;
                sv[q] = on[q] ? __ldcs(S + o) : 0;
                old[q] = on[q] ? CT[o] : 0.f;
                hz[q] = (hthr > 0.f && r[q] >= 0) ? hptr[tb + r[q]].z : 0xFFFFFFFFu;
            }
            float cn[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                cn[q] = (!on[q] || sv[q] == 0) ? 0.f : static_cast<float>(static_cast<double>(sv[q]) * inv);
                if (!on[q]) continue;
                const uint64_t o = static_cast<uint64_t>(tb + r[q]) * ld + j;
                const double diff = static_cast<double>(cn[q]) - static_cast<double>(old[q]);
                dr = fma(diff, diff, dr);
                if (cn[q] != old[q]) CT[o] = cn[q];
                if (sv[q] == 0) atomicAnd(nz + static_cast<uint64_t>(tb + r[q]) * wpr + g, ~lbit);
            }
            if (hthr > 0.f) {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    if (r[q] < 0) break;
                    hipost_maintain(hptr, pairs, tb + r[q], j, on[q] && cn[q] != old[q], old[q], cn[q], hthr, hz[q],
                                    hp_ovf);
                }
            }
        }
    }
    if (active) part[static_cast<uint64_t>(rb) * k + j] = dr;
}

// Per touched column: the row-block partials of write_groups_kernel summed in a
// fixed association (32 segments of row blocks, each summed in order, then the
// 32 segment sums in order: deterministic); the count of touched columns.
// 1024 threads = 32 columns × 32 segments.
__global__ void __launch_bounds__(1024) reduce_groups_kernel(const double* __restrict__ part, uint32_t n_rb, uint32_t k,
                                                             const uint8_t* __restrict__ touched,
                                                             double* __restrict__ drift, unsigned int* n_rec) {
    __shared__ double sh[32][33];
    const uint32_t cl = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const uint32_t c = blockIdx.x * 32 + cl;
    const bool on = c < k && touched[c] != 0;
    const uint32_t per = (n_rb + 31) / 32;
    const uint32_t r0 = seg * per, r1 = min(n_rb, r0 + per);
    double s = 0.0;
    if (on) {
        uint32_t rb = r0;
        for (; rb + 4 <= r1; rb += 4) {  // loads first, then the in-order adds
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = part[static_cast<uint64_t>(rb + q) * k + c];
#pragma unroll
            for (int q = 0; q < 4; ++q) s += v[q];
        }
        for (; rb < r1; ++rb) s += part[static_cast<uint64_t>(rb) * k + c];
    }
    sh[seg][cl] = s;
    __syncthreads();
    if (seg == 0 && c < k) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) t += sh[q][cl];
        drift[c] = on ? t : 0.0;
    }
    if (seg == 0) {
        const unsigned b = __ballot_sync(0xFFFFFFFFu, on);
        if (cl == 0 && b) atomicAdd(n_rec, static_cast<unsigned>(__popc(b)));
    }
}

// Repair candidates: (orderable(sim), doc) keys for one stable radix sort.
__global__ void sim_keys_kernel(const double* __restrict__ sims, int64_t n,
                                unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        keys[i] = orderable(sims[i] + 0.0);  // +0.0 folds -0.0: the reference compares with <, where -0 == +0
        vals[i] = static_cast<uint32_t>(i);
    }
}

__global__ void gather_assign_kernel(const uint32_t* __restrict__ docs, uint32_t m,
                                     const uint32_t* __restrict__ a, uint32_t* __restrict__ out) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x)
        out[c] = a[docs[c]];
}

__global__ void apply_moves_kernel(const uint32_t* __restrict__ pairs, uint32_t m, uint32_t* __restrict__ a) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < m; c += gridDim.x * blockDim.x)
        a[pairs[2 * c]] = pairs[2 * c + 1];
}

// unchanged flags (detect_unchanged + repaired-forces-changed + iteration-1
// rule, engine.cpp:366-376) and max drift.
// same[j]: column j is bit-identical to its value before this update (not
// rewritten, or rewritten with zero drift: Σ(new − old)² = 0 in fp64 of fp32
// differences only for equal columns) — the bound screen's cached-similarity test.
__global__ void flags_kernel(uint32_t k, int first_iter, double eps, const uint8_t* __restrict__ repaired,
                             const double* __restrict__ drift, uint8_t* __restrict__ unchanged,
                             uint8_t* __restrict__ same, unsigned long long* max_drift_bits,
                             unsigned int* n_unchanged, uint8_t* __restrict__ touched) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        const double dj = drift[j];  // 0 for untouched columns
        same[j] = (!first_iter && !repaired[j] && dj == 0.0) ? 1 : 0;
        uint8_t u;
        if (first_iter) {
            u = 0;
        } else {
            u = (dj <= eps) ? 1 : 0;
            if (repaired[j]) u = 0;
            atomicMax(max_drift_bits, static_cast<unsigned long long>(__double_as_longlong(dj)));
        }
        unchanged[j] = u;
        if (u) atomicAdd(n_unchanged, 1u);
        touched[j] = 0;  // the update's last reader of the touched flags: cleared for the next one
    }
}

__global__ void scatter_pos_kernel(const uint32_t* __restrict__ ids, uint32_t n, uint32_t* __restrict__ pos) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
        pos[ids[c]] = c;
}

// Compact copy of the changed columns for the NCC scan: CC[t][c] = Cᵀ[t][ids[c]],
// zero-padded to ld_cc.
__global__ void gather_cols_kernel(const float* __restrict__ CT, uint64_t ld, uint32_t d,
                                   const uint32_t* __restrict__ ids, uint32_t n_ids,
                                   float* __restrict__ CC, uint64_t ld_cc) {
    const uint64_t total = static_cast<uint64_t>(d) * ld_cc;
    for (uint64_t o = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; o < total;
         o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t t = o / ld_cc;
        const uint32_t c = static_cast<uint32_t>(o - t * ld_cc);
        CC[o] = c < n_ids ? CT[t * ld + ids[c]] : 0.f;
    }
}

// Rows rows[0..n) of Cᵀ, densely packed: out[r][j] = Cᵀ[rows[r]][j], j < k.
__global__ void gather_rows_kernel(const float* __restrict__ CT, uint64_t ld, uint32_t k,
                                   const uint32_t* __restrict__ rows, uint32_t n, float* __restrict__ out) {
    const uint64_t total = static_cast<uint64_t>(n) * k;
    for (uint64_t o = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; o < total;
         o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = o / k;
        out[o] = CT[static_cast<uint64_t>(rows[r]) * ld + (o - r * k)];
    }
}

// Seed init (BASELINE): Cᵀ[:, j] = row of document seeds[j] (values as stored).
__global__ void scatter_seeds_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                     const float* __restrict__ val, const uint32_t* __restrict__ seeds,
                                     uint32_t k, float* __restrict__ CT, uint64_t ld) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
    const uint32_t nw = gridDim.x * blockDim.x / kWarp;
    for (uint32_t j = gw; j < k; j += nw) {
        const uint32_t s = seeds[j];
        for (int64_t e = indptr[s] + lane; e < indptr[s + 1]; e += kWarp)
            CT[static_cast<uint64_t>(idx[e]) * ld + j] = val[e];
    }
}

// max 2-norm of the seed rows (bound on the seed centroids' norms for the screen)
__global__ void seed_norm_max_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ val,
                                     const uint32_t* __restrict__ seeds, uint32_t k,
                                     unsigned long long* max_bits) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        const uint32_t s = seeds[j];
        double q = 0.0;
        for (int64_t e = indptr[s]; e < indptr[s + 1]; ++e) q = fma((double)val[e], (double)val[e], q);
        atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(sqrt(q))));
    }
}

// CSR validation: indices strictly ascending within a row and < dims, values
// nonzero, finite and |x| <= 1 (unit-length rows; the fixed-point bound).
__global__ void validate_csr_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                    const float* __restrict__ val, int64_t n, uint32_t dims,
                                    unsigned int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t b = indptr[i], e = indptr[i + 1];
        if (e < b) {
            atomicOr(bad, 1u);
            continue;
        }
        int32_t prev = -1;
        for (int64_t p = b; p < e; ++p) {
            const int32_t t = idx[p];
            const float x = val[p];
            if (t <= prev || t < 0 || static_cast<uint32_t>(t) >= dims) atomicOr(bad, 2u);
            if (x == 0.f) atomicOr(bad, 4u);
            if (!(fabsf(x) <= 1.0f)) atomicOr(bad, 8u);
            if (x < 0.f) atomicOr(bad, 16u);  // not an error: signed corpus (absolute screen bound)
            prev = t;
        }
    }
}

// k-means++ round (engine.cpp:86-96): sim_i = dot(x_i, seed) with the seed
// scattered densely; strictly-greater update keeps the lowest cluster id.
__global__ void kpp_round_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                 const float* __restrict__ val, int64_t n,
                                 const float* __restrict__ dense_seed, uint32_t cluster,
                                 uint32_t* __restrict__ a, double* __restrict__ sims) {
    // a thread per document, its entries in ascending order (the reference's
    // summation order); four gathers in flight per thread
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t beg = indptr[i], end = indptr[i + 1];
        double s = 0.0;
        int64_t e = beg;
        for (; e + 4 <= end; e += 4) {
            int32_t t[4];
            float x[4], c[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                t[r] = __ldg(idx + e + r);
                x[r] = __ldg(val + e + r);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) c[r] = __ldg(dense_seed + t[r]);
#pragma unroll
            for (int r = 0; r < 4; ++r) s = fma(static_cast<double>(x[r]), static_cast<double>(c[r]), s);
        }
        for (; e < end; ++e) s = fma(static_cast<double>(__ldg(val + e)), static_cast<double>(__ldg(dense_seed + __ldg(idx + e))), s);
        if (s > sims[i]) {
            sims[i] = s;
            a[i] = cluster;
        }
    }
}

// ---------------------------------------------------------- k-means++ --
// Device-resident k-means++ rounds (engine.cpp:99-128). The reference draws
// target = u · total and picks the first document whose running fp64 sum
// cum[i] (sequential, document order) exceeds it. The weights w_i are computed
// exactly as the reference does; their prefix is scanned in double-double
// (error ≤ n·2^-104 relative), and the sequential sums are bracketed:
// |cum[i] − E_i| ≤ γ(i+1)·E_i for nonnegative terms, so are the total and the
// target. The first index that may exceed the target (a) and the first that
// certainly does (b) are found by atomicMin over all documents; a == b decides
// the pick exactly. Otherwise (a near-tie with the target, the rare `pick ≥ n`
// and `total = 0` branches) the host replays the round sequentially.
struct KppDD {
    __device__ __forceinline__ double2 operator()(const double2& a, const double2& b) const {
        const double s = a.x + b.x;
        const double v = s - a.x;
        double e = (a.x - (s - v)) + (b.x - v);
        e += a.y + b.y;
        const double hi = s + e;
        return make_double2(hi, e - (hi - s));
    }
};

__global__ void kpp_weights_kernel(const double* __restrict__ sims, const uint8_t* __restrict__ chosen, int64_t n,
                                   double2* __restrict__ w) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double x = 0.0;
        if (!chosen[i]) {
            const double d = 1.0 - sims[i];
            if (d > 0.0) x = d * d;
        }
        w[i] = make_double2(x, 0.0);
    }
}

// out[0] = a, out[1] = b (initialised to n by the host)
__global__ void kpp_pick_kernel(const double2* __restrict__ E, int64_t n, double u, unsigned long long* out) {
    const double2 en = E[n - 1];
    const double tot = en.x + en.y;
    const double dd = static_cast<double>(n) * 0x1p-104 * tot;  // the double-double scan's own error
    const double gn = static_cast<double>(n) * 0x1p-53;
    const double err_n = gn * (1.0 + 2.0 * gn) * tot + dd;
    const double t_lo = u * (tot - err_n) * (1.0 - 0x1p-50);
    const double t_hi = u * (tot + err_n) * (1.0 + 0x1p-50);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 e = E[i];
        const double ei = e.x + e.y;
        const double g = static_cast<double>(i + 1) * 0x1p-53;
        const double err = (g * (1.0 + 2.0 * g) * ei + dd) * (1.0 + 0x1p-50) + 0x1p-1000;
        if (ei + err > t_lo) atomicMin(out + 0, static_cast<unsigned long long>(i));
        if (ei - err > t_hi) atomicMin(out + 1, static_cast<unsigned long long>(i));
    }
}

__global__ void set_u8_kernel(uint8_t* p, int64_t i, uint8_t v) { p[i] = v; }

__global__ void scatter_row_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ idx,
                                   const float* __restrict__ val, int64_t row, float* __restrict__ dense,
                                   int clear) {
    for (int64_t e = indptr[row] + threadIdx.x; e < indptr[row + 1]; e += blockDim.x)
        dense[idx[e]] = clear ? 0.f : val[e];
}

__global__ void fill_u32_kernel(uint32_t* p, int64_t n, uint32_t v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void fill_f64_kernel(double* p, int64_t n, double v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void local_sum_kernel(const double* __restrict__ x, int64_t n, double* part) {
    __shared__ double sh[256];
    double s = 0.0;
    const int64_t per = ceil_div(n, gridDim.x);
    const int64_t b0 = blockIdx.x * per, b1 = imin64(n, b0 + per);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += x[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

}  // namespace sskm_b200
