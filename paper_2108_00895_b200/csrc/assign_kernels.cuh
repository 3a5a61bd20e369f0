// Assignment kernels (replace assign(), engine.cpp:218-322, and dot(),
// sparse_vector.cpp:45-108).
//
// Layout: centroids are stored transposed and dense, Cᵀ[t][j] fp32 with row
// stride `ld` floats (term-major, d × ld, ld = k rounded up to 128), so each
// document nonzero t streams one contiguous k-row segment with coalesced
// 128-bit loads. One warp owns one document; each lane owns V adjacent
// columns of the current 32·V-wide column tile and accumulates in fp64 in the
// document's ascending term order. Products of two fp32 values are exact in
// fp64 and zero centroid entries add exact zeros, so every (doc, centroid)
// similarity is bit-identical to the reference's merge/gallop dot over the
// same fp32-valued centroid (sparse_vector.cpp:72-101). The argmax is fused:
// a lane-local compare over its V columns, then a warp-shuffle reduction under
// the reference tie rule, carried across tiles in registers — no N×k matrix
// ever reaches memory.
#pragma once

#include "common.cuh"

namespace sskm_b200 {

template <int V>
struct VecT;
template <>
struct VecT<1> {
    using type = float;
};
template <>
struct VecT<2> {
    using type = float2;
};
template <>
struct VecT<4> {
    using type = float4;
};

template <int V>
__device__ __forceinline__ void unpack(const typename VecT<V>::type& t, float (&c)[V]) {
    if constexpr (V == 4) {
        c[0] = t.x;
        c[1] = t.y;
        c[2] = t.z;
        c[3] = t.w;
    } else if constexpr (V == 2) {
        c[0] = t.x;
        c[1] = t.y;
    } else {
        c[0] = t;
    }
}

// Per-lane fp64 partial dots of one document against columns
// [col0 + lane·V, col0 + lane·V + V) of M, in ascending entry order.
//
// Rows are addressed in V-float vector units with a 32-bit per-entry offset
// (t · ld/V) computed once per entry by its owning lane, so the hot loop is one
// shuffle + one wide load per entry. Loads are issued U at a time ahead of
// their consumers (a compiler barrier keeps ptxas from re-interleaving them),
// giving U independent L2 requests in flight per warp. The last batch of a
// 32-entry chunk runs over lanes past the row end with x = 0, which adds exact
// zeros and so leaves every fp64 sum bit-identical.
template <int V, int U>
__device__ __forceinline__ void doc_tile_dots(const int32_t* __restrict__ idx,
                                              const float* __restrict__ val, int64_t beg,
                                              int64_t end, const float* __restrict__ M,
                                              uint64_t ld, uint32_t col0, int lane,
                                              double (&acc)[V]) {
    using VT = typename VecT<V>::type;
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0;
    const VT* base = reinterpret_cast<const VT*>(M + col0) + lane;
    const uint32_t ldv = static_cast<uint32_t>(ld / V);
    for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
        const int64_t e = e0 + lane;
        uint32_t off_l = 0;
        float x_l = 0.f;
        if (e < end) {
            off_l = static_cast<uint32_t>(__ldg(idx + e)) * ldv;
            x_l = __ldg(val + e);
        }
        const int n = static_cast<int>(imin64(kWarp, end - e0));
        for (int j = 0; j < n; j += U) {
            VT c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t off = __shfl_sync(0xFFFFFFFFu, off_l, (j + u) & (kWarp - 1));
                c[u] = __ldg(base + off);
            }
            asm volatile("" ::: "memory");
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double x = static_cast<double>(__shfl_sync(0xFFFFFFFFu, x_l, (j + u) & (kWarp - 1)));
                float cf[V];
                unpack<V>(c[u], cf);
                // lanes j+u >= n hold x = 0 (past the row end): exact no-ops
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = fma(x, static_cast<double>(cf[v]), acc[v]);
            }
        }
    }
}

// Exact single dot x_i · Cᵀ[:, col] in ascending entry order (the NCC refresh
// of the own centroid, engine.cpp:271-273): lanes gather in parallel, then
// every lane folds the same sequence so the sum order matches the scan.
__device__ __forceinline__ double doc_col_dot(const int32_t* __restrict__ idx,
                                              const float* __restrict__ val, int64_t beg,
                                              int64_t end, const float* __restrict__ M,
                                              uint64_t ld, uint32_t col, int lane) {
    // all gathers of up to 4 chunks (128 entries) are issued before the fold,
    // so one latency covers most documents; the fold order is unchanged
    constexpr int kChunks = 4;
    double s = 0.0;
    for (int64_t e0 = beg; e0 < end; e0 += kChunks * kWarp) {
        float xs[kChunks], cs[kChunks];
        int32_t ts[kChunks];
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            const int64_t e = e0 + c * kWarp + lane;
            xs[c] = 0.f;
            ts[c] = -1;
            if (e < end) {
                ts[c] = __ldg(idx + e);
                xs[c] = __ldg(val + e);
            }
        }
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
            cs[c] = ts[c] >= 0 ? __ldg(M + static_cast<uint64_t>(ts[c]) * ld + col) : 0.f;
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            const int64_t c0 = e0 + c * kWarp;
            if (c0 >= end) break;
            const int n = static_cast<int>(imin64(kWarp, end - c0));
            for (int j = 0; j < n; ++j) {
                const double x = static_cast<double>(__shfl_sync(0xFFFFFFFFu, xs[c], j));
                const double cv = static_cast<double>(__shfl_sync(0xFFFFFFFFu, cs[c], j));
                s = fma(x, cv, s);
            }
        }
    }
    return s;
}

// doc_col_dot with the fold through a per-warp shared buffer: the lanes form
// the exact fp64 products x_t*c_t in parallel (fp32 x fp32 is exact in fp64, so
// s + p_t is bit-identical to fma(x_t, c_t, s)), then every lane folds them in
// ascending term order from broadcast 16-byte shared loads.
__device__ __forceinline__ double doc_col_dot_sm(const int32_t* __restrict__ idx,
                                                 const float* __restrict__ val, int64_t beg,
                                                 int64_t end, const float* __restrict__ M,
                                                 uint64_t ld, uint32_t col, int lane, double* wsm) {
    constexpr int kChunks = 4;
    double s = 0.0;
    for (int64_t e0 = beg; e0 < end; e0 += kChunks * kWarp) {
        float xs[kChunks];
        int32_t ts[kChunks];
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            const int64_t e = e0 + c * kWarp + lane;
            xs[c] = 0.f;
            ts[c] = -1;
            if (e < end) {
                ts[c] = __ldg(idx + e);
                xs[c] = __ldg(val + e);
            }
        }
        double ps[kChunks];
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            const float cv = ts[c] >= 0 ? __ldg(M + static_cast<uint64_t>(ts[c]) * ld + col) : 0.f;
            ps[c] = static_cast<double>(xs[c]) * static_cast<double>(cv);
        }
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
            const int64_t c0 = e0 + c * kWarp;
            if (c0 >= end) break;
            const int n = static_cast<int>(imin64(kWarp, end - c0));
            wsm[lane] = ps[c];
            __syncwarp();
            const double2* w2 = reinterpret_cast<const double2*>(wsm);
            if (n == kWarp) {
#pragma unroll
                for (int j = 0; j < kWarp / 2; ++j) {
                    const double2 q = w2[j];
                    s += q.x;
                    s += q.y;
                }
            } else {
                int j = 0;
                for (; j + 2 <= n; j += 2) {
                    const double2 q = w2[j >> 1];
                    s += q.x;
                    s += q.y;
                }
                if (j < n) s += wsm[j];
            }
            __syncwarp();
        }
    }
    return s;
}

enum ScanInit : int {
    kInitFull = 0,    // best = -2, arg = 0 (engine.cpp:252-253), all columns
    kInitNcc = 1,     // NCC pass A: cache or refreshed own dot, changed columns only
    kInitRescan = 2,  // NCC pass B: from pass A's result, all columns
};

// One column tile of one assignment pass. The pass over all k columns is
// issued tile-major (one launch per tile) so that the tile's slice of Cᵀ —
// d × W fp32, sized to stay resident in the 126 MB L2 — is streamed from HBM
// about once per iteration while the CSR rows stream past it; the per-document
// running (best, arg) lives in a[] / sims[] between tiles.
struct TileArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const float* M;            // matrix scanned (Cᵀ, or the compact changed-column copy)
    uint64_t ld;               // row stride of M
    uint32_t col0;             // first column of this launch's tiles
    uint32_t span;             // columns this launch covers (one tile of 32·V, or more: short work lists)
    uint32_t ncols;            // total columns of M (tile may be partial)
    const uint32_t* col_ids;   // cluster id per column of M (nullptr = identity)
    const uint32_t* order;     // work item -> document (nullptr = identity)
    int64_t n_work;
    int first, last;           // first / last tile of the pass
    uint32_t* a;               // running argmax (in/out)
    double* sims;              // running max (in/out)
    // NCC pass A
    const uint8_t* unchanged;  // per cluster
    const uint32_t* a_start;   // assignment at the start of the step
    const double* sims_start;  // cached sims at the start of the step
    const float* CT;           // full Cᵀ (own-centroid refresh)
    uint64_t ld_ct;
    uint32_t* rescan_list;
    unsigned long long* n_rescan;
};

template <int V, int INIT, int U>
__global__ void __launch_bounds__(256, 2) assign_tile_kernel(TileArgs p) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    // contiguous chunk of the (cluster-ordered) work list per block: warps of a
    // block, resident on one SM, share the hot rows of their cluster in L1
    const int64_t chunk = static_cast<int64_t>(ceil_div(p.n_work, gridDim.x));
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t w1 = imin64(p.n_work, w0 + chunk);
    for (int64_t w = w0 + warp; w < w1; w += nwarps) {
        const int64_t i = p.order ? static_cast<int64_t>(__ldg(p.order + w)) : w;
        const int64_t beg = __ldg(p.indptr + i), end = __ldg(p.indptr + i + 1);
        double best;
        uint32_t arg;
        if (!p.first || INIT == kInitRescan) {
            best = p.sims[i];
            arg = p.a[i];
        } else if constexpr (INIT == kInitFull) {
            best = -2.0;
            arg = 0;
        } else {
            const uint32_t old_a = p.a_start[i];
            const bool own_changed = p.unchanged[old_a] == 0;
            // unchanged own centroid: the cache is current (engine.cpp:268-270);
            // otherwise refresh the baseline (engine.cpp:271-273)
            best = own_changed ? doc_col_dot(p.idx, p.val, beg, end, p.CT, p.ld_ct, old_a, lane)
                               : p.sims_start[i];
            arg = old_a;
        }
        {
            // each lane keeps its own running (max, id) over the launch's tiles
            // (the tie rule is a total order: any combination order gives the
            // same winner), combined across the warp once
            double lb = best;
            uint32_t la = arg;
            const uint32_t cend = min(p.ncols, p.col0 + p.span);
            for (uint32_t c0 = p.col0; c0 < cend; c0 += 32u * V) {
                double acc[V];
                doc_tile_dots<V, U>(p.idx, p.val, beg, end, p.M, p.ld, c0, lane, acc);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const uint32_t col = c0 + static_cast<uint32_t>(lane) * V + v;
                    if (col < p.ncols) {
                        const uint32_t id = p.col_ids ? __ldg(p.col_ids + col) : col;
                        if (better(acc[v], id, lb, la)) {
                            lb = acc[v];
                            la = id;
                        }
                    }
                }
            }
            warp_argmax(lb, la);
            best = lb;
            arg = la;
        }
        if (lane == 0) {
            p.a[i] = arg;
            p.sims[i] = best;
            if constexpr (INIT == kInitNcc) {
                // the refreshed scan did not beat the cached max: unchanged
                // centroids may tie or exceed it (engine.cpp:303-305)
                if (p.last) {
                    const uint32_t old_a = p.a_start[i];
                    if (p.unchanged[old_a] == 0 && !(best > p.sims_start[i])) {
                        const unsigned long long pos = atomicAdd(p.n_rescan, 1ull);
                        p.rescan_list[pos] = static_cast<uint32_t>(i);
                    }
                }
            }
        }
    }
}

// Short work lists (what the screens leave: hundreds of documents against up to
// 50,000 columns): a warp per (document, column span), so the scan's
// parallelism comes from the columns too; each warp leaves its span's exact
// (max, id) and a second kernel folds the spans into the running state with
// the same total order.
template <int V, int U>
__global__ void __launch_bounds__(256, 2) assign_span_kernel(TileArgs p, uint32_t n_spans, double* __restrict__ part_s,
                                                             uint32_t* __restrict__ part_a) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    const uint32_t sp = blockIdx.y;
    const uint32_t c_beg = sp * p.span, c_end = min(p.ncols, c_beg + p.span);
    for (int64_t w = static_cast<int64_t>(blockIdx.x) * nwarps + warp; w < p.n_work;
         w += static_cast<int64_t>(gridDim.x) * nwarps) {
        const int64_t i = p.order ? static_cast<int64_t>(__ldg(p.order + w)) : w;
        const int64_t beg = __ldg(p.indptr + i), end = __ldg(p.indptr + i + 1);
        double lb = -1e300;
        uint32_t la = kNone;
        for (uint32_t c0 = c_beg; c0 < c_end; c0 += 32u * V) {
            double acc[V];
            doc_tile_dots<V, U>(p.idx, p.val, beg, end, p.M, p.ld, c0, lane, acc);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const uint32_t col = c0 + static_cast<uint32_t>(lane) * V + v;
                if (col < c_end) {
                    const uint32_t id = p.col_ids ? __ldg(p.col_ids + col) : col;
                    if (better(acc[v], id, lb, la)) {
                        lb = acc[v];
                        la = id;
                    }
                }
            }
        }
        warp_argmax(lb, la);
        if (lane == 0) {
            part_s[w * n_spans + sp] = lb;
            part_a[w * n_spans + sp] = la;
        }
    }
}

template <int INIT>
__global__ void assign_span_reduce_kernel(TileArgs p, uint32_t n_spans, const double* __restrict__ part_s,
                                          const uint32_t* __restrict__ part_a) {
    static_assert(INIT != kInitNcc, "the NCC pass refreshes its baseline in the tile kernel");
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < p.n_work;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = p.order ? static_cast<int64_t>(p.order[w]) : w;
        double best = INIT == kInitFull ? -2.0 : p.sims[i];  // engine.cpp:252-253; the rescan's running state
        uint32_t arg = INIT == kInitFull ? 0u : p.a[i];
        for (uint32_t sp = 0; sp < n_spans; ++sp) {
            const double s = part_s[w * n_spans + sp];
            const uint32_t a = part_a[w * n_spans + sp];
            if (a != kNone && better(s, a, best, arg)) {
                best = s;
                arg = a;
            }
        }
        p.a[i] = arg;
        p.sims[i] = best;
    }
}

// ---------------------------------------------------------------------------
// Screened scan: fp32 FFMA over the tile, exact fp64 only where needed.
//
// The fp64 similarity the reference computes and an fp32 FMA accumulation of
// the same products differ by at most
//     δ_i = (γ32(n_i) + γ64(n_i)) · ||x_i||₂ · max_j ||c_j||₂,   γ(n) = n·u/(1−n·u)
// (sequential summation bound with Σ|x_t c_t| ≤ ||x||·||c||). The screen keeps,
// per document, the fp32 best, its column and the fp32 runner-up across all
// tiles. When best − runner-up > 2δ the fp32 winner is the unique fp64 argmax
// (no tie possible), and its similarity is then recomputed exactly in fp64 in
// ascending term order — bit-identical to the reference. Documents the screen
// cannot certify take the exact fp64 scan. The hot loop is thus one shuffle,
// one wide load and V FFMAs per entry: no fp32->fp64 conversions (the XU pipe
// they run on is quarter rate) and half the register footprint.
// ---------------------------------------------------------------------------

// L2 eviction policies: the CSR streams past (evict_first, no L1
// allocation) while the current column tile of Cᵀ is kept (evict_last).
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float4 ld_keep(const float4* p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float2 ld_keep(const float2* p, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_keep(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

template <int V, int U>
__device__ __forceinline__ void doc_tile_dots32(const int32_t* __restrict__ idx,
                                                const float* __restrict__ val, int64_t beg,
                                                int64_t end, const float* __restrict__ M,
                                                uint64_t ld, uint32_t col0, int lane,
                                                uint64_t pol_keep, uint64_t pol_stream,
                                                float (&acc)[V]) {
    using VT = typename VecT<V>::type;
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;
    const VT* base = reinterpret_cast<const VT*>(M + col0) + lane;
    const uint32_t ldv = static_cast<uint32_t>(ld / V);
    for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
        const int64_t e = e0 + lane;
        uint32_t off_l = 0;
        float x_l = 0.f;
        if (e < end) {
            off_l = static_cast<uint32_t>(ld_stream_i32(idx + e, pol_stream)) * ldv;
            x_l = ld_stream_f32(val + e, pol_stream);
        }
        const int n = static_cast<int>(imin64(kWarp, end - e0));
        // fully unrolled over the 32-entry chunk: shuffle source lanes are
        // immediates; batches past n are skipped, lanes >= n carry x = 0
#pragma unroll
        for (int j = 0; j < kWarp; j += U) {
            if (j >= n) break;
            VT c[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t off = __shfl_sync(0xFFFFFFFFu, off_l, j + u);
                c[u] = ld_keep(base + off, pol_keep);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float x = __shfl_sync(0xFFFFFFFFu, x_l, j + u);
                float cf[V];
                unpack<V>(c[u], cf);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = fmaf(x, cf[v], acc[v]);
            }
        }
    }
}

// (best, arg, second) fold; equal bests make second == best (uncertified).
__device__ __forceinline__ void top2_push(float s, uint32_t id, float& b, uint32_t& a, float& s2) {
    if (s > b || (s == b && id < a)) {
        s2 = fmaxf(s2, b);
        b = s;
        a = id;
    } else {
        s2 = fmaxf(s2, s);
    }
}

__device__ __forceinline__ void warp_top2(float& b, uint32_t& a, float& s2) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ob = __shfl_xor_sync(0xFFFFFFFFu, b, off);
        const uint32_t oa = __shfl_xor_sync(0xFFFFFFFFu, a, off);
        const float os2 = __shfl_xor_sync(0xFFFFFFFFu, s2, off);
        if (ob > b || (ob == b && oa < a)) {
            s2 = fmaxf(os2, b);
            b = ob;
            a = oa;
        } else {
            s2 = fmaxf(s2, ob);
        }
    }
}

struct ResolveArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const float* CT;
    uint64_t ld_ct;
    const uint32_t* order;
    int64_t n_work;
    double cmax;               // upper bound on every centroid column's 2-norm
    const double* xnorm2;      // per-document ||x||² (computed once at upload)
    int nonneg;                // all document weights > 0 (so centroids >= 0): relative bound
    const float* sb;
    const float* ss;
    const uint32_t* sa;
    // NCC
    const uint8_t* unchanged;
    const uint32_t* a_start;
    const double* sims_start;
    uint32_t* a;
    double* sims;
    uint32_t* exact_list;      // uncertified documents -> exact fp64 scan
    unsigned long long* n_exact;
    uint32_t* rescan_list;
    unsigned long long* n_rescan;
};

struct ScreenArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const float* M;
    uint64_t ld;
    uint32_t col0;
    uint32_t ncols;
    const uint32_t* col_ids;   // nullptr = identity
    const uint32_t* order;     // work item -> document
    int64_t n_work;
    int first;
    const uint32_t* skip_id;   // per document: cluster excluded from the screen (NCC own), or nullptr
    float* sb;                 // running fp32 best   (per document)
    float* ss;                 // running fp32 second
    uint32_t* sa;              // running fp32 argmax (kNone = no candidate)
};

template <int V, int U>
__global__ void __launch_bounds__(256, 2) screen_tile_kernel(ScreenArgs p) {
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    const int64_t chunk = static_cast<int64_t>(ceil_div(p.n_work, gridDim.x));
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t w1 = imin64(p.n_work, w0 + chunk);
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    for (int64_t w = w0 + warp; w < w1; w += nwarps) {
        const int64_t i = p.order ? static_cast<int64_t>(__ldg(p.order + w)) : w;
        const int64_t beg = __ldg(p.indptr + i), end = __ldg(p.indptr + i + 1);
        const uint32_t skip = p.skip_id ? __ldg(p.skip_id + i) : kNone;
        float b = -INFINITY, s2 = -INFINITY;
        uint32_t a = kNone;
        if (!p.first) {
            b = p.sb[i];
            s2 = p.ss[i];
            a = p.sa[i];
        }
        float acc[V];
        doc_tile_dots32<V, U>(p.idx, p.val, beg, end, p.M, p.ld, p.col0, lane, pol_keep, pol_stream, acc);
        float lb = -INFINITY, ls2 = -INFINITY;
        uint32_t la = kNone;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const uint32_t col = p.col0 + static_cast<uint32_t>(lane) * V + v;
            if (col < p.ncols) {
                const uint32_t id = p.col_ids ? __ldg(p.col_ids + col) : col;
                if (id != skip) top2_push(acc[v], id, lb, la, ls2);
            }
        }
        warp_top2(lb, la, ls2);
        if (lane == 0) {
            if (la != kNone) {
                top2_push(lb, la, b, a, s2);
                s2 = fmaxf(s2, ls2);
            }
            p.sb[i] = b;
            p.ss[i] = s2;
            p.sa[i] = a;
        }
    }
}

// ---------------------------------------------------------------------------
// Postings screen: the centroid matrix as an inverted index.
//
// Centroids are ~7% dense on the BASELINE corpora (most terms occur in few
// clusters), so the dense scan spends >90% of its bytes on zeros. The postings
// view stores, per cluster tile T (KT clusters) and term t, the list of
// (cluster, value) pairs with a nonzero centroid weight — the paper's index
// over centroids (§3.2) in GPU form. A warp owns one document and a
// KT-float accumulator in shared memory; for each of the document's terms in
// ascending order, the 32 lanes stride over that term's posting list and do
// acc[c] = fma(x_t, v, acc[c]). Clusters within one list are distinct, so no
// atomics are needed (a __syncwarp orders consecutive lists). The fp32 result
// per (doc, cluster) is the same ascending-term FMA chain as the dense screen,
// so the same certification bound applies.
// ---------------------------------------------------------------------------
struct PostingsArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const uint32_t* pptr;      // d + 1 offsets into pairs for this cluster tile (< 2^32)
    const uint2* pairs;        // (local cluster, float bits)
    uint32_t c0;               // first column of the tile (in M's column space)
    uint32_t kt;               // columns in this tile
    const uint32_t* col_ids;   // column -> cluster id (nullptr = identity)
    const uint32_t* order;
    int64_t n_work;
    int first;
    const uint32_t* skip_id;
    float* sb;
    float* ss;
    uint32_t* sa;
    ResolveArgs r;             // used when the last tile certifies in place (FUSE >= 0)
};

template <int INIT, bool SM = false>
__device__ __forceinline__ void resolve_doc(const ResolveArgs& p, int64_t i, int64_t beg, int64_t end, int lane,
                                            float b, float s2, uint32_t sa, double* wsm = nullptr);

#ifndef SSKM_PAIR_L1
#define SSKM_PAIR_L1 0
#endif
// Posting pairs bypass L1 (hit rate ~6%): L1TEX's SRAM is left to the
// shared-memory accumulators the same warps update.
// Shared-memory accumulator access through a 32-bit shared address computed
// once per warp (a generic pointer makes ptxas rebuild the shared window base
// on every access inside the predicated loop).
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v));
}

__device__ __forceinline__ uint2 ld_pair(const uint2* p, uint64_t pol) {
    uint2 pr;
#if SSKM_PAIR_L1
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(pr.x), "=r"(pr.y) : "l"(p), "l"(pol));
#else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(pr.x), "=r"(pr.y) : "l"(p), "l"(pol));
#endif
    return pr;
}

// SUB lanes serve one posting list; the warp's G = 32/SUB lane groups work on
// G consecutive terms at once, each group into its own KT-float accumulator
// (no conflicts between groups; clusters within a list are distinct). The G
// partial sums are added in a fixed order at the end. Any summation order
// obeys the same γ(n + 32) bound, which the resolve step uses.
template <int KT, int SUB, int FUSE>
__global__ void __launch_bounds__(256) postings_screen_kernel(PostingsArgs p) {
    constexpr int G = kWarp / SUB;
    extern __shared__ float smem_acc[];
    const int lane = threadIdx.x & (kWarp - 1);
    const int grp = lane / SUB, sl = lane % SUB;
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    float* accw = smem_acc + static_cast<size_t>(warp) * G * KT;
    float* accg = accw + grp * KT;
    const uint32_t acc_s = static_cast<uint32_t>(__cvta_generic_to_shared(accg));
    const uint2* __restrict__ pairs = p.pairs;
    const int64_t chunk = static_cast<int64_t>(ceil_div(p.n_work, gridDim.x));
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t w1 = imin64(p.n_work, w0 + chunk);
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    for (int64_t w = w0 + warp; w < w1; w += nwarps) {
        const int64_t i = p.order ? static_cast<int64_t>(__ldg(p.order + w)) : w;
        const int64_t beg = __ldg(p.indptr + i), end = __ldg(p.indptr + i + 1);
        const uint32_t skip = p.skip_id ? __ldg(p.skip_id + i) : kNone;
#pragma unroll
        for (int c = lane * 4; c < G * KT; c += kWarp * 4)
            *reinterpret_cast<float4*>(accw + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
            const int64_t e = e0 + lane;
            uint32_t lb = 0, le = 0;
            float x_l = 0.f;
            if (e < end) {
                const int32_t t = ld_stream_i32(p.idx + e, pol_stream);
                x_l = ld_stream_f32(p.val + e, pol_stream);
                lb = __ldg(p.pptr + t);
                le = __ldg(p.pptr + t + 1);
            }
            const int n = static_cast<int>(imin64(kWarp, end - e0));
            if constexpr (G == 1) {
                // one warp per list, next term's first 32 postings prefetched
                // while the current term accumulates (hides one L2 round trip)
                uint32_t qb = __shfl_sync(0xFFFFFFFFu, lb, 0) + lane, qe = __shfl_sync(0xFFFFFFFFu, le, 0);
                float x = __shfl_sync(0xFFFFFFFFu, x_l, 0);
                uint2 pr = qb < qe ? ld_pair(pairs + qb, pol_keep) : make_uint2(0u, 0u);
                for (int j = 0; j < n; ++j) {
                    const int jn = (j + 1) & (kWarp - 1);
                    const uint32_t nb = __shfl_sync(0xFFFFFFFFu, lb, jn) + lane;
                    uint32_t ne = __shfl_sync(0xFFFFFFFFu, le, jn);
                    const float nx = __shfl_sync(0xFFFFFFFFu, x_l, jn);
                    ne = j + 1 < n ? ne : 0u;
                    const uint2 npr = nb < ne ? ld_pair(pairs + nb, pol_keep) : make_uint2(0u, 0u);
                    if (qb < qe) {
                        const uint32_t a = acc_s + pr.x * 4u;
                        sts_f32(a, fmaf(x, __uint_as_float(pr.y), lds_f32(a)));
                    }
                    // most lists fit the prefetched first 32; keep the rare tail compact
#pragma unroll 1
                    for (uint32_t q = qb + kWarp; q < qe; q += kWarp) {
                        const uint2 t2 = ld_pair(pairs + q, pol_keep);
                        const uint32_t a = acc_s + t2.x * 4u;
                        sts_f32(a, fmaf(x, __uint_as_float(t2.y), lds_f32(a)));
                    }
                    __syncwarp();
                    qb = nb;
                    qe = ne;
                    x = nx;
                    pr = npr;
                }
            } else {
                for (int j0 = 0; j0 < n; j0 += G) {
                    const int j = j0 + grp;  // lanes past n hold empty lists
                    const uint32_t qb = __shfl_sync(0xFFFFFFFFu, lb, j);
                    const uint32_t qe = __shfl_sync(0xFFFFFFFFu, le, j);
                    const float x = __shfl_sync(0xFFFFFFFFu, x_l, j);
                    for (uint32_t q = qb + sl; q < qe; q += SUB) {
                        const uint2 pr = ld_pair(p.pairs + q, pol_keep);
                        accg[pr.x] = fmaf(x, __uint_as_float(pr.y), accg[pr.x]);
                    }
                    __syncwarp();
                }
            }
        }
        // combine the G partial accumulators (fixed order), then top-2
        float tb = -INFINITY, ts2 = -INFINITY;
        uint32_t ta = kNone;
        const uint32_t accw_s = static_cast<uint32_t>(__cvta_generic_to_shared(accw));
        if (p.col_ids) {
            for (int c = lane; c < static_cast<int>(p.kt); c += kWarp) {
                float v = lds_f32(accw_s + 4u * c);
#pragma unroll
                for (int g = 1; g < G; ++g) v += lds_f32(accw_s + 4u * (g * KT + c));
                const uint32_t id = __ldg(p.col_ids + p.c0 + static_cast<uint32_t>(c));
                if (id != skip) top2_push(v, id, tb, ta, ts2);
            }
        } else {
            for (int c = lane; c < static_cast<int>(p.kt); c += kWarp) {
                float v = lds_f32(accw_s + 4u * c);
#pragma unroll
                for (int g = 1; g < G; ++g) v += lds_f32(accw_s + 4u * (g * KT + c));
                const uint32_t id = p.c0 + static_cast<uint32_t>(c);
                if (id != skip) top2_push(v, id, tb, ta, ts2);
            }
        }
        warp_top2(tb, ta, ts2);
        float b = -INFINITY, s2 = -INFINITY;
        uint32_t a = kNone;
        if (!p.first) {
            b = p.sb[i];
            s2 = p.ss[i];
            a = p.sa[i];
        }
        if (ta != kNone) {
            top2_push(tb, ta, b, a, s2);
            s2 = fmaxf(s2, ts2);
        }
        if constexpr (FUSE >= 0) {
            // last cluster tile: certify here instead of in a separate pass
            resolve_doc<FUSE>(p.r, i, beg, end, lane, b, s2, a);
        } else if (lane == 0) {
            p.sb[i] = b;
            p.ss[i] = s2;
            p.sa[i] = a;
        }
        __syncwarp();
    }
}

__global__ void postings_work_kernel(const int32_t* __restrict__ idx, int64_t nnz, const uint32_t* __restrict__ cnt,
                                     unsigned long long* total) {
    unsigned long long s = 0;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        s += cnt[idx[e]];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(total, s);
}

// Postings build from the dense column tile [c0, c0 + kt) of M: per-row counts,
// then (after an exclusive scan) the pairs. Within a list the pairs are laid
// out round-robin by shared-memory bank (rank-0 pair of every bank, then
// rank-1, ...), so the 32 pairs a warp processes together mostly hit distinct
// accumulator banks. Lane l scans columns j = l (mod 32), i.e. exactly bank l
// (tiles start at multiples of 32). The order inside one list never changes a
// result: every cluster occurs once per list.
// Entries kept in a postings build: nonzero and |v| >= thr (thr = 0: every
// nonzero; thr > 0: the high entries of the bound screen).
__device__ __forceinline__ bool post_keep(float v, float thr) { return v != 0.f && fabsf(v) >= thr; }

__global__ void postings_count_kernel(const float* __restrict__ M, uint64_t ld, uint32_t d, uint32_t c0,
                                      uint32_t kt, uint32_t* __restrict__ cnt, float thr) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t t = gw; t < d; t += nw) {
        const float* row = M + t * ld + c0;
        int c = 0;
        for (uint32_t j = lane; j < kt; j += kWarp) c += post_keep(row[j], thr);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, off);
        if (lane == 0) cnt[t] = c;
    }
}

__global__ void __launch_bounds__(256) postings_fill_kernel(const float* __restrict__ M, uint64_t ld, uint32_t d,
                                                            uint32_t c0, uint32_t kt, const uint32_t* __restrict__ pptr,
                                                            uint2* __restrict__ pairs, float thr) {
    constexpr int kMaxRank = 64;  // kt <= 2048 clusters per tile
    __shared__ uint32_t s_mask[8][kMaxRank], s_base[8][kMaxRank];
    const int lane = threadIdx.x & (kWarp - 1);
    const int wib = (threadIdx.x / kWarp) & 7;
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    const unsigned lt = (1u << lane) - 1u;
    const int ranks = static_cast<int>((kt + kWarp - 1) / kWarp);
    for (uint64_t t = gw; t < d; t += nw) {
        const float* row = M + t * ld + c0;
        uint32_t cnt = 0;
        for (uint32_t j = lane; j < kt; j += kWarp) cnt += post_keep(row[j], thr);
        uint32_t run = 0;
        for (int r = 0; r < ranks; ++r) {
            const unsigned m = __ballot_sync(0xFFFFFFFFu, cnt > static_cast<uint32_t>(r));
            if (lane == 0) {
                s_mask[wib][r] = m;
                s_base[wib][r] = run;
            }
            run += __popc(m);
        }
        __syncwarp();
        const uint32_t base = pptr[t];
        uint32_t r = 0;
        for (uint32_t j = lane; j < kt; j += kWarp) {
            const float v = row[j];
            if (post_keep(v, thr)) {
                pairs[base + s_base[wib][r] + __popc(s_mask[wib][r] & lt)] = make_uint2(j, __float_as_uint(v));
                ++r;
            }
        }
        __syncwarp();
    }
}

// Certify one document's screen result (b, s2, sa) and write the exact answer
// (or queue the document for the exact scan). Called by resolve_kernel and,
// fused, by the screen kernels on their last cluster tile.
template <int INIT, bool SM>
__device__ __forceinline__ void resolve_doc(const ResolveArgs& p, int64_t i, int64_t beg, int64_t end, int lane,
                                            float b, float s2, uint32_t sa, double* wsm) {
        // SM: the caller provides a 32-double per-warp buffer for the fold
        auto dot = [&](uint32_t col) {
            if constexpr (SM) return doc_col_dot_sm(p.idx, p.val, beg, end, p.CT, p.ld_ct, col, lane, wsm);
            else return doc_col_dot(p.idx, p.val, beg, end, p.CT, p.ld_ct, col, lane);
        };
        // ||x||₂ (fp64) for the error bound: precomputed per document
        const double q = p.xnorm2[i];
        const double n = static_cast<double>(end - beg);
        const double u32 = 0x1p-24, u64 = 0x1p-53;
        const double n32 = n + 32.0;  // screen: any summation order, up to 32 partial sums
        const double g32 = n32 * u32 / (1.0 - n32 * u32), g64 = n * u64 / (1.0 - n * u64);
        const double delta = (g32 + g64) * sqrt(q) * (1.0 + 1e-12) * p.cmax * (1.0 + 1e-12);
        // Error model of a screened value s32 against the reference's fp64 s64:
        //  signed data:      |s32 − s64| ≤ δ                        (absolute, Cauchy–Schwarz)
        //  nonnegative data: |s32 − s64| ≤ g'·s32, g' = g/(1−g) + γ64 (Σ|x_t c_t| = s itself)
        const double g = g32 / (1.0 - g32) + g64 + 1e-15;
        // (+ n·2^-126 absolute: fp32 products below the normal range)
        const double tiny = n * 0x1p-126;
        auto upper = [&](double v) { return p.nonneg ? (v >= 0.0 ? v * (1.0 + g) : v * (1.0 - g)) + tiny : v + delta; };
        auto lower = [&](double v) { return p.nonneg ? (v >= 0.0 ? v * (1.0 - g) : v * (1.0 + g)) - tiny : v - delta; };
        const double bd = static_cast<double>(b), s2d = static_cast<double>(s2);
        double best;
        uint32_t arg;
        bool certain;
        bool own_changed = false;
        double old_sim = 0.0;
        if constexpr (INIT == kInitFull) {
            // the screen covered every column; the reference's (-2, 0) start only
            // survives when every similarity is <= -2 (left to the exact scan)
            certain = sa != kNone && lower(bd) > upper(s2d);
            best = 0.0;
            arg = sa;
            if (certain) {
                best = dot(sa);
                certain = best > -2.0;
            }
        } else {
            // NCC pass A: cached or refreshed own similarity (engine.cpp:268-273);
            // rescan pass: the exact running best from pass A
            const uint32_t a0 = INIT == kInitRescan ? p.a[i] : p.a_start[i];
            old_sim = INIT == kInitRescan ? p.sims[i] : p.sims_start[i];
            own_changed = INIT == kInitNcc && p.unchanged[a0] == 0;
            const double sim0 = own_changed ? dot(a0)
                                            : old_sim;
            best = sim0;
            arg = a0;
            if (sa == kNone || upper(bd) < sim0) {
                certain = true;  // no screened column can reach the baseline
            } else if (lower(bd) > sim0 && lower(bd) > upper(s2d)) {
                best = dot(sa);
                arg = sa;
                certain = true;
            } else {
                certain = false;
            }
        }
        if (lane == 0) {
            if (certain) {
                p.a[i] = arg;
                p.sims[i] = best;
                if constexpr (INIT == kInitNcc) {
                    if (own_changed && !(best > old_sim)) {  // engine.cpp:303-305
                        const unsigned long long pos = atomicAdd(p.n_rescan, 1ull);
                        p.rescan_list[pos] = static_cast<uint32_t>(i);
                    }
                }
            } else {
                const unsigned long long pos = atomicAdd(p.n_exact, 1ull);
                p.exact_list[pos] = static_cast<uint32_t>(i);
            }
        }
}

// Certify the screen's answer per document (warp per document).
template <int INIT>
__global__ void __launch_bounds__(256) resolve_kernel(ResolveArgs p) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    __shared__ __align__(16) double fold[256];
    double* wsm = fold + (threadIdx.x & ~(kWarp - 1));
    // software pipeline: the next document's id, extent and screen result are
    // loaded while the current one is resolved
    const uint64_t n_work = static_cast<uint64_t>(p.n_work);
    auto fetch = [&](uint64_t w, int64_t& i, int64_t& beg, int64_t& end, float& b, float& s2, uint32_t& sa) {
        i = p.order ? static_cast<int64_t>(__ldg(p.order + w)) : static_cast<int64_t>(w);
        beg = __ldg(p.indptr + i);
        end = __ldg(p.indptr + i + 1);
        b = __ldg(p.sb + i);
        s2 = __ldg(p.ss + i);
        sa = __ldg(p.sa + i);
    };
    if (gw >= n_work) return;
    int64_t i, beg, end;
    float b, s2;
    uint32_t sa;
    fetch(gw, i, beg, end, b, s2, sa);
    for (uint64_t w = gw; w < n_work; w += nw) {
        int64_t ni = 0, nbeg = 0, nend = 0;
        float nb = 0.f, ns2 = 0.f;
        uint32_t nsa = 0;
        if (w + nw < n_work) fetch(w + nw, ni, nbeg, nend, nb, ns2, nsa);
        resolve_doc<INIT, true>(p, i, beg, end, lane, b, s2, sa, wsm);
        i = ni, beg = nbeg, end = nend, b = nb, s2 = ns2, sa = nsa;
    }
}

// ||x_i||² per document (fp64), once per upload.
// Squared row norms (fp64); flags rows above unit length (bit 32 of *bad).
__global__ void doc_norm2_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ val, int64_t n,
                                 double* __restrict__ out, unsigned int* bad) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t i = gw; i < static_cast<uint64_t>(n); i += nw) {
        double q = 0.0;
        for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += kWarp) {
            const double x = static_cast<double>(val[e]);
            q = fma(x, x, q);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(0xFFFFFFFFu, q, off);
        if (lane == 0) {
            out[i] = q;
            if (!(q <= 1.0 + 1e-5)) atomicOr(bad, 32u);
        }
    }
}

__global__ void iota_kernel(uint32_t* __restrict__ p, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = static_cast<uint32_t>(i);
}

// NCC dot accounting when the exact full scan replaced the changed-list scan
// (ncc_epsilon = 0): unchanged centroids keep bit-identical similarities, all
// <= the cached max, so "the refreshed changed scan did not beat the cache"
// (engine.cpp:303) is exactly !(final best > cached sim) for a changed-own doc.
__global__ void ncc_rescan_count_kernel(const uint32_t* __restrict__ a_start, const double* __restrict__ sims_start,
                                        const double* __restrict__ sims, const uint8_t* __restrict__ unchanged,
                                        int64_t n, unsigned long long* n_rescan) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c += unchanged[a_start[i]] == 0 && !(sims[i] > sims_start[i]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(n_rescan, c);
}

// Σ sims (fixed-shape tree: bitwise reproducible for a given n) and the
// reassignment count against the owner map of the sums (= assignments at the
// start of the assign step).
__global__ void finish_assign_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ a_start,
                                     const double* __restrict__ sims, int64_t n,
                                     double* __restrict__ part, unsigned long long* reassigned) {
    __shared__ double sh[256];
    __shared__ unsigned int shc[256];
    double s = 0.0;
    unsigned int c = 0;
    const int64_t per = ceil_div(n, gridDim.x);
    const int64_t b0 = blockIdx.x * per, b1 = imin64(n, b0 + per);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        s += sims[i];
        c += a[i] != a_start[i];
    }
    sh[threadIdx.x] = s;
    shc[threadIdx.x] = c;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            sh[threadIdx.x] += sh[threadIdx.x + off];
            shc[threadIdx.x] += shc[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = sh[0];
        atomicAdd(reassigned, static_cast<unsigned long long>(shc[0]));
    }
}

// Σ part[0..n) in index order (one thread), the partials staged in shared
// memory by the block first (n ≤ 4096).
__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* out) {
    __shared__ double sh[4096];
    for (int i = threadIdx.x; i < n; i += blockDim.x) sh[i] = part[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += sh[i];
        *out = s;
    }
}

}  // namespace sskm_b200
