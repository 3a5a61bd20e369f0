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
__device__ __forceinline__ void load_row(const float* __restrict__ p, float (&c)[V]) {
    if constexpr (V == 4) {
        float4 t = __ldg(reinterpret_cast<const float4*>(p));
        c[0] = t.x;
        c[1] = t.y;
        c[2] = t.z;
        c[3] = t.w;
    } else if constexpr (V == 2) {
        float2 t = __ldg(reinterpret_cast<const float2*>(p));
        c[0] = t.x;
        c[1] = t.y;
    } else {
        c[0] = __ldg(p);
    }
}

// Per-lane fp64 partial dots of one document against columns
// [col0 + lane·V, col0 + lane·V + V) of M, in ascending entry order.
template <int V>
__device__ __forceinline__ void doc_tile_dots(const int32_t* __restrict__ idx,
                                              const float* __restrict__ val, int64_t beg,
                                              int64_t end, const float* __restrict__ M,
                                              uint64_t ld, uint32_t col0, int lane,
                                              double (&acc)[V]) {
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0;
    const float* base = M + col0 + static_cast<uint32_t>(lane) * V;
    for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
        const int64_t e = e0 + lane;
        int t_l = 0;
        float x_l = 0.f;
        if (e < end) {
            t_l = __ldg(idx + e);
            x_l = __ldg(val + e);
        }
        const int n = static_cast<int>(imin64(kWarp, end - e0));
        constexpr int U = 8;
        int j = 0;
        for (; j + U <= n; j += U) {
            float c[U][V];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = __shfl_sync(0xFFFFFFFFu, t_l, j + u);
                load_row<V>(base + static_cast<uint64_t>(t) * ld, c[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double x = static_cast<double>(__shfl_sync(0xFFFFFFFFu, x_l, j + u));
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = fma(x, static_cast<double>(c[u][v]), acc[v]);
            }
        }
        for (; j < n; ++j) {
            const int t = __shfl_sync(0xFFFFFFFFu, t_l, j);
            const double x = static_cast<double>(__shfl_sync(0xFFFFFFFFu, x_l, j));
            float c[V];
            load_row<V>(base + static_cast<uint64_t>(t) * ld, c);
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = fma(x, static_cast<double>(c[v]), acc[v]);
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
    double s = 0.0;
    for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
        const int64_t e = e0 + lane;
        float x_l = 0.f, c_l = 0.f;
        if (e < end) {
            x_l = __ldg(val + e);
            c_l = __ldg(M + static_cast<uint64_t>(__ldg(idx + e)) * ld + col);
        }
        const int n = static_cast<int>(imin64(kWarp, end - e0));
        for (int j = 0; j < n; ++j) {
            const double x = static_cast<double>(__shfl_sync(0xFFFFFFFFu, x_l, j));
            const double c = static_cast<double>(__shfl_sync(0xFFFFFFFFu, c_l, j));
            s = fma(x, c, s);
        }
    }
    return s;
}

// Scan one document against `ncols` columns of M (column c is cluster
// col_ids ? col_ids[c] : c), folding into (best, arg) under the tie rule.
template <int V>
__device__ __forceinline__ void scan_columns(const int32_t* __restrict__ idx,
                                             const float* __restrict__ val, int64_t beg,
                                             int64_t end, const float* __restrict__ M, uint64_t ld,
                                             uint32_t ncols, const uint32_t* __restrict__ col_ids,
                                             int lane, double& best, uint32_t& arg) {
    for (uint32_t col0 = 0; col0 < ncols; col0 += kWarp * V) {
        double acc[V];
        doc_tile_dots<V>(idx, val, beg, end, M, ld, col0, lane, acc);
        double lb = best;
        uint32_t la = arg;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const uint32_t col = col0 + static_cast<uint32_t>(lane) * V + v;
            if (col < ncols) {
                const uint32_t id = col_ids ? __ldg(col_ids + col) : col;
                if (better(acc[v], id, lb, la)) {
                    lb = acc[v];
                    la = id;
                }
            }
        }
        warp_argmax(lb, la);
        best = lb;
        arg = la;
    }
}

enum ScanInit : int {
    kInitFull = 0,    // best = -2, arg = 0 (engine.cpp:252-253), all columns
    kInitNcc = 1,     // NCC pass A: cache or refreshed own dot, changed columns only
    kInitRescan = 2,  // NCC pass B: from pass A's result, all columns
};

struct AssignArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const float* M;            // matrix scanned (Cᵀ, or the compact changed-column copy)
    uint64_t ld;               // row stride of M
    uint32_t ncols;            // columns of M to scan
    const uint32_t* col_ids;   // cluster id per column of M (nullptr = identity)
    const float* CT;           // full Cᵀ (own-centroid refresh)
    uint64_t ld_ct;
    const uint32_t* doc_list;  // documents to process (nullptr = 0..n_work-1)
    int64_t n_work;
    const uint8_t* unchanged;  // per cluster
    uint32_t* a;
    double* sims;
    uint32_t* rescan_list;     // pass A output
    unsigned long long* n_rescan;
};

template <int V, int INIT>
__global__ void __launch_bounds__(256) assign_kernel(AssignArgs p) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t w = gw; w < static_cast<uint64_t>(p.n_work); w += nw) {
        const int64_t i = p.doc_list ? static_cast<int64_t>(p.doc_list[w]) : static_cast<int64_t>(w);
        const int64_t beg = __ldg(p.indptr + i), end = __ldg(p.indptr + i + 1);
        double best;
        uint32_t arg;
        bool own_changed = false;
        double old_sim = 0.0;
        if constexpr (INIT == kInitFull) {
            best = -2.0;
            arg = 0;
        } else if constexpr (INIT == kInitRescan) {
            best = p.sims[i];
            arg = p.a[i];
        } else {
            const uint32_t old_a = p.a[i];
            old_sim = p.sims[i];
            own_changed = p.unchanged[old_a] == 0;
            // unchanged own centroid: the cache is current (engine.cpp:268-270);
            // otherwise refresh the baseline (engine.cpp:271-273)
            best = own_changed ? doc_col_dot(p.idx, p.val, beg, end, p.CT, p.ld_ct, old_a, lane)
                               : old_sim;
            arg = old_a;
        }
        scan_columns<V>(p.idx, p.val, beg, end, p.M, p.ld, p.ncols, p.col_ids, lane, best, arg);
        if (lane == 0) {
            p.a[i] = arg;
            p.sims[i] = best;
            if constexpr (INIT == kInitNcc) {
                // the refreshed scan did not beat the cached max: unchanged
                // centroids may tie or exceed it (engine.cpp:303-305)
                if (own_changed && !(best > old_sim)) {
                    const unsigned long long pos = atomicAdd(p.n_rescan, 1ull);
                    p.rescan_list[pos] = static_cast<uint32_t>(i);
                }
            }
        }
    }
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

__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += part[i];
        *out = s;
    }
}

}  // namespace sskm_b200
