// Bound screen: exact assignment from the high centroid entries only.
//
// Split every centroid weight at a threshold θ. For a document x and cluster j,
//   s_j = Σ_{t: |c_tj| ≥ θ} x_t c_tj  +  Σ_{t: 0 < |c_tj| < θ} x_t c_tj,
// and the second sum is bounded by θ·‖x‖₁. So with acc_j the fp32 sum over
// the high entries (postings built with |v| ≥ θ, a ~1-2% slice of all pairs on
// the TF-IDF corpora: frequent terms carry small centroid weights),
//   s_j ≤ UB_j = acc_j + δ + θ·‖x‖₁,  δ = (γ32(n+32) + γ64(n))·‖x‖₂·max‖c‖ + n·2^-126
// bounds the reference's fp64 dot (sparse_vector.cpp:72-101) from above.
//
// Each document starts from an exact fp64 baseline (best, arg): its current
// cluster (full scan), the cached or refreshed own similarity (NCC pass A,
// engine.cpp:268-273) or the pass-A result (rescan, :303-305). A touched
// cluster with UB_j ≥ best gets an exact fp64 dot (doc_col_dot_sm, bit-equal
// to the reference) and the tie rule s > best || (s == best && j < arg)
// (:259); an untouched cluster is bounded by θ·‖x‖₁ + γ64 alone, so documents
// whose baseline does not beat that go to the exact scan instead. Every
// cluster that could win or tie is evaluated exactly: the result is the
// reference's argmax, independent of θ (θ only moves work between the
// screen, the candidate dots and the exact scan).
#pragma once

#include "assign_kernels.cuh"

namespace sskm_b200 {

struct BoundInitArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const float* CT;
    uint64_t ld_ct;
    const uint32_t* order;     // work item -> document (nullptr = identity)
    int64_t n_work;
    const double* xnorm2;
    const double* xnorm1;
    double theta, cmax;
    uint32_t k;
    uint32_t* a;               // in/out: running exact argmax
    double* sims;              // in/out: running exact max
    const uint8_t* unchanged;
    const uint32_t* a_start;
    const double* sims_start;
    uint8_t* take;             // per work item: 1 = bound screen, 0 = exact scan
    uint32_t* exact_list;      // documents for the exact scan
    unsigned long long* n_exact;
};

// θ·‖x‖₁ plus the fp64 rounding of the reference's dot: no cluster without a
// high entry shared with x can exceed this.
__device__ __forceinline__ double low_bound(double theta, double x1, double q, double n, double cmax) {
    const double u64 = 0x1p-53;
    const double g64 = n * u64 / (1.0 - n * u64);
    return theta * x1 * (1.0 + 1e-12) + g64 * sqrt(q) * cmax * (1.0 + 1e-12) + n * 0x1p-126;
}

template <int INIT>
__global__ void __launch_bounds__(256) bound_init_kernel(BoundInitArgs p) {
    __shared__ __align__(16) double fold[256];
    double* wsm = fold + (threadIdx.x & ~(kWarp - 1));
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t w = gw; w < static_cast<uint64_t>(p.n_work); w += nw) {
        const int64_t i = p.order ? static_cast<int64_t>(p.order[w]) : static_cast<int64_t>(w);
        const int64_t beg = p.indptr[i], end = p.indptr[i + 1];
        double best;
        uint32_t arg;
        if constexpr (INIT == kInitFull) {
            arg = p.a[i];
            best = arg < p.k ? doc_col_dot_sm(p.idx, p.val, beg, end, p.CT, p.ld_ct, arg, lane, wsm) : -2.0;
        } else if constexpr (INIT == kInitNcc) {
            arg = p.a_start[i];
            best = p.unchanged[arg] == 0 ? doc_col_dot_sm(p.idx, p.val, beg, end, p.CT, p.ld_ct, arg, lane, wsm)
                                         : p.sims_start[i];
        } else {
            arg = p.a[i];
            best = p.sims[i];
        }
        const double lb = low_bound(p.theta, p.xnorm1[i], p.xnorm2[i], static_cast<double>(end - beg), p.cmax);
        const bool take = best > lb && (INIT != kInitFull || arg < p.k);
        if (lane == 0) {
            p.take[w] = take ? 1 : 0;
            if (take) {
                p.a[i] = arg;
                p.sims[i] = best;
            } else {
                const unsigned long long pos = atomicAdd(p.n_exact, 1ull);
                p.exact_list[pos] = static_cast<uint32_t>(i);
            }
        }
    }
}

struct BoundArgs {
    const int64_t* indptr;
    const int32_t* idx;
    const float* val;
    const uint32_t* pptr;      // high postings of the tile
    const uint2* pairs;
    uint32_t c0, kt;
    const uint32_t* col_ids;   // column -> cluster id (nullptr = identity)
    const uint32_t* col_of;    // cluster id -> column (kNone = absent); with col_ids
    const uint32_t* list;      // documents taken by the bound screen
    int64_t n_list;
    const float* CT;
    uint64_t ld_ct;
    const double* xnorm2;
    const double* xnorm1;
    double theta, cmax;
    uint32_t k;
    uint32_t* a;
    double* sims;
    unsigned long long* n_cand;  // exact candidate dots
    unsigned long long* n_pairs;  // high pairs accumulated (θ adaptation)
};

using PairT = uint2;
__device__ __forceinline__ PairT ld_pk(const PairT* p, uint64_t pol) { return ld_pair(p, pol); }

template <int KT>
struct BoundSmem {
    static constexpr int kCap = KT / 2;  // touched clusters tracked before a dense sweep
    // fold buffer | accumulators | touched list | term slots | term-at | touched count
    static constexpr size_t per_warp = kWarp * sizeof(double) + KT * sizeof(float) + kCap * sizeof(uint16_t) +
                                       kWarp * sizeof(uint4) + kWarp + 16;
};

template <int KT>
__global__ void __launch_bounds__(256, 4) bound_screen_kernel(BoundArgs p) {
    using SM = BoundSmem<KT>;
    constexpr int kCap = SM::kCap;
    extern __shared__ __align__(16) unsigned char smem_b[];
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    unsigned char* base = smem_b + static_cast<size_t>(warp) * SM::per_warp;
    double* fold = reinterpret_cast<double*>(base);
    float* acc = reinterpret_cast<float*>(base + kWarp * sizeof(double));
    uint16_t* tl = reinterpret_cast<uint16_t*>(base + kWarp * sizeof(double) + KT * sizeof(float));
    uint4* ts = reinterpret_cast<uint4*>(base + kWarp * sizeof(double) + KT * sizeof(float) + kCap * sizeof(uint16_t));
    uint8_t* term_at = reinterpret_cast<uint8_t*>(ts + kWarp);
    uint32_t* ntouch_s = reinterpret_cast<uint32_t*>(term_at + kWarp);
    const uint32_t acc_s = static_cast<uint32_t>(__cvta_generic_to_shared(acc));
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int c = lane * 4; c < KT; c += kWarp * 4) *reinterpret_cast<float4*>(acc + c) = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    const PairT* __restrict__ pairs = p.pairs;
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    const int64_t chunk = static_cast<int64_t>(ceil_div(p.n_list, gridDim.x));
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * chunk;
    const int64_t w1 = imin64(p.n_list, w0 + chunk);
    unsigned long long cands = 0, npairs = 0;
    for (int64_t w = w0 + warp; w < w1; w += nwarps) {
        const int64_t i = __ldg(p.list + w);
        const int64_t beg = __ldg(p.indptr + i), end = __ldg(p.indptr + i + 1);
        if (lane == 0) *ntouch_s = 0u;
        __syncwarp();
        // the running best's own column: its exact value is `best` already, and
        // it is where most of a document's high pairs land — skipping it keeps
        // the lanes' atomics apart
        uint32_t own_l;
        {
            const uint32_t a0 = __ldg(p.a + i);
            const uint32_t col = p.col_ids ? (a0 < p.k ? __ldg(p.col_of + a0) : kNone) : a0;
            own_l = col - p.c0 < p.kt ? col - p.c0 : kNone;
        }
        for (int64_t e0 = beg; e0 < end; e0 += kWarp) {
            const int64_t e = e0 + lane;
            uint32_t lb = 0, le = 0;
            float x = 0.f;
            if (e < end) {
                const int32_t t = ld_stream_i32(p.idx + e, pol_stream);
                x = ld_stream_f32(p.val + e, pol_stream);
                lb = __ldg(p.pptr + t);
                le = __ldg(p.pptr + t + 1);
            }
            // the chunk's high pairs, flattened: 32-slot windows, one pair per
            // lane (high lists are short, ~1.3 pairs per term on c1, so lanes
            // stay busy). Slot s belongs to the term whose exclusive prefix is
            // the last <= s. Lanes of different terms may meet the same cluster:
            // shared float atomics (fp32 order then varies, which the bound
            // tolerates; results never depend on it).
            const uint32_t cnt = le - lb;
            uint32_t incl = cnt;
#pragma unroll
            for (int off = 1; off < kWarp; off <<= 1) {
                const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                if (lane >= off) incl += v;
            }
            const uint32_t excl = incl - cnt, total = __shfl_sync(0xFFFFFFFFu, incl, kWarp - 1);
            npairs += cnt;
            ts[lane] = make_uint4(lb, excl, __float_as_uint(x), 0u);
            for (uint32_t base = 0; base < total; base += kWarp) {
                uint32_t hb = 0;
                if (cnt > 0 && excl < base + kWarp && excl + cnt > base) {
                    const uint32_t pos = (excl > base ? excl : base) - base;  // this term's first slot here
                    hb = 1u << pos;
                    term_at[pos] = static_cast<uint8_t>(lane);
                }
                const uint32_t heads = __reduce_or_sync(0xFFFFFFFFu, hb);
                __syncwarp();
                const uint32_t sl = base + lane;
                if (sl < total) {
                    const int ph = 31 - __clz(heads & (0xFFFFFFFFu >> (31 - lane)));
                    const uint4 T = ts[term_at[ph]];
                    const PairT pr = ld_pk(pairs + T.x + (sl - T.y), pol_keep);
                    if (pr.x != own_l) {
                        const float old = atomicAdd(acc + pr.x, __uint_as_float(T.z) * __uint_as_float(pr.y));
                        if (old == 0.f) {  // first touch (an exact return to 0 only duplicates)
                            const uint32_t pos = atomicAdd(ntouch_s, 1u);
                            if (pos < static_cast<uint32_t>(kCap)) tl[pos] = static_cast<uint16_t>(pr.x);
                        }
                    }
                }
                __syncwarp();
            }
        }
        __syncwarp();
        const uint32_t ntouch = *ntouch_s;
        // candidates: touched clusters whose upper bound reaches the running best
        double best = p.sims[i];
        uint32_t arg = p.a[i];
        const double q = __ldg(p.xnorm2 + i);
        const double nn = static_cast<double>(end - beg);
        const double u32 = 0x1p-24, u64 = 0x1p-53;
        const double n32 = nn + 32.0;
        const double g32 = n32 * u32 / (1.0 - n32 * u32), g64 = nn * u64 / (1.0 - nn * u64);
        const double bx = p.theta * __ldg(p.xnorm1 + i) * (1.0 + 1e-12) +
                          (g32 + g64) * sqrt(q) * p.cmax * (1.0 + 1e-12) + nn * 0x1p-126;
        const bool dense = ntouch > static_cast<uint32_t>(kCap);
        const uint32_t count = dense ? p.kt : ntouch;
        for (uint32_t c0 = 0; c0 < count; c0 += kWarp) {
            const uint32_t k = c0 + lane;
            bool cand = false;
            uint32_t gid = 0;
            double ub = 0.0;
            if (k < count) {
                const uint32_t jl = dense ? k : tl[k];
                const float v = lds_f32(acc_s + jl * 4u);
                gid = p.col_ids ? __ldg(p.col_ids + p.c0 + jl) : p.c0 + jl;
                ub = static_cast<double>(v) + bx;
                cand = gid != arg && ub >= best;
            }
            unsigned cm = __ballot_sync(0xFFFFFFFFu, cand);
            while (cm) {
                const int src = __ffs(cm) - 1;
                cm &= cm - 1;
                const uint32_t g = __shfl_sync(0xFFFFFFFFu, gid, src);
                const double u = __shfl_sync(0xFFFFFFFFu, ub, src);
                if (u >= best) {  // best only grows: re-check
                    const double s = doc_col_dot_sm(p.idx, p.val, beg, end, p.CT, p.ld_ct, g, lane, fold);
                    ++cands;
                    if (s > best || (s == best && g < arg)) {
                        best = s;
                        arg = g;
                    }
                }
            }
        }
        __syncwarp();
        if (dense) {
            for (int c = lane * 4; c < KT; c += kWarp * 4)
                *reinterpret_cast<float4*>(acc + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (uint32_t k = lane; k < ntouch; k += kWarp) sts_f32(acc_s + tl[k] * 4u, 0.f);
        }
        __syncwarp();
        if (lane == 0) {
            p.a[i] = arg;
            p.sims[i] = best;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) npairs += __shfl_xor_sync(0xFFFFFFFFu, npairs, off);  // per-lane terms
    if (lane == 0) {
        atomicAdd(p.n_cand, cands);
        atomicAdd(p.n_pairs, npairs);
    }
}

// NCC pass A over the bound-screened documents: queue the rescan exactly as
// the reference decides it (engine.cpp:303-305); the exact-scan documents
// queue themselves in assign_tile_kernel.
__global__ void bound_ncc_rescan_kernel(const uint32_t* __restrict__ list, int64_t n_list,
                                        const uint32_t* __restrict__ a_start, const double* __restrict__ sims_start,
                                        const double* __restrict__ sims, const uint8_t* __restrict__ unchanged,
                                        uint32_t* __restrict__ rescan_list, unsigned long long* n_rescan) {
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < n_list;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t i = list[w];
        if (unchanged[a_start[i]] == 0 && !(sims[i] > sims_start[i])) {
            const unsigned long long pos = atomicAdd(n_rescan, 1ull);
            rescan_list[pos] = i;
        }
    }
}

// ‖x‖₁ per document (fp64), once per upload.
__global__ void doc_norm1_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ val, int64_t n,
                                 double* __restrict__ out) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t i = gw; i < static_cast<uint64_t>(n); i += nw) {
        double q = 0.0;
        for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += kWarp) q += fabs(static_cast<double>(val[e]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(0xFFFFFFFFu, q, off);
        // upper bound: the fp64 sum's rounding (< n·2^-53 relative) covered
        const double n = static_cast<double>(indptr[i + 1] - indptr[i]);
        if (lane == 0) out[i] = q * (1.0 + (n + 2.0) * 0x1p-52);
    }
}

}  // namespace sskm_b200
