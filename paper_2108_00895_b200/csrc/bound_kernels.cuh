// Bound screen: exact assignment from the high centroid entries only.
//
// Split every centroid weight at a threshold θ. For a document x and cluster j,
//   s_j = Σ_{t: |c_tj| ≥ θ} x_t c_tj  +  Σ_{t: 0 < |c_tj| < θ} x_t c_tj,
// and the second sum is bounded by θ·‖x‖₁. The first sum is accumulated over
// the "high postings" of the cluster tile (term → (cluster, value) with
// |value| ≥ θ: a 1-2% slice of all centroid nonzeros on the TF-IDF corpora,
// frequent terms carry small centroid weights) as an exact integer sum of
// fixed-point products q_t = rn(fl32(x_t·c_tj)·2^30). Against the reference's
// fp64 dot (sparse_vector.cpp:72-101):
//   s_j ≤ UB_j = acc_j·2^-30 + θ·‖x‖₁ + (γ32(n+32) + γ64(n))·‖x‖₂·max‖c‖ + n·2^-30 + n·2^-126
// (fp32 product rounding ≤ u32·Σ|x_t c_t| ≤ u32·‖x‖₂‖c‖, fixed-point rounding
// ≤ 2^-31 per product, the reference's own fp64 rounding ≤ γ64·‖x‖₂‖c‖).
// Integer addition is associative, so acc_j — and hence which clusters become
// candidates — is independent of the order the lanes add in.
//
// Each document starts from an exact fp64 baseline (best, arg): its current
// cluster (full scan; the cached similarity when that column is bit-identical
// to the one the cache was computed against), the cached or refreshed own
// similarity (NCC pass A, engine.cpp:268-273) or the pass-A result (rescan,
// :303-305). The own dot is computed inside the screen, its gathers issued with
// the chunk's posting loads. A touched cluster with UB_j ≥ best gets an exact
// fp64 dot (doc_col_dot_sm, bit-equal to the reference) and the tie rule
// s > best || (s == best && j < arg) (:259); an untouched cluster is bounded by
// θ·‖x‖₁ + γ64 alone, so documents whose baseline does not beat that go to the
// exact scan instead. Every cluster that could win or tie is evaluated exactly:
// the result is the reference's argmax, independent of θ (θ only moves work
// between the screen, the candidate dots and the exact scan).
#pragma once

#include <cuda_fp16.h>

#include "assign_kernels.cuh"

namespace sskm_b200 {

#ifndef SSKM_BOUND_MINB
#define SSKM_BOUND_MINB 4  // resident 256-thread blocks per SM the register budget is cut for
#endif

#ifndef SSKM_UB_GROUPS
#define SSKM_UB_GROUPS 32
#endif
constexpr int kUbGroups = SSKM_UB_GROUPS;  // drift bound: clusters grouped by id mod kUbGroups (32 or 64)
constexpr int kUbPerLane = kUbGroups / 32;  // groups lane, lane + 32, ... belong to a lane
static_assert(kUbGroups == 32 || kUbGroups == 64, "the fold buffer holds at most 64 group maxima");
constexpr unsigned short kHalfInf = 0x7C00u;
constexpr float kFixScale = 0x1p30f;    // fixed-point products: q = rn(p · 2^30)
constexpr double kFixUnit = 0x1p-30;

struct BoundArgs {
    const int64_t* indptr;
    const uint32_t* indptr32;  // 32-bit copy of indptr (nnz < 2^32 per device)
    const int32_t* idx;
    const float* val;
    const uint4* hptr;         // per term: (first high pair, count, bits of the largest low |weight|, 0)
    const uint2* pairs;        // (column in tile, value bits)
    uint32_t c0, kt;
    const uint32_t* col_ids;   // column -> cluster id (nullptr = identity)
    const uint32_t* col_of;    // cluster id -> column (kNone = absent); with col_ids
    const uint32_t* order;     // work item -> document (nullptr = identity)
    int64_t n_work;
    const float* CT;           // full Cᵀ: own dots and candidate dots
    uint64_t ld_ct;
    const float2* xb;          // per document (‖x‖₁, ‖x‖₂), rounded up
    double theta, cmax;
    uint32_t k;
    int first;                 // first tile: establish the baseline and decide take
    int single_tile;           // the tile holds every column (its low maxima bound every cluster)
    int last;                  // last tile of the pass
    const unsigned long long* hp_overflow;  // the postings build dropped lists (then only Σ|x|·L_t bounds)
    uint32_t* a;               // in/out: running exact argmax
    double* sims;              // in/out: running exact max
    const uint8_t* unchanged;  // NCC: cached own similarity valid
    const uint8_t* same;       // full scan: column bit-identical since the cache (nullptr = no cache)
    const uint32_t* a_start;
    const double* sims_start;
    uint8_t* take;             // per work item: 1 = bound screen, 0 = exact scan
    uint32_t* exact_list;      // documents for the exact scan
    unsigned long long* n_exact;
    unsigned long long* n_cand;      // exact candidate dots
    unsigned long long* n_pairs;     // high pairs accumulated (θ adaptation)
    unsigned long long* n_doc_nnz;   // document nonzeros read (roofline bytes)
    unsigned long long* n_visits;    // documents visited, summed over tiles (roofline bytes)
    unsigned long long* n_cand_nnz;  // nonzeros of the candidate dots (centroid values gathered)
    unsigned long long* n_own;       // own dots computed in the screen
    // drift bound (full-scan passes over every document; nullptr otherwise):
    // per document and cluster group g (cluster id mod 32) a certified upper
    // bound on its similarity to every cluster of the group other than its
    // own (fp16, rounded up), and the iteration it holds for (skip_kernel)
    __half* ub;
    uint32_t* ub_it;
    uint32_t iter;
    const unsigned long long* n_work_dev;  // work-list length on the device (overrides n_work)
    unsigned long long* n_hovf;      // documents whose hash table overflowed (HT > 0)
    unsigned long long* n_own_nnz;   // nonzeros of the own dots (own-column weights gathered: roofline bytes)
};

// Per-warp shared memory of the bound screen (bytes). HT > 0: the
// accumulators are a hash table of HT slots keyed by column (one pass over
// every column, however many: configs 2 and 4), else KT slots, one per column
// of a cluster tile.
template <int KT, int HT = 0>
struct BoundSmem {
    static constexpr int kCap = 256;  // touched slots tracked before a dense sweep of the table
    static constexpr int kSlots = HT > 0 ? HT : KT;
    static constexpr uint32_t o_acc = 0;                          // int32[kSlots] fixed-point accumulators
    // u16[HT] hash keys: column + 1 (0 = empty): hash passes need k <= 65,534. (16-bit keys
    // bring the 1024-slot tables to 6 KB per warp: 32 resident warps per SM instead of 24.)
    static constexpr uint32_t o_key = o_acc + kSlots * 4;
    static constexpr uint32_t o_fold = o_key + (HT > 0 ? HT * 2 : 0);  // double[32] fold buffer
    static constexpr uint32_t o_tl = o_fold + 32 * 8;      // u16[kCap] touched list
    static constexpr uint32_t o_cnt = o_tl + kCap * 2;     // u32 touched count
    static constexpr uint32_t o_stats = o_cnt + 16;        // u32[12] per-warp statistics (slot 7: the work range's end)
    static constexpr size_t per_warp = o_stats + 48;
};

__device__ __forceinline__ uint32_t sm_ld_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sm_st_u32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ uint32_t sm_ld_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sm_st_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(static_cast<uint16_t>(v)));
}
__device__ __forceinline__ int sm_atom_add(uint32_t a, int v) {
    int old;
    asm volatile("atom.shared.add.s32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v));
    return old;
}
__device__ __forceinline__ uint32_t sm_atom_cas16(uint32_t a, uint32_t cmp, uint32_t v) {
    uint16_t old;
    asm volatile("atom.shared.cas.b16 %0, [%1], %2, %3;"
                 : "=h"(old)
                 : "r"(a), "h"(static_cast<uint16_t>(cmp)), "h"(static_cast<uint16_t>(v)));
    return old;
}

// Loads and a conversion as volatile asm: the compiler keeps them where they
// are written (it otherwise converts a gathered weight right after its load,
// stalling the warp on it before the next chunk's loads are issued).
__device__ __forceinline__ uint4 ld_u4_nc(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_f32_nc(const float* p) {
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double cvt_f64(float v) {
    double r;
    asm volatile("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(v));
    return r;
}

// Fold the lanes' exact fp64 products of one chunk into s in ascending entry
// order (every lane folds the same sequence: s is warp-uniform).
__device__ __forceinline__ double fold_chunk(double s, double prod, int n, int lane, double* wsm) {
    wsm[lane] = prod;
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
    return s;
}

// Candidate dot (rare: ~0.3 per document) kept out of line so its gather
// arrays do not add to the screen loop's register pressure.
#ifndef SSKM_CAND_INLINE
#define SSKM_CAND_INLINE 1
#endif
#if SSKM_CAND_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
double cand_dot(const int32_t* __restrict__ idx, const float* __restrict__ val, int64_t beg,
                                        int64_t end, const float* __restrict__ M, uint64_t ld, uint32_t col, int lane,
                                        double* wsm) {
    return doc_col_dot_sm(idx, val, beg, end, M, ld, col, lane, wsm);
}

// γ(n) = n·u/(1 − n·u) ≤ n·u·(1 + 2·n·u) for n·u ≤ 1/2 (no fp64 division).
__device__ __forceinline__ double gamma_ub(double n, double u) {
    const double nu = n * u;
    return nu * (1.0 + 2.0 * nu);
}

// A warp per document, 32 entries (one chunk) at a time. The pipeline keeps
// the next document's extents and start cluster one document ahead (its id two
// ahead) and every chunk's (term, weight) one chunk ahead, across document
// boundaries; per chunk, the terms' high-postings extents and own-column
// weights are gathered together, then each lane takes its term's high pairs,
// up to 4 loads in flight, into the fixed-point accumulators with shared
// integer atomics; the first touch of a cluster appends it to the touched list.
// Offsets are 32-bit (the host requires nnz < 2^32 per device for this kernel)
// and the statistics counters live in shared memory, to keep the pipelined
// loads in registers.
template <int KT, int INIT, int HT = 0>
__global__ void __launch_bounds__(256, SSKM_BOUND_MINB) bound_screen_kernel(BoundArgs p) {
    using SM = BoundSmem<KT, HT>;
    constexpr int kCap = SM::kCap;
    constexpr int kSlots = SM::kSlots;
    extern __shared__ __align__(16) unsigned char smem_b[];
    const int lane = threadIdx.x & (kWarp - 1);
    const int warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    unsigned char* base = smem_b + static_cast<size_t>(warp) * SM::per_warp;
    const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(base));
    double* fold = reinterpret_cast<double*>(base + SM::o_fold);
    const uint32_t s_acc = sb + SM::o_acc, s_tl = sb + SM::o_tl, s_cnt = sb + SM::o_cnt, s_st = sb + SM::o_stats;
    const uint32_t s_key = sb + SM::o_key;
    for (int c = lane; c < kSlots; c += kWarp) sm_st_u32(s_acc + 4u * c, 0u);
    if constexpr (HT > 0)
        for (int c = lane; c < HT / 2; c += kWarp) sm_st_u32(s_key + 4u * c, 0u);  // two keys per word
    if (lane < 12 && lane != 7) sm_st_u32(s_st + 4u * lane, 0u);
    __syncwarp();
    const uint2* __restrict__ pairs = p.pairs;
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    // the block's work range; with a device-side list length (drift-bound work
    // list) its end lives in the warp's statistics slot 7, re-read where used
    // (a register would have to survive the whole pipeline)
    const uint32_t n_work = static_cast<uint32_t>(p.n_work_dev ? *p.n_work_dev : p.n_work);
    const uint32_t chunk = static_cast<uint32_t>(ceil_div(n_work, gridDim.x));
    const uint32_t w0 = blockIdx.x * chunk;
    if (lane == 0) sm_st_u32(s_st + 28u, min(n_work, w0 + chunk));
    __syncwarp();
#define w1 sm_ld_u32(s_st + 28u)
    const bool first = p.first != 0;
    const bool hp_ovf = *p.hp_overflow != 0;
    const uint32_t* __restrict__ indptr = reinterpret_cast<const uint32_t*>(p.indptr32);
    auto doc_of = [&](uint32_t ww) -> uint32_t { return p.order ? __ldg(p.order + ww) : ww; };
    auto start_of = [&](uint32_t i) -> uint32_t {
        if constexpr (INIT == kInitNcc) return first ? __ldg(p.a_start + i) : p.a[i];
        return p.a[i];
    };
    auto stat = [&](int k, uint32_t v) {  // per-warp statistics (lane 0; a reduction, nothing waits on it)
        if (lane == 0) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(s_st + 4u * k), "r"(v));
    };
    uint32_t w = w0 + warp;
    uint32_t i_n = 0, i_nn = 0, arg_n = 0, beg_n = 0, end_n = 0;
    if (w < w1) {
        i_n = doc_of(w);
        beg_n = __ldg(indptr + i_n);
        end_n = __ldg(indptr + i_n + 1);
        arg_n = start_of(i_n);
    }
    if (w + nwarps < w1) i_nn = doc_of(w + nwarps);
    int32_t t_n = 0;
    float x_n = 0.f;
    uint4 ext_n = make_uint4(0u, 0u, 0u, 0u);  // the prefetched chunk's postings extents
    if (w < w1 && beg_n + lane < end_n) {
        t_n = ld_stream_i32(p.idx + beg_n + lane, pol_stream);
        x_n = ld_stream_f32(p.val + beg_n + lane, pol_stream);
        ext_n = ld_u4_nc(p.hptr + t_n);
    }
    for (; w < w1; w += nwarps) {
        const uint32_t i = i_n, beg = beg_n, end = end_n;
        uint32_t arg = arg_n;
        const uint32_t wn = w + nwarps;
        if (wn < w1) {
            i_n = i_nn;
            beg_n = __ldg(indptr + i_n);
            end_n = __ldg(indptr + i_n + 1);
            arg_n = start_of(i_n);
        }
        if (wn + nwarps < w1) i_nn = doc_of(wn + nwarps);
        // baseline of this document (first tile), or the running state
        bool active = true, need_dot = false;
        double best = 0.0;
        if (first) {
            if constexpr (INIT == kInitFull) {
                if (arg >= p.k) {
                    best = -2.0;
                } else {
                    need_dot = p.same == nullptr || p.same[arg] == 0;
                    if (!need_dot) best = p.sims[i];
                }
            } else if constexpr (INIT == kInitNcc) {
                need_dot = p.unchanged[arg] == 0;
                if (!need_dot) best = __ldg(p.sims_start + i);
            } else {
                best = p.sims[i];
            }
        } else {
            active = p.take[w] != 0;
            best = p.sims[i];
        }
        const float2 xb = __ldg(p.xb + i);
        const uint32_t own_col = p.col_ids ? (arg < p.k ? __ldg(p.col_of + arg) : kNone) : arg;
        const uint32_t own_l = HT > 0 ? own_col : (own_col - p.c0 < p.kt ? own_col - p.c0 : kNone);
        if (lane == 0) {
            sm_st_u32(s_cnt, 0u);
            if constexpr (HT > 0) sm_st_u32(s_cnt + 4u, 0u);  // hash table overflow of this document
        }
        __syncwarp();
        double s_own = 0.0;
        int accmax = 0;      // ≥ every accumulator's final value (0: untouched clusters)
        float lowsum = 0.f;  // Σ |x_t|·(largest low |weight| of term t): bounds every cluster's low part
        bool pref_done = false;
        if (active) {
            stat(0, 1u);
            stat(1, end - beg);
            for (uint32_t e0 = beg; e0 < end; e0 += kWarp) {
                const bool valid = e0 + lane < end;
                const int32_t t = t_n;
                const float x = x_n;
                const uint4 ext = ext_n;  // issued one chunk earlier
                // the next chunk first (this document's, else the next document's),
                // so its loads fly while this chunk waits on its own
                bool nv;
                {
                    const bool last = e0 + kWarp >= end;
                    const uint32_t en = last ? beg_n + lane : e0 + kWarp + lane;
                    const uint32_t lim = last ? (wn < w1 ? end_n : 0u) : end;
                    nv = en < lim;
                    t_n = 0;
                    x_n = 0.f;
                    if (nv) {
                        t_n = ld_stream_i32(p.idx + en, pol_stream);
                        x_n = ld_stream_f32(p.val + en, pol_stream);
                    }
                    if (last) pref_done = true;
                }
                // this chunk's own-column weight (first used by the fold, after the pairs)
                float cv = 0.f;
                if (valid && need_dot) cv = ld_f32_nc(p.CT + static_cast<uint64_t>(t) * p.ld_ct + arg);
                // the chunk's high pairs, flattened into windows of 32 slots (one
                // pair per lane, all loads of a window in flight together); slot
                // s belongs to the first lane whose inclusive prefix exceeds s,
                // found by a 5-step binary search over the lanes' prefixes
                const uint32_t cnt = ext.y;
                lowsum = fmaf(fabsf(x), __uint_as_float(ext.z), lowsum);
                uint32_t incl = cnt;
#pragma unroll
                for (int off = 1; off < kWarp; off <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                    if (lane >= off) incl += o;
                }
                const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, kWarp - 1);
                const uint32_t adj = ext.x - (incl - cnt);  // pair index = adj + slot
                const float xs = x * kFixScale;
                // two windows per round: both windows' pair loads are in flight
                // before either window's accumulator updates
                auto slot = [&](uint32_t sl, uint2& pr, float& xq) {
                    int lo = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const uint32_t v = __shfl_sync(0xFFFFFFFFu, incl, lo + step - 1);
                        if (v <= sl) lo += step;
                    }
                    const uint32_t base_o = __shfl_sync(0xFFFFFFFFu, adj, lo & (kWarp - 1));
                    xq = __shfl_sync(0xFFFFFFFFu, xs, lo & (kWarp - 1));
                    pr = sl < total ? ld_pair(pairs + (base_o + sl), pol_keep) : make_uint2(kNone, 0u);
                };
                auto accumulate = [&](const uint2 pr, const float xq) {
                    if (pr.x != kNone && pr.x != own_l) {
                        const int qv = __float2int_rn(xq * __uint_as_float(pr.y));
                        if (qv != 0) {
                            if constexpr (HT > 0) {
                                // linear probing from a multiplicative hash; the lane
                                // that claims an empty slot records it as touched
                                uint32_t h = (pr.x * 0x9E3779B1u) >> (32 - __builtin_ctz(HT));
                                uint32_t slot = kNone;
#pragma unroll 1
                                for (int probe = 0; probe < 64; ++probe) {
                                    uint32_t key = sm_ld_u16(s_key + 2u * h);
                                    if (key == 0) {
                                        key = sm_atom_cas16(s_key + 2u * h, 0u, pr.x + 1u);
                                        if (key == 0) {
                                            const uint32_t pos = static_cast<uint32_t>(sm_atom_add(s_cnt, 1));
                                            if (pos < static_cast<uint32_t>(kCap)) sm_st_u16(s_tl + 2u * pos, h);
                                            key = pr.x + 1u;
                                        }
                                    }
                                    if (key == pr.x + 1u) {
                                        slot = h;
                                        break;
                                    }
                                    h = (h + 1u) & static_cast<uint32_t>(HT - 1);
                                }
                                if (slot != kNone) {
                                    const int old = sm_atom_add(s_acc + 4u * slot, qv);
                                    accmax = max(accmax, old + qv);
                                } else {
                                    sm_st_u32(s_cnt + 4u, 1u);  // table full: this document goes to the exact scan
                                }
                            } else {
                                const int old = sm_atom_add(s_acc + 4u * pr.x, qv);
                                accmax = max(accmax, old + qv);  // every final value is some old + qv
                                if (old == 0) {  // first touch (a return to exactly 0 only duplicates)
                                    const uint32_t pos = static_cast<uint32_t>(sm_atom_add(s_cnt, 1));
                                    if (pos < static_cast<uint32_t>(kCap)) sm_st_u16(s_tl + 2u * pos, pr.x);
                                }
                            }
                        }
                    }
                };
                for (uint32_t wb = 0; wb < total; wb += 2 * kWarp) {
                    uint2 pa, pb;
                    float xa, xb2;
                    slot(wb + lane, pa, xa);
                    if (wb + kWarp < total) {  // a second window only when there are pairs for it
                        slot(wb + kWarp + lane, pb, xb2);
                        accumulate(pa, xa);
                        accumulate(pb, xb2);
                    } else {
                        accumulate(pa, xa);
                    }
                }
                // the next chunk's extents, now that its terms have arrived: in
                // flight during this chunk's fold and the loop turn
                ext_n = nv ? ld_u4_nc(p.hptr + t_n) : make_uint4(0u, 0u, 0u, 0u);
                __syncwarp();
                stat(2, total);
                if (need_dot)  // own dot, ascending entry order, exact in fp64
                    s_own = fold_chunk(s_own, cvt_f64(x) * cvt_f64(cv), static_cast<int>(min(32u, end - e0)), lane,
                                       fold);
            }
        }
        if (!pref_done) {  // empty or skipped document: prefetch the next one's first chunk
            t_n = 0;
            x_n = 0.f;
            ext_n = make_uint4(0u, 0u, 0u, 0u);
            if (wn < w1 && beg_n + lane < end_n) {
                t_n = ld_stream_i32(p.idx + beg_n + lane, pol_stream);
                x_n = ld_stream_f32(p.val + beg_n + lane, pol_stream);
                ext_n = ld_u4_nc(p.hptr + t_n);
            }
        }
        __syncwarp();
        const uint32_t ntouch = sm_ld_u32(s_cnt);
        const double nn = static_cast<double>(end - beg);
        const double g32 = gamma_ub(nn + 32.0, 0x1p-24), g64 = gamma_ub(nn, 0x1p-53);
        const double tiny = nn * kFixUnit + nn * 0x1p-126;
        // the lanes' fp32 sums of nonnegative terms, each within (1 + (n/32 + 1)·2^-24)
        double low = static_cast<double>(lowsum);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) low += __shfl_xor_sync(0xFFFFFFFFu, low, off);
        low = low * (1.0 + (nn / 32.0 + 2.0) * 0x1p-23) * (1.0 + 1e-12);
        const double theta_x1 = p.theta * xb.x * (1.0 + 1e-12);
        // θ·‖x‖₁ bounds only weights below θ: not valid once lists were dropped
        const double lowb = hp_ovf ? low : fmin(low, theta_x1);
        if (first && active) {
            if (need_dot) {
                best = s_own;
                stat(3, 1u);
                stat(8, end - beg);
            }
            // no cluster without a high entry shared with x can exceed lb
            // (the tile's low maxima bound the clusters of this tile only)
            const double lb = (p.single_tile ? lowb : theta_x1) + g64 * xb.y * p.cmax * (1.0 + 1e-12) + tiny;
            bool take = best > lb && (INIT != kInitFull || arg < p.k);
            if constexpr (HT > 0) {
                if (sm_ld_u32(s_cnt + 4u) != 0) {
                    take = false;
                    stat(6, 1u);
                }
            }
            if (lane == 0) {
                p.take[w] = take ? 1 : 0;
                if (!take) {
                    const unsigned long long pos = atomicAdd(p.n_exact, 1ull);
                    p.exact_list[pos] = i;
                }
            }
            active = take;
        }
        const bool dense = ntouch > static_cast<uint32_t>(kCap);  // sweep every slot
        accmax = __reduce_max_sync(0xFFFFFFFFu, accmax);
        if (active) {
            // candidates: touched clusters whose upper bound reaches the running
            // best, gathered 32 at a time (one per lane) and evaluated in
            // descending bound order, so the likely winner raises `best` first
            // and prunes the rest (a bound below best cannot win or tie)
            const double bx = lowb + (g32 + g64) * xb.y * p.cmax * (1.0 + 1e-12) + tiny;
            // no touched cluster can reach best: nothing to evaluate
            const uint32_t count =
                static_cast<double>(accmax) * kFixUnit + bx >= best ? (dense ? (HT > 0 ? kSlots : p.kt) : ntouch) : 0u;
            if (p.ub) {
                // every other cluster j of this tile: s_j <= acc_j·2^-30 + bx (the own
                // cluster's pairs were never accumulated; untouched clusters have
                // acc = 0). Lane g keeps the largest accumulator of the clusters
                // with id ≡ g (mod 32): the group's bound, the maximum over the
                // tiles; withdrawn below if the document moves (its new cluster's
                // pairs were accumulated). The fold buffer is free until the
                // candidate dots.
                const uint32_t s_gm = sb + SM::o_fold;
#pragma unroll
                for (int q = 0; q < kUbPerLane; ++q) sm_st_u32(s_gm + 4u * (lane + kWarp * q), 0u);
                __syncwarp();
                constexpr uint32_t kGMask = static_cast<uint32_t>(kUbGroups - 1);
                if (dense) {
                    int m[kUbPerLane];
#pragma unroll
                    for (int q = 0; q < kUbPerLane; ++q) m[q] = 0;
                    for (int c = lane; c < kSlots; c += kWarp * kUbPerLane) {
#pragma unroll
                        for (int q = 0; q < kUbPerLane; ++q) {
                            const int cc = c + kWarp * q;  // kSlots is a multiple of 64
                            const int v = static_cast<int>(sm_ld_u32(s_acc + 4u * cc));
                            if constexpr (HT > 0) {
                                const uint32_t key = sm_ld_u16(s_key + 2u * cc);
                                if (key != 0 && v > 0)
                                    asm volatile("red.shared.max.s32 [%0], %1;" ::"r"(s_gm + 4u * ((key - 1u) & kGMask)), "r"(v));
                            } else {
                                m[q] = max(m[q], v);  // column c0 + cc, c0 a multiple of 64: group = cc mod kUbGroups
                            }
                        }
                    }
                    if constexpr (HT == 0) {
#pragma unroll
                        for (int q = 0; q < kUbPerLane; ++q) sm_st_u32(s_gm + 4u * (lane + kWarp * q), static_cast<uint32_t>(m[q]));
                    }
                } else {
                    for (uint32_t kk = lane; kk < ntouch; kk += kWarp) {
                        const uint32_t jl = sm_ld_u16(s_tl + 2u * kk);
                        const int v = static_cast<int>(sm_ld_u32(s_acc + 4u * jl));
                        uint32_t col = p.c0 + jl;
                        if constexpr (HT > 0) col = sm_ld_u16(s_key + 2u * jl) - 1u;
                        if (v > 0) asm volatile("red.shared.max.s32 [%0], %1;" ::"r"(s_gm + 4u * (col & kGMask)), "r"(v));
                    }
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < kUbPerLane; ++q) {
                    const int gmax = static_cast<int>(sm_ld_u32(s_gm + 4u * (lane + kWarp * q)));
                    __half u = __float2half_ru(__double2float_ru(static_cast<double>(gmax) * kFixUnit + bx));
                    __half* ug = p.ub + static_cast<uint64_t>(i) * kUbGroups + lane + kWarp * q;
                    if (!first) u = __hmax(u, *ug);
                    *ug = u;
                }
                if (first && lane == 0) p.ub_it[i] = p.iter;
                __syncwarp();  // the fold buffer goes back to the candidate dots
            }
            uint32_t c_gid = 0;   // this lane's pending candidate
            double c_ub = -1e300;
            bool c_on = false;
            auto drain = [&](bool all) {
                // evaluate pending candidates, best bound first; with !all only
                // until a lane is free again
                while (true) {
                    c_on = c_on && c_ub >= best;
                    const unsigned on = __ballot_sync(0xFFFFFFFFu, c_on);
                    if (!on || (!all && on != 0xFFFFFFFFu)) break;
                    double mu = c_on ? c_ub : -1e300;
                    int ml = lane;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) {
                        const double ou = __shfl_xor_sync(0xFFFFFFFFu, mu, off);
                        const int ol = __shfl_xor_sync(0xFFFFFFFFu, ml, off);
                        if (ou > mu || (ou == mu && ol < ml)) {
                            mu = ou;
                            ml = ol;
                        }
                    }
                    const uint32_t g = __shfl_sync(0xFFFFFFFFu, c_gid, ml);
                    if (lane == ml) c_on = false;
                    const double sx = cand_dot(p.idx, p.val, beg, end, p.CT, p.ld_ct, g, lane, fold);
                    stat(4, 1u);
                    stat(5, end - beg);
                    if (sx > best || (sx == best && g < arg)) {
                        best = sx;
                        arg = g;
                    }
                }
            };
            for (uint32_t k0 = 0; k0 < count; k0 += kWarp) {
                const uint32_t kk = k0 + lane;
                bool cand = false;
                uint32_t gid = 0;
                double ub = 0.0;
                if (kk < count) {
                    const uint32_t jl = dense ? kk : sm_ld_u16(s_tl + 2u * kk);
                    uint32_t col = p.c0 + jl;
                    bool used = true;
                    if constexpr (HT > 0) {
                        const uint32_t key = sm_ld_u16(s_key + 2u * jl);
                        used = key != 0;
                        col = key - 1u;
                    }
                    if (used) {
                        gid = p.col_ids ? __ldg(p.col_ids + col) : col;
                        ub = static_cast<double>(static_cast<int>(sm_ld_u32(s_acc + 4u * jl))) * kFixUnit + bx;
                        cand = gid != arg && ub >= best;
                    }
                }
                unsigned cm = __ballot_sync(0xFFFFFFFFu, cand);
                // place the new candidates into free lanes (evaluating pending
                // ones whenever every lane is occupied)
                while (cm) {
                    drain(false);
                    const unsigned fr = ~__ballot_sync(0xFFFFFFFFu, c_on);
                    const int dst_rank = __popc(fr & ((1u << lane) - 1u));  // this free lane's rank
                    const int take_n = min(__popc(fr), __popc(cm));
                    // the r-th remaining candidate goes to the r-th free lane
                    int src = -1;
                    if ((fr >> lane) & 1u) {
                        if (dst_rank < take_n) {
                            unsigned m = cm;
                            for (int r = 0; r < dst_rank; ++r) m &= m - 1;
                            src = __ffs(m) - 1;
                        }
                    }
                    const uint32_t g2 = __shfl_sync(0xFFFFFFFFu, gid, src < 0 ? 0 : src);
                    const double u2 = __shfl_sync(0xFFFFFFFFu, ub, src < 0 ? 0 : src);
                    if (src >= 0) {
                        c_gid = g2;
                        c_ub = u2;
                        c_on = true;
                    }
                    for (int r = 0; r < take_n; ++r) cm &= cm - 1;
                }
            }
            drain(true);
            if (lane == 0) {
                if (p.ub && p.last && arg != p.a_start[i])
                    p.ub[static_cast<uint64_t>(i) * kUbGroups] = __ushort_as_half(kHalfInf);
                p.a[i] = arg;
                p.sims[i] = best;
            }
        } else if (first && p.ub && lane == 0) {
            p.ub[static_cast<uint64_t>(i) * kUbGroups] = __ushort_as_half(kHalfInf);  // exact scan: no bound
        }
        // clear the touched accumulators
        __syncwarp();
        if (dense) {
            for (int c = lane; c < kSlots; c += kWarp) sm_st_u32(s_acc + 4u * c, 0u);
            if constexpr (HT > 0)
                for (int c = lane; c < HT / 2; c += kWarp) sm_st_u32(s_key + 4u * c, 0u);
        } else {
            for (uint32_t kk = lane; kk < ntouch; kk += kWarp) {
                const uint32_t sl = sm_ld_u16(s_tl + 2u * kk);
                sm_st_u32(s_acc + 4u * sl, 0u);
                if constexpr (HT > 0) sm_st_u16(s_key + 2u * sl, 0u);
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        atomicAdd(p.n_visits, static_cast<unsigned long long>(sm_ld_u32(s_st + 0)));
        atomicAdd(p.n_doc_nnz, static_cast<unsigned long long>(sm_ld_u32(s_st + 4)));
        atomicAdd(p.n_pairs, static_cast<unsigned long long>(sm_ld_u32(s_st + 8)));
        atomicAdd(p.n_own, static_cast<unsigned long long>(sm_ld_u32(s_st + 12)));
        atomicAdd(p.n_cand, static_cast<unsigned long long>(sm_ld_u32(s_st + 16)));
        atomicAdd(p.n_cand_nnz, static_cast<unsigned long long>(sm_ld_u32(s_st + 20)));
        if (HT > 0 && p.n_hovf) atomicAdd(p.n_hovf, static_cast<unsigned long long>(sm_ld_u32(s_st + 24)));
        if (p.n_own_nnz) atomicAdd(p.n_own_nnz, static_cast<unsigned long long>(sm_ld_u32(s_st + 32)));
    }
#undef w1
}

// Drift bound (full-scan passes). The bound screen leaves, for every document
// that kept its cluster a and every cluster group g (cluster id mod 32),
// U_ig >= s_ij for every j != a of the group: the reference's fp64 dot against
// the centroids of that iteration t_s. Centroid columns then move by
// δ_j = ||c_j^new − c_j^old||_2 per update, so in real arithmetic x·c_j grows
// by at most ||x||_2·Σδ_j, and
//   s_ij(t) <= U_ig + ||x||_2·(D_g(t) − D_g(t_s)) + 2·γ64(n)·||x||_2·cmax,
// D_g = the running sum of the updates' max δ_j over the group's clusters (the
// two γ64 terms convert between the reference's rounded dots and real ones at
// t_s and at t). One global D (the maximum over all clusters) is dominated by
// the few clusters that move a lot — on c1 the largest drift is 10-50× the
// 90th percentile — and would hold every document hostage to them; per group,
// an unstable cluster only weakens its own group's bound, which is far from
// most documents' similarity anyway. A document whose own column is
// bit-identical to the previous iteration's (`same`: its cached similarity is
// exact) and whose cached own similarity exceeds every group's bound strictly
// keeps its cluster with exactly the reference's result — no other cluster can
// win or tie — and needs no screen. Every other document goes to a work list
// for the bound screen, ascending within each block's 1024-document range.
// (Documents whose own column moved need an own dot in any case; the screen
// computes it fused with its loads — measured: neither a separate own-dot pass
// nor an own-dot-first path inside the screen pays, most such documents fail
// the test.) The paper's use of centroid stability (unchanged clusters,
// engine.cpp:268-275) is the ε = 0 case of this bound.
struct SkipArgs {
    const int64_t* indptr;
    int64_t n;
    const uint32_t* a;
    const double* sims;
    const uint8_t* same;
    const __half* ub;        // [n][32]
    const uint32_t* ub_it;
    const double* dcum;      // D_g by iteration: [iteration][32]
    uint32_t iter;
    const float2* xb;
    double cmax;
    uint32_t* list;
    unsigned long long* n_list;
    unsigned long long* n_kept;  // documents kept out of the screen
};

#ifndef SSKM_SKIP_DOCS
#define SSKM_SKIP_DOCS 512  // documents per block (two per thread): 1024 -> 0.046 ms, 512 -> 0.040, 256 -> 0.043 on c1
#endif
constexpr int kSkipDocsPerBlock = SSKM_SKIP_DOCS;

// Per-group running drift: D_g(it) = D_g(it − 1) + sqrt(max_{j ≡ g} drift²_j)·(1 + 1e-9)
// (0 growth when the update cannot be followed: the host then invalidates the
// bounds). One block of 32 warps, warp g = group g.
__global__ void __launch_bounds__(1024) group_drift_kernel(const double* __restrict__ drift_sq, uint32_t k, int ok,
                                                           double* __restrict__ dcum, uint32_t iter) {
    const int lane = threadIdx.x & (kWarp - 1);
    for (int g = threadIdx.x / kWarp; g < kUbGroups; g += blockDim.x / kWarp) {
        double m = 0.0;
        if (ok)
            for (uint32_t j = g + kUbGroups * lane; j < k; j += kUbGroups * kWarp) m = fmax(m, drift_sq[j]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xFFFFFFFFu, m, off));
        if (lane == 0) {
            const double prev = iter > 0 ? dcum[static_cast<uint64_t>(iter - 1) * kUbGroups + g] : 0.0;
            // a NaN or negative drift cannot be followed either: the host checks the maximum
            dcum[static_cast<uint64_t>(iter) * kUbGroups + g] = prev + (ok && m > 0.0 ? sqrt(m) * (1.0 + 1e-9) : 0.0);
        }
    }
}

constexpr int kSkipHist = 64;  // iterations of group drift kept in shared memory (older bounds read global memory)

// A thread per document (four consecutive documents each): its 32 group
// bounds arrive as four 16-byte loads; the growth factors
// G[t][g] = (D_g(now) − D_g(t))·(1 + 1e-9), rounded up to fp32, of the last
// kSkipHist iterations sit in shared memory (row stride 33: lanes whose bounds
// date from different iterations hit different banks).
__global__ void __launch_bounds__(256) skip_kernel(SkipArgs p) {
    __shared__ float G[kSkipHist][kUbGroups + 1];
    __shared__ uint32_t wsum[8];
    __shared__ unsigned long long base_sm;
    const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x / kWarp, nwarps = blockDim.x / kWarp;
    const uint32_t t_lo = p.iter >= static_cast<uint32_t>(kSkipHist) ? p.iter - (kSkipHist - 1) : 0u;
    const double* __restrict__ dnow = p.dcum + static_cast<uint64_t>(p.iter) * kUbGroups;
    for (uint32_t e = threadIdx.x; e < (p.iter - t_lo + 1) * kUbGroups; e += blockDim.x) {
        const uint32_t r = e / kUbGroups, g = e % kUbGroups;
        G[r][g] = __double2float_ru((dnow[g] - p.dcum[static_cast<uint64_t>(t_lo + r) * kUbGroups + g]) * (1.0 + 1e-9));
    }
    __syncthreads();
    const int64_t d0 = static_cast<int64_t>(blockIdx.x) * kSkipDocsPerBlock;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(kSkipDocsPerBlock), p.n - d0));
    constexpr int kPer = kSkipDocsPerBlock / 256;
    const int my0 = threadIdx.x * kPer;  // four consecutive documents per thread
    bool kp[kPer];
    uint32_t mine = 0, out = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        kp[q] = false;
        if (my0 + q >= cnt) continue;
        const int64_t i = d0 + my0 + q;
        kp[q] = true;
        if (p.same[p.a[i]]) {
            const uint4* __restrict__ row = reinterpret_cast<const uint4*>(p.ub + static_cast<uint64_t>(i) * kUbGroups);
            constexpr int kV = kUbGroups / 8;  // 16-byte loads per document
            uint4 w[kV];
#pragma unroll
            for (int v = 0; v < kV; ++v) w[v] = row[v];
            const uint32_t its = p.ub_it[i];
            const float x2 = p.xb[i].y;
            float bmax = 0.f;  // every rounding upward; +inf marks a withdrawn bound
            auto fold2 = [&](uint32_t hh, float g0, float g1) {
                const __half2 h2 = *reinterpret_cast<const __half2*>(&hh);
                bmax = fmaxf(bmax, __fmaf_ru(x2, g0, __low2float(h2)));
                bmax = fmaxf(bmax, __fmaf_ru(x2, g1, __high2float(h2)));
            };
            if (its >= t_lo && its <= p.iter) {
                const float* __restrict__ gr = G[its - t_lo];
#pragma unroll
                for (int v = 0; v < kV; ++v) {
                    fold2(w[v].x, gr[8 * v + 0], gr[8 * v + 1]);
                    fold2(w[v].y, gr[8 * v + 2], gr[8 * v + 3]);
                    fold2(w[v].z, gr[8 * v + 4], gr[8 * v + 5]);
                    fold2(w[v].w, gr[8 * v + 6], gr[8 * v + 7]);
                }
            } else if (its > p.iter) {
                bmax = __int_as_float(0x7f800000);  // not a stamp of this run: no bound
            } else {  // a bound older than the shared history
                const double* __restrict__ dt = p.dcum + static_cast<uint64_t>(its) * kUbGroups;
                auto gg = [&](int g) { return __double2float_ru((dnow[g] - dt[g]) * (1.0 + 1e-9)); };
#pragma unroll
                for (int v = 0; v < kV; ++v) {
                    fold2(w[v].x, gg(8 * v + 0), gg(8 * v + 1));
                    fold2(w[v].y, gg(8 * v + 2), gg(8 * v + 3));
                    fold2(w[v].z, gg(8 * v + 4), gg(8 * v + 5));
                    fold2(w[v].w, gg(8 * v + 6), gg(8 * v + 7));
                }
            }
            const double nn = static_cast<double>(p.indptr[i + 1] - p.indptr[i]);
            const double b = static_cast<double>(bmax) + 2.0 * gamma_ub(nn, 0x1p-53) * x2 * p.cmax * (1.0 + 1e-12) +
                             nn * 0x1p-126;
            kp[q] = !(p.sims[i] > b);
        }
        mine += kp[q];
        out += !kp[q];
    }
    uint32_t incl = mine;
#pragma unroll
    for (int off = 1; off < kWarp; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += o;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) out += __shfl_xor_sync(0xFFFFFFFFu, out, off);
    if (lane == kWarp - 1) wsum[warp] = incl;
    if (lane == 0 && out) atomicAdd(p.n_kept, static_cast<unsigned long long>(out));
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (int w = 0; w < nwarps; ++w) {
        if (w < warp) before += wsum[w];
        total += wsum[w];
    }
    if (threadIdx.x == 0) base_sm = total ? atomicAdd(p.n_list, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    unsigned long long o = base_sm + before + (incl - mine);
#pragma unroll
    for (int q = 0; q < kPer; ++q)
        if (kp[q]) p.list[o++] = static_cast<uint32_t>(d0 + my0 + q);
}

// High postings of the cluster tile [c0, c0 + kt) of M in one pass over M:
// per term, the (column, value) pairs with |value| ≥ thr in ascending column,
// at a block-reserved offset (one atomic per 8 terms). Lists land in any order;
// hptr[t] = (first pair, count, largest |value| below thr, 0). Pairs beyond
// `cap` are not written (the host grows the buffer and rebuilds when
// *total > cap).
// With `slack`, every list gets room to grow (cnt/2 + 4 slots, filled with
// (kNone, 0)) and hptr[t].w = (sorted length << 16) | capacity: the column
// rewrite then maintains the lists in place from one iteration to the next
// (hipost_maintain); a row without room (w = 0) raises the rebuild flag on its
// first append.
__global__ void __launch_bounds__(256, 8) hipost_build_kernel(const float* __restrict__ M, uint64_t ld, uint32_t d,
                                                           uint32_t c0, uint32_t kt, float thr,
                                                           uint4* __restrict__ hptr, uint2* __restrict__ pairs,
                                                           unsigned long long cap, unsigned long long* total,
                                                           unsigned long long* overflow, int slack) {
    __shared__ uint32_t s_cnt[8];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x / kWarp;
    const unsigned lt = (1u << lane) - 1u;
    const uint32_t kt4 = kt & ~3u;
    for (uint64_t tb = static_cast<uint64_t>(blockIdx.x) * 8; tb < d; tb += static_cast<uint64_t>(gridDim.x) * 8) {
        const uint64_t t = tb + warp;
        const float* row = M + t * ld + c0;
        uint32_t cnt = 0;
        float lowmax = 0.f, allmax = 0.f;
        if (t < d) {
            // 16-byte loads over the row (tiles start at multiples of 4 columns)
            for (uint32_t j = 4u * lane; j < kt4; j += 4u * kWarp) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(row + j));
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const bool k = post_keep(e[r], thr);
                    cnt += k;
                    lowmax = k ? lowmax : fmaxf(lowmax, fabsf(e[r]));
                    allmax = fmaxf(allmax, fabsf(e[r]));
                }
            }
            for (uint32_t j = kt4 + lane; j < kt; j += kWarp) {
                const bool k = post_keep(row[j], thr);
                cnt += k;
                lowmax = k ? lowmax : fmaxf(lowmax, fabsf(row[j]));
                allmax = fmaxf(allmax, fabsf(row[j]));
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, off);
            lowmax = fmaxf(lowmax, __shfl_xor_sync(0xFFFFFFFFu, lowmax, off));
            allmax = fmaxf(allmax, __shfl_xor_sync(0xFFFFFFFFu, allmax, off));
        }
        // with slack: room for cnt/2 + 4 more (capacity and sorted length share
        // hptr.w as 16-bit halves, so rows past 40,000 entries get none)
        const bool grow = slack && cnt <= 40000u;
        const uint32_t room = t < d ? cnt + (grow ? cnt / 2 + 4 : 0) : 0;
        if (lane == 0) s_cnt[warp] = room;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) sum += s_cnt[q];
            s_base = sum ? atomicAdd(total, static_cast<unsigned long long>(sum)) : 0ull;
        }
        __syncthreads();
        unsigned long long b = s_base;
        for (int q = 0; q < warp; ++q) b += s_cnt[q];
        if (t < d) {
            // a list past the buffer's end is dropped, and the term's bound then
            // covers every weight of the row (count 0, L_t = max |value|): the
            // screen stays exact, only looser (the host grows the buffer after)
            const bool fits = b + room <= cap;
            if (lane == 0) {
                hptr[t] = fits ? make_uint4(static_cast<uint32_t>(b), cnt, __float_as_uint(lowmax),
                                            grow ? (cnt << 16) | room : 0u)
                               : make_uint4(0u, 0u, __float_as_uint(allmax), 0u);
                if (!fits) atomicOr(overflow, 1ull);
            }
            if (fits)
                for (uint32_t q = cnt + lane; q < room; q += kWarp) pairs[b + q] = make_uint2(kNone, 0u);
            if (cnt > 0 && fits) {
                // 16-byte loads again (the row is in L1/L2 now); each lane's kept
                // values go to its prefix position within the 128 columns
                uint32_t run = 0;
                for (uint32_t j0 = 0; j0 < kt4 && run < cnt; j0 += 4u * kWarp) {
                    const uint32_t j = j0 + 4u * lane;
                    float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (j < kt4) v4 = __ldg(reinterpret_cast<const float4*>(row + j));
                    const float e[4] = {v4.x, v4.y, v4.z, v4.w};
                    uint32_t mine = 0;
#pragma unroll
                    for (int r = 0; r < 4; ++r) mine += post_keep(e[r], thr);
                    uint32_t incl = mine;
#pragma unroll
                    for (int off = 1; off < kWarp; off <<= 1) {
                        const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, off);
                        if (lane >= off) incl += o;
                    }
                    uint64_t o = b + run + (incl - mine);
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (post_keep(e[r], thr)) pairs[o++] = make_uint2(j + r, __float_as_uint(e[r]));
                    run += __shfl_sync(0xFFFFFFFFu, incl, kWarp - 1);
                }
                for (uint32_t j0 = kt4; j0 < kt && run < cnt; j0 += kWarp) {  // the tail columns
                    const uint32_t j = j0 + lane;
                    const float v = j < kt ? row[j] : 0.f;
                    const bool keep = j < kt && post_keep(v, thr);
                    const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
                    if (keep) pairs[b + run + __popc(m & lt)] = make_uint2(j, __float_as_uint(v));
                    run += __popc(m);
                }
            }
        }
        __syncthreads();  // s_cnt / s_base reuse
    }
}

__global__ void doc_freq_kernel(const int32_t* __restrict__ idx, int64_t nnz, uint32_t* __restrict__ df) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(df + idx[e], 1u);
}

// Σ_t df_t · |high list of t| (the high pairs all documents would accumulate).
__global__ void pairs_expect_kernel(const uint4* __restrict__ hptr, const uint32_t* __restrict__ df, uint32_t d,
                                    unsigned long long* out) {
    unsigned long long s = 0;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < d; t += gridDim.x * blockDim.x)
        s += static_cast<unsigned long long>(df[t]) * hptr[t].y;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, off);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// NCC pass A over the bound-screened documents: queue the rescan exactly as
// the reference decides it (engine.cpp:303-305); the exact-scan documents
// queue themselves in assign_tile_kernel.
__global__ void bound_ncc_rescan_kernel(const uint32_t* __restrict__ order, int64_t n_work,
                                        const uint8_t* __restrict__ take, const uint32_t* __restrict__ a_start,
                                        const double* __restrict__ sims_start, const double* __restrict__ sims,
                                        const uint8_t* __restrict__ unchanged, uint32_t* __restrict__ rescan_list,
                                        unsigned long long* n_rescan) {
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < n_work;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (!take[w]) continue;
        const uint32_t i = order ? order[w] : static_cast<uint32_t>(w);
        if (unchanged[a_start[i]] == 0 && !(sims[i] > sims_start[i])) {
            const unsigned long long pos = atomicAdd(n_rescan, 1ull);
            rescan_list[pos] = i;
        }
    }
}

__global__ void narrow_u32_kernel(const int64_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint32_t>(in[i]);
}

// Per-document bound inputs, once per upload: (‖x‖₁, ‖x‖₂) rounded up to fp32
// (rounding up keeps every bound valid; one 8-byte load per document).
__global__ void doc_bound_norms_kernel(const int64_t* __restrict__ indptr, const float* __restrict__ val, int64_t n,
                                       const double* __restrict__ xnorm2, float2* __restrict__ out) {
    const int lane = threadIdx.x & (kWarp - 1);
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * blockDim.x / kWarp;
    for (uint64_t i = gw; i < static_cast<uint64_t>(n); i += nw) {
        double q = 0.0;
        for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += kWarp) q += fabs(static_cast<double>(val[e]));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) q += __shfl_xor_sync(0xFFFFFFFFu, q, off);
        // the fp64 sums' rounding (< (n + 2)·2^-53 relative) covered
        const double m = static_cast<double>(indptr[i + 1] - indptr[i]);
        const double x1 = q * (1.0 + (m + 2.0) * 0x1p-52);
        const double x2 = sqrt(xnorm2[i] * (1.0 + (m + 2.0) * 0x1p-52)) * (1.0 + 0x1p-50);
        if (lane == 0) out[i] = make_float2(__double2float_ru(x1), __double2float_ru(x2));
    }
}

}  // namespace sskm_b200
