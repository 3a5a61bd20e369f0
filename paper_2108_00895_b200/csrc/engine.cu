// sskm_b200 engine: device-resident Lloyd iterations behind the C-ABI in
// include/sskm_b200.h. Host C++ orchestrates; all per-document and
// per-centroid work runs in the kernels of assign_kernels.cuh and
// update_kernels.cuh on one CUDA stream.
//
// Mirrors the reference loop (engine.cpp:345-425):
//   update  = compute_centroids (:137-195) + detect_unchanged (:197-216) + repaired rule (:371-376)
//   assign  = assign (:218-322) + objective Σ sims (:403-405)
//   run     = stop on no reassignment (:409-412) or drift < conv_sq_dist after iteration 1 (:413-416)
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/sskm_b200.h"
#include "assign_kernels.cuh"
#include "bound_kernels.cuh"
#include "common.cuh"
#include "index_kernels.cuh"
#include "update_kernels.cuh"

namespace sskm_b200 {

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

// Device scalars, one allocation.
struct Scalars {
    unsigned long long n_moved;
    unsigned long long n_rescan;
    unsigned long long n_exact;
    unsigned long long reassigned;
    unsigned long long max_drift_bits;
    unsigned long long donor_key;
    unsigned long long donor_idx;
    unsigned int n_rec;
    unsigned int n_chg;
    unsigned int n_empty;
    unsigned int n_unchanged;
    unsigned int bad;
    unsigned int zero_flag;
    unsigned int hp_ovf;  // in-place high-postings maintenance ran out of room (rebuild)
    double objective;
};

// Scalars and the screens' counters, contiguous (Engine::pull_block).
struct CounterBlock {
    Scalars s;
    unsigned long long bctr[8];  // bound screen counters
    unsigned long long sk[4];    // drift-bound pass: work-list length, documents kept (zeroed with bctr)
    unsigned long long hp[2];    // high-postings build: pairs reserved, lists dropped (kept across passes)
};

static_assert(offsetof(CounterBlock, sk) == offsetof(CounterBlock, bctr) + 8 * sizeof(unsigned long long),
              "the screen's and the drift-bound pass's counters are zeroed by one memset");

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    bool owned = true;
    void alloc(size_t count) {
        if (count <= n && p) return;
        free();
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        n = count;
        owned = true;
    }
    // a fixed-size window of another allocation (never grown, not freed here)
    void view(T* ptr, size_t count) {
        free();
        p = ptr;
        n = count;
        owned = false;
    }
    void free() {
        if (p && owned) cudaFree(p);
        p = nullptr;
        n = 0;
        owned = true;
    }
    ~DevBuf() { free(); }
};

__global__ void zero_update_kernel(uint8_t* repaired_flag, uint32_t k, Scalars* sc) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) repaired_flag[j] = 0;
    if (j == 0) *sc = Scalars{};
}

// Zeroes what the assign's closing kernels accumulate into: the cluster sizes
// and the reassignment count, objective, range check and empty count.
__global__ void zero_closing_kernel(unsigned long long* counts, uint32_t k, Scalars* sc) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) counts[j] = 0ull;
    if (j == 0) {
        sc->reassigned = 0ull;
        sc->objective = 0.0;
        sc->bad = 0u;
        sc->n_empty = 0u;
    }
}

class Engine {
public:
    explicit Engine(int device) : device_(device) {
        int n_dev = 0;
        CK(cudaGetDeviceCount(&n_dev));
        if (device < 0 || device >= n_dev) throw InvalidArgument("invalid CUDA device ordinal");
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw CudaError("sskm_b200 requires an sm_100 (B200) device");
        sms_ = prop.multiProcessorCount;
        if (const char* e = std::getenv("SSKM_TILE_BYTES")) tile_bytes_ = std::strtoull(e, nullptr, 10);
        if (const char* e = std::getenv("SSKM_ORDER")) order_enabled_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_NCC_FULL_FRAC")) ncc_full_frac_ = std::atof(e);
        if (const char* e = std::getenv("SSKM_FUSE_RESOLVE")) fuse_resolve_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_BOUND")) bound_enabled_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_SKIP")) skip_enabled_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_SPECULATE")) speculate_ok_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_INDEX_ACCOUNTING")) index_accounting_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_WG_ROWS")) wg_rows_ = std::atoi(e);
        if (const char* e = std::getenv("SSKM_REBUILD_LATE")) rebuild_late_ = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("SSKM_SECOND_PASS")) second_pass_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_SECOND_RATIO")) second_pass_ratio_ = static_cast<float>(std::atof(e));
        if (const char* e = std::getenv("SSKM_SECOND_MIN")) second_pass_min_ = std::strtoull(e, nullptr, 10);
        if (const char* e = std::getenv("SSKM_KEEP_LISTS")) keep_lists_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_HASH")) hash_enabled_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_DEBUG")) debug_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_THETA")) {
            theta_ = static_cast<float>(std::atof(e));
            theta_adapt_ = false;
        }
        if (const char* e = std::getenv("SSKM_THETA0")) {  // starting point of the adaptive θ
            theta0_ = static_cast<float>(std::atof(e));
            theta0_set_ = true;
        }
        if (const char* e = std::getenv("SSKM_POST_KT")) post_kt_max_ = static_cast<uint32_t>(std::atoi(e));
        if (const char* e = std::getenv("SSKM_POST_WARPS")) post_warps_ = std::max(1, std::min(8, std::atoi(e)));
        if (const char* e = std::getenv("SSKM_DENSE_ABOVE")) dense_above_ = std::atof(e);
        if (const char* e = std::getenv("SSKM_SCREEN_KIND")) screen_kind_ = std::atoi(e);
        if (const char* e = std::getenv("SSKM_SCREEN")) screen_enabled_ = std::atoi(e) != 0;
        if (const char* e = std::getenv("SSKM_SCREEN_BLOCKS_PER_SM")) screen_blocks_per_sm_ = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("SSKM_BLOCKS_PER_SM")) blocks_per_sm_ = std::max(1, std::atoi(e));
        CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        for (auto& e : ev_) CK(cudaEventCreate(&e));
        for (auto& e : user_ev_) CK(cudaEventCreate(&e));
        // the step's scalars and the screens' counters in one device block with
        // one pinned host mirror: one copy brings them all back
        ctr_block_.alloc(1);
        CK(cudaMemsetAsync(ctr_block_.p, 0, sizeof(CounterBlock), stream_));
        scal_.view(&ctr_block_.p->s, 1);
        bctr_.view(ctr_block_.p->bctr, 8);
        hpctr_.view(ctr_block_.p->hp, 2);
        skip_ctr_.view(ctr_block_.p->sk, 4);
        CK(cudaMallocHost(&hblock_, sizeof(CounterBlock)));
        hs_ = &hblock_->s;
        // the screen keeps hot Cᵀ rows in L1: give L1 the whole carveout
        for (auto k : {screen_tile_kernel<1, 16>, screen_tile_kernel<2, 16>, screen_tile_kernel<4, 16>})
            CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    }

    ~Engine() {
        cudaSetDevice(device_);
        cudaStreamSynchronize(stream_);
        for (auto& e : ev_) cudaEventDestroy(e);
        if (stage_[0]) cudaFreeHost(stage_[0]);  // one allocation, two halves
        for (int b = 0; b < 2; ++b)
            if (stage_ev_[b]) cudaEventDestroy(stage_ev_[b]);
        for (auto& e : user_ev_) cudaEventDestroy(e);
        cudaStreamDestroy(stream_);
        if (hblock_) cudaFreeHost(hblock_);
    }

    // Every kernel goes through here: one place to count launches (bench's
    // gpu_launches) and to pin the stream.
    template <typename... KArgs, typename... Args>
    void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, Args&&... args) {
        kernel<<<grid, block, 0, stream_>>>(std::forward<Args>(args)...);
        ++launches_;
    }

    uint64_t launches() const { return launches_; }

    void timer_record(int slot) {
        if (slot < 0 || slot >= kUserEvents) throw InvalidArgument("timer slot out of range");
        CK(cudaEventRecord(user_ev_[slot], stream_));
    }

    double timer_elapsed(int a, int b) {
        if (a < 0 || a >= kUserEvents || b < 0 || b >= kUserEvents) throw InvalidArgument("timer slot out of range");
        CK(cudaEventSynchronize(user_ev_[b]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, user_ev_[a], user_ev_[b]));
        return ms;
    }

    void synchronize() { CK(cudaStreamSynchronize(stream_)); }

    // ------------------------------------------------------------ corpus --
    // Host -> device copy of a large pageable buffer through two pinned 8 MB
    // staging buffers (halves of one allocation): the host copies (parallel
    // threads, ~43 GB/s) into one while the other's DMA runs. The driver's own
    // pageable path runs at ~8-10 GB/s here. One allocation of 16 MB: page-
    // locking costs ~6 ms per call plus ~0.1-0.4 ms per MB on this host — the
    // two 64 MB buffers of round 1 cost 60-80 ms per engine, more than the
    // 0.56 GB c1 upload itself.
    void h2d(void* dst, const void* src, size_t bytes) {
        constexpr size_t kChunk = size_t(8) << 20;
        if (bytes >= (size_t(8) << 20) && !stage_failed_ && !stage_[0]) {
            const auto ta0 = std::chrono::steady_clock::now();
            const cudaError_t ea = cudaMallocHost(&stage_[0], 2 * kChunk);
            if (debug_)
                std::fprintf(stderr, "[sskm] pinned staging %zu MB: %.2f ms\n", (2 * kChunk) >> 20,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta0).count());
            if (ea != cudaSuccess) {  // no pinned memory: pageable copies
                (void)cudaGetLastError();
                stage_[0] = nullptr;
                stage_failed_ = true;
            } else {
                stage_[1] = static_cast<char*>(stage_[0]) + kChunk;
                for (int b = 0; b < 2; ++b) {
                    CK(cudaEventCreateWithFlags(&stage_ev_[b], cudaEventDisableTiming));
                    stage_used_[b] = false;
                }
            }
        }
        if (bytes < (size_t(8) << 20) || stage_failed_) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_));
            return;
        }
        size_t off = 0;
        for (int i = 0; off < bytes; ++i, off += kChunk) {
            const int b = i & 1;
            const size_t len = std::min(kChunk, bytes - off);
            const auto tw0 = std::chrono::steady_clock::now();
            if (stage_used_[b]) CK(cudaEventSynchronize(stage_ev_[b]));
            const auto tw1 = std::chrono::steady_clock::now();
            const char* s = static_cast<const char*>(src) + off;
            char* d = static_cast<char*>(stage_[b]);
            constexpr size_t kPiece = size_t(1) << 20;
            const int64_t pieces = static_cast<int64_t>(ceil_div(len, kPiece));
#pragma omp parallel for schedule(static)
            for (int64_t q = 0; q < pieces; ++q) {
                const size_t o = static_cast<size_t>(q) * kPiece;
                std::memcpy(d + o, s + o, std::min(kPiece, len - o));
            }
            const auto tw2 = std::chrono::steady_clock::now();
            CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage_[b], len, cudaMemcpyHostToDevice, stream_));
            CK(cudaEventRecord(stage_ev_[b], stream_));
            stage_used_[b] = true;
            h2d_wait_ms_ += std::chrono::duration<double, std::milli>(tw1 - tw0).count();
            h2d_copy_ms_ += std::chrono::duration<double, std::milli>(tw2 - tw1).count();
        }
    }

    void upload(int64_t n, uint32_t dims, const int64_t* indptr, const int32_t* indices,
                const float* values, int64_t doc_offset, int64_t n_total) {
        counts_fresh_ = false;
        CK(cudaSetDevice(device_));
        // nothing of the previous corpus / configuration stays usable: the
        // buffers below are resized for the new corpus, and a failed validation
        // must not leave a context whose sizes disagree with its buffers
        corpus_ = false;
        state_ = false;
        ub_valid_ = false;
        df_ready_ = false;
        k_ = 0;
        if (n <= 0) throw InvalidArgument("empty corpus");
        if (dims == 0) throw InvalidArgument("dims must be positive");
        if (indptr[0] != 0) throw InvalidArgument("indptr[0] must be 0");
        const int64_t nnz = indptr[n];
        if (nnz < 0 || nnz > (int64_t(1) << 40)) throw InvalidArgument("bad nnz");
        if (n > 0xFFFFFFF0ll) throw InvalidArgument("too many documents for 32-bit ids");
        n_ = n;
        d_ = dims;
        nnz_ = nnz;
        doc_offset_ = doc_offset;
        n_total_ = n_total > 0 ? n_total : n;
        const auto tu0 = std::chrono::steady_clock::now();
        indptr_.alloc(n + 1);
        idx_.alloc(nnz);
        val_.alloc(nnz);
        const auto tu1 = std::chrono::steady_clock::now();
        h2d(indptr_.p, indptr, (n + 1) * sizeof(int64_t));
        if (nnz) {
            h2d(idx_.p, indices, nnz * sizeof(int32_t));
            h2d(val_.p, values, nnz * sizeof(float));
        }
        CK(cudaStreamSynchronize(stream_));
        const auto tu2 = std::chrono::steady_clock::now();
        if (debug_)
            std::fprintf(stderr, "[sskm] upload: alloc %.2f ms, copy %.2f ms (staging: host copies %.2f ms, waits %.2f ms)\n",
                         std::chrono::duration<double, std::milli>(tu1 - tu0).count(),
                         std::chrono::duration<double, std::milli>(tu2 - tu1).count(), h2d_copy_ms_, h2d_wait_ms_);
        reset_scalars();
        launch(validate_csr_kernel, grid_for(n, 256), 256, indptr_.p, idx_.p, val_.p, n, dims,
                                                                   &scal_.p->bad);
        CK_LAUNCH();
        pull_scalars();
        if (hs_->bad & 1u) throw InvalidArgument("indptr must be non-decreasing");
        if (hs_->bad & 2u)
            throw InvalidArgument("SparseVector: dims not strictly increasing (or out of range)");
        if (hs_->bad & 4u) throw InvalidArgument("SparseVector: zero weight");
        if (hs_->bad & 8u)
            throw InvalidArgument("document weights must be finite with |x| <= 1 (unit-length rows)");
        nonneg_ = (hs_->bad & 16u) == 0;
        xnorm2_.alloc(n);
        launch(doc_norm2_kernel, grid_for(n * 32, 256), 256, indptr_.p, val_.p, n, xnorm2_.p, &scal_.p->bad);
        CK_LAUNCH();
        pull_scalars();
        // every fixed-point bound (screen accumulators, the int64 sums and their
        // 128-bit norms) assumes ||x||_2 <= 1: rows must be unit length (fp32
        // rounding allowed) or shorter, e.g. empty (corpus.cpp:256-261 rejects
        // any non-unit row of a matrix file)
        if (hs_->bad & 32u) throw InvalidArgument("row is not unit length (norm above 1)");
        xb_.alloc(n);
        launch(doc_bound_norms_kernel, grid_for(n * 32, 256), 256, indptr_.p, val_.p, n, xnorm2_.p, xb_.p);
        CK_LAUNCH();
        // the bound screen's 32-bit offsets (its registers hold a pipeline of
        // them); above 2^32 nonzeros per device the postings screens are used
        bound_ok_ = nnz_ < (int64_t(1) << 32);
        if (bound_ok_) {
            indptr32_.alloc(n + 1);
            launch(narrow_u32_kernel, grid_for(n + 1, 256), 256, indptr_.p, n + 1, indptr32_.p);
            CK_LAUNCH();
        }
        // fixed-point scale: N_total · 2^K <= 2^62 with |x| <= 1
        int lg = 0;
        while ((int64_t(1) << lg) < n_total_) ++lg;
        K_ = 62 - lg;
        a_.alloc(n);
        a_sum_.alloc(n);
        a_start_.alloc(n);
        sims_.alloc(n);
        sims_start_.alloc(n);
        moved_.alloc(n);
        rescan_.alloc(n);
        corpus_ = true;
        state_ = false;
    }

    // ------------------------------------------------------------ config --
    static void validate(const sskm_run_config& c, uint64_t n_docs) {
        // RunConfig::validate, engine.cpp:47-64 (same messages)
        if (c.k < 2) throw InvalidArgument("k must be at least 2");
        if (c.k > n_docs)
            throw InvalidArgument("k (" + std::to_string(c.k) + ") exceeds the number of documents (" +
                                  std::to_string(n_docs) + ")");
        for (uint32_t i = 0; i < c.n_lambdas; ++i) {
            if (!(c.lambdas[i] > 0.0 && c.lambdas[i] < 1.0)) throw InvalidArgument("lambda must be in (0, 1)");
            if (i > 0 && !(c.lambdas[i] > c.lambdas[i - 1]))
                throw InvalidArgument("lambdas must be strictly ascending");
        }
        if (!(c.conv_sq_dist > 0.0)) throw InvalidArgument("conv_sq_dist must be positive");
        if (c.ncc_epsilon < 0.0) throw InvalidArgument("ncc_epsilon must be nonnegative");
        if (c.max_iters < 1) throw InvalidArgument("max_iters must be at least 1");
        if (c.mode < SSKM_MODE_BASELINE || c.mode > SSKM_MODE_NCC_INDEX)
            throw InvalidArgument("unknown mode (expected baseline, ncc, or ncc+index)");
    }

    void configure(const sskm_run_config& c) {
        counts_fresh_ = false;
        CK(cudaSetDevice(device_));
        if (!corpus_) throw InvalidArgument("upload a corpus before configuring");
        validate(c, static_cast<uint64_t>(n_total_));
        cfg_ = c;
        hp_valid_ = false;
        // θ per pass kind: tile passes start from the mean document length
        // (measured optima: 0.004 for 41 terms, 0.003 for 69,
        // 0.0005 for 650 — long documents make candidate dots dear, so a
        // lower θ, more high pairs and tighter bounds pay); hash passes from 0.02
        {
            const double len = static_cast<double>(nnz_) / static_cast<double>(std::max<int64_t>(1, n_));
            const float t0 = theta0_set_ ? theta0_
                                         : static_cast<float>(std::min(0.01, std::max(2e-4, 0.003 * std::pow(69.0 / std::max(1.0, len), 0.8))));
            for (auto& q : tctl_) q = ThetaCtl{};
            for (auto& q : tctl_) q.theta = t0;
            hash_theta0_ = theta0_set_ ? theta0_ : 0.02f;
            hash_theta_started_ = false;
        }
        lambdas_.assign(c.lambdas, c.lambdas + c.n_lambdas);
        cfg_.lambdas = lambdas_.data();
        // size every buffer for this (corpus, k); DevBuf::alloc only grows
        k_ = c.k;
        ld_ = static_cast<uint32_t>(round_up(k_, 128));
        const uint64_t dk = static_cast<uint64_t>(d_) * ld_;
        ct_.alloc(dk);
        S_.alloc(dk);
        unchanged_.alloc(k_);
        touched_.alloc(k_);
        repaired_flag_.alloc(k_);
        same_.alloc(k_);
        counts_.alloc(k_);
        chg_ids_.alloc(k_);
        drift_.alloc(k_);
        Q_.alloc(2 * static_cast<size_t>(k_));
        part_.alloc(ceil_div(d_, kRowBlock) * k_);
        state_ = false;
        have_cc_ = have_ids_ = false;
        cache_trusted_ = false;
        if (cfg_.mode != SSKM_MODE_BASELINE) cc_.alloc(static_cast<uint64_t>(d_) * ld_);
        obj_part_.alloc(kObjBlocks);
        prealloc();
    }

    // -------------------------------------------------------------- init --
    void reset_sums() {
        hp_valid_ = false;  // Cᵀ is about to be (re)initialised
        CK(cudaMemsetAsync(S_.p, 0, static_cast<uint64_t>(d_) * ld_ * sizeof(long long), stream_));
        // every group marked: Cᵀ may hold values the fresh sums do not (seeds,
        // teacher forcing); the first rewrite clears the marks of empty groups
        nz_.alloc(static_cast<size_t>(d_) * (ld_ / 32));
        CK(cudaMemsetAsync(nz_.p, 0xFF, static_cast<size_t>(d_) * (ld_ / 32) * sizeof(unsigned int), stream_));
        CK(cudaMemsetAsync(Q_.p, 0, 2 * static_cast<size_t>(k_) * sizeof(unsigned long long), stream_));
        launch(fill_u32_kernel, grid_for(n_, 256), 256, a_sum_.p, n_, kNone);
        CK_LAUNCH();
        CK(cudaMemsetAsync(touched_.p, 0, k_, stream_));
    }

    void init_from_seeds(const uint32_t* seeds_global) {
        need_config();
        hp_valid_ = false;
        std::vector<uint32_t> local(k_);
        for (uint32_t j = 0; j < k_; ++j) {
            const int64_t g = seeds_global[j];
            if (g < 0 || g >= n_total_) throw InvalidArgument("seed out of range");
            if (g < doc_offset_ || g >= doc_offset_ + n_)
                throw InvalidArgument("seed document is not on this shard");
            local[j] = static_cast<uint32_t>(g - doc_offset_);
        }
        DevBuf<uint32_t> dseeds;
        dseeds.alloc(k_);
        CK(cudaMemcpyAsync(dseeds.p, local.data(), k_ * 4, cudaMemcpyHostToDevice, stream_));
        CK(cudaMemsetAsync(ct_.p, 0, static_cast<uint64_t>(d_) * ld_ * sizeof(float), stream_));
        launch(scatter_seeds_kernel, grid_for(static_cast<int64_t>(k_) * 32, 256), 256, 
            indptr_.p, idx_.p, val_.p, dseeds.p, k_, ct_.p, ld_);
        CK_LAUNCH();
        seed_cmax(dseeds.p);
        seed_assign_state();
        sskm_iteration_stats st{};
        full_assign(&st);
        CK(cudaStreamSynchronize(stream_));
    }

    // Single-GPU k-means++ (engine.cpp:66-130), device-resident: per round the
    // seed's dots (kpp_round_kernel), the weights and their double-double prefix,
    // and an exact pick from bracketed sequential sums (kpp_pick_kernel); 16
    // bytes come back per round. A round whose pick the brackets cannot decide
    // (or SSKM_KPP_HOST=1) is replayed on the host in document order, as before.
    void init_kmeanspp(uint64_t seed, uint32_t* seeds_out) {
        need_config();
        if (n_ != n_total_) throw InvalidArgument("k-means++ seeding needs the whole corpus on one GPU");
        std::mt19937_64 gen(seed);
        auto uniform_unit = [&] { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
        auto uniform_index = [&](size_t n) {
            size_t i = static_cast<size_t>(uniform_unit() * static_cast<double>(n));
            return i < n ? i : n - 1;
        };
        const size_t n = static_cast<size_t>(n_);
        const bool host_only = std::getenv("SSKM_KPP_HOST") && std::atoi(std::getenv("SSKM_KPP_HOST")) != 0;
        std::vector<uint8_t> chosen(n, 0);
        std::vector<double> sims, cum;
        DevBuf<float> dense;
        dense.alloc(d_);
        DevBuf<uint8_t> dchosen;
        dchosen.alloc(n);
        DevBuf<double2> w, E;
        w.alloc(n);
        E.alloc(n);
        DevBuf<unsigned long long> ab;
        ab.alloc(2);
        size_t scan_bytes = 0;
        CK(cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, w.p, E.p, KppDD{}, static_cast<int>(n), stream_));
        DevBuf<unsigned char> scan_tmp;
        scan_tmp.alloc(scan_bytes);
        CK(cudaMemsetAsync(dense.p, 0, d_ * sizeof(float), stream_));
        CK(cudaMemsetAsync(dchosen.p, 0, n, stream_));
        launch(fill_u32_kernel, grid_for(n_, 256), 256, a_.p, n_, 0);
        launch(fill_f64_kernel, grid_for(n_, 256), 256, sims_.p, n_, -2.0);
        CK_LAUNCH();
        std::vector<uint32_t> seeds;
        kpp_host_rounds_ = 0;
        auto add_seed = [&](size_t doc, uint32_t cluster) {
            chosen[doc] = 1;
            seeds.push_back(static_cast<uint32_t>(doc));
            launch(set_u8_kernel, 1, 1, dchosen.p, static_cast<int64_t>(doc), static_cast<uint8_t>(1));
            launch(scatter_row_kernel, 1, 256, indptr_.p, idx_.p, val_.p, doc, dense.p, 0);
            launch(kpp_round_kernel, grid_for(n_, 256), 256, indptr_.p, idx_.p, val_.p, n_, dense.p, cluster, a_.p,
                   sims_.p);
            launch(scatter_row_kernel, 1, 256, indptr_.p, idx_.p, val_.p, doc, dense.p, 1);
            CK_LAUNCH();
        };
        // the reference's sequential round (engine.cpp:101-126) on the host
        auto host_round = [&](bool have_u, double u) -> size_t {
            sims.resize(n);
            cum.resize(n);
            CK(cudaMemcpyAsync(sims.data(), sims_.p, n * 8, cudaMemcpyDeviceToHost, stream_));
            CK(cudaStreamSynchronize(stream_));
            ++kpp_host_rounds_;
            double total = 0.0;
            for (size_t i = 0; i < n; ++i) {
                double wv = 0.0;
                if (!chosen[i]) {
                    const double dd = 1.0 - sims[i];
                    if (dd > 0.0) wv = dd * dd;
                }
                total += wv;
                cum[i] = total;
            }
            size_t pick;
            if (total > 0.0) {
                const double target = (have_u ? u : uniform_unit()) * total;
                pick = static_cast<size_t>(std::upper_bound(cum.begin(), cum.end(), target) - cum.begin());
                if (pick >= n) {
                    pick = n - 1;
                    while (chosen[pick]) --pick;
                }
            } else {
                pick = 0;
                while (chosen[pick]) ++pick;
            }
            return pick;
        };
        add_seed(uniform_index(n), 0);
        bool pending = false;  // a draw taken from the generator, not yet consumed by a round
        double u = 0.0;
        for (uint32_t c = 1; c < k_; ++c) {
            size_t pick;
            if (host_only) {
                pick = host_round(false, 0.0);
            } else {
                launch(kpp_weights_kernel, grid_for(n_, 256), 256, sims_.p, dchosen.p, n_, w.p);
                size_t tb = scan_bytes;
                CK(cub::DeviceScan::InclusiveScan(scan_tmp.p, tb, w.p, E.p, KppDD{}, static_cast<int>(n), stream_));
                ++launches_;
                // the draw of this round (the reference consumes it only when the total is positive)
                if (!pending) {
                    u = uniform_unit();
                    pending = true;
                }
                const unsigned long long init[2] = {static_cast<unsigned long long>(n), static_cast<unsigned long long>(n)};
                CK(cudaMemcpyAsync(ab.p, init, sizeof(init), cudaMemcpyHostToDevice, stream_));
                launch(kpp_pick_kernel, grid_for(n_, 256), 256, E.p, n_, u, ab.p);
                CK_LAUNCH();
                unsigned long long res[2];
                double2 last;
                CK(cudaMemcpyAsync(res, ab.p, sizeof(res), cudaMemcpyDeviceToHost, stream_));
                CK(cudaMemcpyAsync(&last, E.p + (n - 1), sizeof(last), cudaMemcpyDeviceToHost, stream_));
                CK(cudaStreamSynchronize(stream_));
                const bool positive = last.x + last.y > 0.0;  // a sum of nonnegative terms is 0 only if all are
                if (positive && res[0] == res[1] && res[0] < n) {
                    pick = static_cast<size_t>(res[0]);
                    pending = false;
                } else if (positive) {
                    pick = host_round(true, u);
                    pending = false;
                } else {
                    pick = host_round(true, u);  // total = 0: the lowest unchosen document; the draw stays pending
                }
            }
            add_seed(pick, c);
        }        // Cᵀ = the seed documents (informational; the first update recomputes all)
        DevBuf<uint32_t> dseeds;
        dseeds.alloc(k_);
        CK(cudaMemcpyAsync(dseeds.p, seeds.data(), k_ * 4, cudaMemcpyHostToDevice, stream_));
        CK(cudaMemsetAsync(ct_.p, 0, static_cast<uint64_t>(d_) * ld_ * sizeof(float), stream_));
        launch(scatter_seeds_kernel, grid_for(static_cast<int64_t>(k_) * 32, 256), 256, 
            indptr_.p, idx_.p, val_.p, dseeds.p, k_, ct_.p, ld_);
        CK_LAUNCH();
        seed_cmax(dseeds.p);
        reset_sums();
        CK(cudaMemsetAsync(unchanged_.p, 0, k_, stream_));
        ub_valid_ = false;
        iteration_ = 0;
        dcum_rows_ = 0;
        have_cc_ = have_ids_ = false;
        state_ = true;
        CK(cudaStreamSynchronize(stream_));
        if (seeds_out) std::memcpy(seeds_out, seeds.data(), k_ * 4);
    }

    // ------------------------------------------------------------ update --
    // compute_centroids + detect_unchanged for a single context (1 GPU).
    void update(sskm_iteration_stats* st) {
        need_state();
        CK(cudaEventRecord(ev_[0], stream_));
        iteration_ += 1;
        repaired_.clear();
        if (counts_fresh_) {
            // the last assign counted its clusters: none empty, every assignment in
            // range; one kernel clears the repaired flags and the step's scalars
            launch(zero_update_kernel, grid_for(k_, 256), 256, repaired_flag_.p, k_, scal_.p);
        } else {
            local_counts_device();
            repair_empty_single();
            reset_scalars();
        }
        counts_fresh_ = false;
        // rows that moved since the sums were last brought up to date
        launch(moved_kernel, grid_for(n_, 256), 256, a_.p, a_sum_.p, n_, moved_.p, &scal_.p->n_moved);
        CK_LAUNCH();
        launch(delta_local_kernel, grid_for(n_ * 32, 256), 256, 
            indptr_.p, idx_.p, val_.p, moved_.p, &scal_.p->n_moved, a_.p, a_sum_.p, a_sum_.p, S_.p, ld_, K_,
            touched_.p, Q_.p, nz_.p);
        CK_LAUNCH();
        finish_update(st);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        st->update_ms = ms;
        last_update_ms_ = ms;
    }

    // Multi-GPU update: apply rows gathered from every rank, then finish.
    void update_apply(int64_t n_moved, const uint32_t* old_c, const uint32_t* new_c, const int64_t* row_ptr,
                      const int32_t* idx, const float* val, const uint32_t* repaired, uint32_t n_repaired,
                      sskm_iteration_stats* st) {
        counts_fresh_ = false;
        need_state();
        CK(cudaEventRecord(ev_[0], stream_));
        iteration_ += 1;
        repaired_.assign(repaired, repaired + n_repaired);
        CK(cudaMemsetAsync(repaired_flag_.p, 0, k_, stream_));
        if (!repaired_.empty()) {
            std::vector<uint8_t> f(k_, 0);
            for (uint32_t j : repaired_) f[j] = 1;
            CK(cudaMemcpyAsync(repaired_flag_.p, f.data(), k_, cudaMemcpyHostToDevice, stream_));
        }
        // local owner map catches up (the local rows are part of the gathered set)
        fill_sum_owner_local();
        reset_scalars();
        if (n_moved > 0) {
            launch(delta_packed_kernel, grid_for(n_moved * 32, 256), 256, 
                n_moved, old_c, new_c, row_ptr, idx, val, S_.p, ld_, K_, touched_.p, Q_.p, nz_.p);
            CK_LAUNCH();
        }
        finish_update(st);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        st->update_ms = ms;
        st->n_moved = static_cast<uint64_t>(n_moved);
    }

    // ------------------------------------------------ multi-device phases --
    // The update of a MultiEngine step (multi.cuh), split at its exchange
    // points. Every device holds the full sums S and applies the moved rows of
    // every shard itself, reading the peers' shards over NVLink.
    struct PeerView {
        const int64_t* indptr;
        const int32_t* idx;
        const float* val;
        const uint32_t* moved;
        const unsigned long long* n_moved;
        const uint32_t* a;
        const uint32_t* a_sum;
        int64_t n;
    };
    PeerView peer_view() const {
        return {indptr_.p, idx_.p, val_.p, moved_.p, &scal_.p->n_moved, a_.p, a_sum_.p, n_};
    }
    int device() const { return device_; }
    int64_t doc_offset() const { return doc_offset_; }

    // 1. local cluster sizes, copied to the host
    void mp_begin(unsigned long long* counts_host) {
        counts_fresh_ = false;
        need_state();
        CK(cudaSetDevice(device_));
        CK(cudaEventRecord(ev_[0], stream_));
        iteration_ += 1;
        repaired_.clear();
        local_counts_device();
        CK(cudaMemcpyAsync(counts_host, counts_.p, k_ * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           stream_));
        pull_scalars();
        if (hs_->bad) throw InvalidArgument("assignment out of range");
    }

    // 2. this step's repairs (moves of local documents, as (local doc, cluster)
    // pairs; the repaired clusters of every device), then the moved list
    void mp_moved(const std::vector<uint32_t>& local_moves, const std::vector<uint32_t>& repaired,
                  cudaEvent_t done) {
        counts_fresh_ = false;
        CK(cudaSetDevice(device_));
        repaired_ = repaired;
        CK(cudaMemsetAsync(repaired_flag_.p, 0, k_, stream_));
        if (!repaired.empty()) {
            std::vector<uint8_t> f(k_, 0);
            for (uint32_t j : repaired) f[j] = 1;
            CK(cudaMemcpyAsync(repaired_flag_.p, f.data(), k_, cudaMemcpyHostToDevice, stream_));
        }
        if (!local_moves.empty()) {
            CK(cudaMemcpyAsync(moves_.p, local_moves.data(), local_moves.size() * 4, cudaMemcpyHostToDevice,
                               stream_));
            launch(apply_moves_kernel, 1, 256, moves_.p, static_cast<uint32_t>(local_moves.size() / 2), a_.p);
        }
        reset_scalars();
        launch(moved_kernel, grid_for(n_, 256), 256, a_.p, a_sum_.p, n_, moved_.p, &scal_.p->n_moved);
        CK_LAUNCH();
        CK(cudaEventRecord(done, stream_));
        if (!repaired.empty() || !local_moves.empty()) CK(cudaStreamSynchronize(stream_));  // host vectors
    }

    // 3. every shard's moved rows into the local sums, read from the peers
    void mp_delta(const std::vector<PeerView>& peers, const std::vector<cudaEvent_t>& moved_done,
                  cudaEvent_t done) {
        CK(cudaSetDevice(device_));
        for (cudaEvent_t e : moved_done) CK(cudaStreamWaitEvent(stream_, e, 0));
        for (const PeerView& q : peers)
            launch(delta_local_kernel, grid_for(q.n * 32, 256), 256, q.indptr, q.idx, q.val, q.moved, q.n_moved, q.a,
                   q.a_sum, static_cast<uint32_t*>(nullptr), S_.p, ld_, K_, touched_.p, Q_.p, nz_.p);
        CK_LAUNCH();
        CK(cudaEventRecord(done, stream_));
    }

    // 4. once every device has read this shard: the sums' owner map catches
    // up, then the column rewrite and flags (identical on every device)
    void mp_finish(const std::vector<cudaEvent_t>& delta_done, sskm_iteration_stats* st) {
        CK(cudaSetDevice(device_));
        for (cudaEvent_t e : delta_done) CK(cudaStreamWaitEvent(stream_, e, 0));
        fill_sum_owner_local();
        finish_update(st);
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
        st->update_ms = ms;
    }

    // Rows `ids` (local) of the shard as host CSR (seed rows for a multi-device init).
    void get_rows(const std::vector<uint32_t>& ids, std::vector<int64_t>& ptr, std::vector<int32_t>& idx,
                  std::vector<float>& val) {
        need_config();
        CK(cudaSetDevice(device_));
        const int64_t n = static_cast<int64_t>(ids.size());
        ptr.assign(n + 1, 0);
        idx.clear();
        val.clear();
        if (n == 0) return;
        DevBuf<uint32_t> dids;
        DevBuf<int64_t> lens, offs;
        dids.alloc(n);
        lens.alloc(n + 1);
        offs.alloc(n + 1);
        CK(cudaMemcpyAsync(dids.p, ids.data(), n * 4, cudaMemcpyHostToDevice, stream_));
        launch(row_lens_kernel, grid_for(n + 1, 256), 256, dids.p, n, indptr_.p, lens.p);
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, lens.p, offs.p, static_cast<int>(n + 1), stream_));
        DevBuf<unsigned char> tb;
        tb.alloc(tmp);
        CK(cub::DeviceScan::ExclusiveSum(tb.p, tmp, lens.p, offs.p, static_cast<int>(n + 1), stream_));
        ++launches_;
        CK(cudaMemcpyAsync(ptr.data(), offs.p, (n + 1) * 8, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        const int64_t nnz = ptr[n];
        DevBuf<int32_t> di, dl;
        DevBuf<float> dv;
        di.alloc(std::max<int64_t>(nnz, 1));
        dv.alloc(std::max<int64_t>(nnz, 1));
        dl.alloc(n);
        launch(pack_rows_kernel, grid_for(n * 32, 256), 256, dids.p, n, indptr_.p, idx_.p, val_.p, offs.p, dl.p, di.p,
               dv.p);
        CK_LAUNCH();
        idx.resize(nnz);
        val.resize(nnz);
        if (nnz) {
            CK(cudaMemcpyAsync(idx.data(), di.p, nnz * 4, cudaMemcpyDeviceToHost, stream_));
            CK(cudaMemcpyAsync(val.data(), dv.p, nnz * 4, cudaMemcpyDeviceToHost, stream_));
        }
        CK(cudaStreamSynchronize(stream_));
    }

    // ------------------------------------------------------------ assign --
    void assign(sskm_iteration_stats* st) {
        need_state();
        const bool full = iteration_ <= 1 || cfg_.mode == SSKM_MODE_BASELINE;
        st->iteration = iteration_;
        st->index_active = 0;
        st->index_queries = 0;
        st->candidates_total = 0;
        st->index_build_seconds = 0.0;
        if (full) {
            full_assign(st);
        } else {
            ncc_assign(st);
            // engine.cpp:384-386: the reference builds its Lemma-1 index when
            // more than index_activation_threshold centroids changed
            if (cfg_.mode == SSKM_MODE_NCC_INDEX && index_accounting_ && n_chg_ > cfg_.index_activation_threshold &&
                cfg_.n_lambdas > 0)
                index_account(st);
        }
    }

    // ---------------------------------------------------------- ncc+index --
    // Buffers whose size follows the centroids grow with headroom, so the
    // iteration-to-iteration drift does not reallocate every time.
    template <typename T>
    static void grow(DevBuf<T>& b, size_t count) {
        if (count > b.n) b.alloc(count + count / 4);
    }

    // The reference's Lemma-1 index over the current centroids and its queries
    // (index_kernels.cuh), replayed after the exact NCC assign to report the
    // reference's index_queries, candidates_total and dot_products.
    void index_account(sskm_iteration_stats* st) {
        const uint32_t L = cfg_.n_lambdas;
        CK(cudaEventRecord(ev_[6], stream_));
        // 1. supports, (|w| desc, term asc) per centroid
        const int64_t want = static_cast<int64_t>(sms_) * 2048;
        uint32_t nch = static_cast<uint32_t>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(want, k_), d_ / 16 + 1)));
        const uint32_t rows = static_cast<uint32_t>(ceil_div(d_, nch));
        nch = static_cast<uint32_t>(ceil_div(d_, rows));
        const uint64_t ncnt = static_cast<uint64_t>(k_) * nch;
        ix_cnt_.alloc(ncnt + 1);
        ix_off_.alloc(ncnt + 1);
        CK(cudaMemsetAsync(ix_cnt_.p + ncnt, 0, 4, stream_));
        const dim3 g2(static_cast<unsigned>(ceil_div(k_, 128)), nch);
        idx_support_count_kernel<<<g2, 128, 0, stream_>>>(ct_.p, ld_, d_, k_, rows, nch, ix_cnt_.p);
        ++launches_;
        CK_LAUNCH();
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ix_cnt_.p, ix_off_.p, static_cast<int>(ncnt + 1), stream_));
        grow(ix_tmp_, tmp);
        CK(cub::DeviceScan::ExclusiveSum(ix_tmp_.p, tmp, ix_cnt_.p, ix_off_.p, static_cast<int>(ncnt + 1), stream_));
        ++launches_;
        ix_cptr_.alloc(k_ + 1);
        // cluster c starts at off[c * nch]; the total is off[k * nch]
        CK(cudaMemcpy2DAsync(ix_cptr_.p, sizeof(uint64_t), ix_off_.p, sizeof(uint64_t) * nch, sizeof(uint64_t), k_ + 1,
                             cudaMemcpyDeviceToDevice, stream_));
        uint64_t nnz_c = 0;
        CK(cudaMemcpyAsync(&nnz_c, ix_off_.p + ncnt, 8, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        if (nnz_c >= (1ull << 31)) throw std::runtime_error("ncc+index: centroid supports too large for the index build");
        grow(ix_keys_, 2 * nnz_c + 1);
        idx_support_fill_kernel<<<g2, 128, 0, stream_>>>(ct_.p, ld_, d_, k_, rows, nch, ix_off_.p, ix_keys_.p);
        ++launches_;
        CK_LAUNCH();
        tmp = 0;
        CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, ix_keys_.p, ix_keys_.p + nnz_c, static_cast<int>(nnz_c),
                                              static_cast<int>(k_), ix_cptr_.p, ix_cptr_.p + 1, stream_));
        grow(ix_tmp_, tmp);
        CK(cub::DeviceSegmentedSort::SortKeys(ix_tmp_.p, tmp, ix_keys_.p, ix_keys_.p + nnz_c, static_cast<int>(nnz_c),
                                              static_cast<int>(k_), ix_cptr_.p, ix_cptr_.p + 1, stream_));
        ++launches_;
        const uint64_t* keys = ix_keys_.p + nnz_c;
        // 2. windows per (λ, centroid)
        ix_lam_.alloc(L);
        CK(cudaMemcpyAsync(ix_lam_.p, lambdas_.data(), sizeof(double) * L, cudaMemcpyHostToDevice, stream_));
        grow(ix_mval_, static_cast<size_t>(L) * nnz_c + 1);
        ix_jlen_.alloc(static_cast<size_t>(L) * k_);
        launch(idx_window_kernel, static_cast<unsigned>(ceil_div(static_cast<int64_t>(k_) * L * 32, 128)), 128, keys,
               ix_cptr_.p, k_, ix_lam_.p, L, nnz_c, ix_mval_.p, ix_jlen_.p);
        CK_LAUNCH();
        CK(cudaEventRecord(ev_[7], stream_));
        // 3. per-document rescan flags and λ selection
        ix_rescan_.alloc(n_);
        if (last_full_equiv_) {
            launch(idx_rescan_formula_kernel, grid_for(n_, 256), 256, a_start_.p, sims_start_.p, sims_.p,
                   unchanged_.p, n_, ix_rescan_.p);
        } else {
            CK(cudaMemsetAsync(ix_rescan_.p, 0, n_, stream_));
            if (last_n_rescan_ > 0)
                launch(idx_rescan_scatter_kernel, grid_for(static_cast<int64_t>(last_n_rescan_), 256), 256, rescan_.p,
                       static_cast<int64_t>(last_n_rescan_), ix_rescan_.p);
        }
        ix_sel_.alloc(n_);
        ix_list_.alloc(n_);
        ix_ctr_.alloc(5);
        CK(cudaMemsetAsync(ix_ctr_.p, 0, 5 * sizeof(unsigned long long), stream_));
        IndexSelArgs sa{};
        sa.indptr = indptr_.p;
        sa.idx = idx_.p;
        sa.val = val_.p;
        sa.CT = ct_.p;
        sa.ld_ct = ld_;
        sa.n = n_;
        sa.a_start = a_start_.p;
        sa.sims_start = sims_start_.p;
        sa.unchanged = unchanged_.p;
        sa.rescan = ix_rescan_.p;
        sa.lambdas = ix_lam_.p;
        sa.n_lambdas = L;
        sa.n_changed = n_chg_;
        sa.n_unchanged = k_ - n_chg_;
        sa.sel = ix_sel_.p;
        sa.counters = ix_ctr_.p;
        launch(idx_select_kernel, grid_for(n_ * 32, 256), 256, sa);
        CK_LAUNCH();
        // 4. queries, per cluster tile and λ
        constexpr uint32_t KT = 1024;
        auto qk = idx_query_kernel<KT>;
        const int warps = 8;
        const size_t smem = static_cast<size_t>(warps) * 2 * KT * sizeof(uint32_t);
        CK(cudaFuncSetAttribute(qk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qk, warps * 32, smem));
        ix_lcnt_.alloc(d_ + 1);
        ix_lptr_.alloc(d_ + 1);
        ix_fill_.alloc(d_);
        // documents grouped by λ: one compact pass per λ into consecutive ranges
        std::vector<int64_t> l_beg(L + 1, 0);
        {
            int64_t pos = 0;
            for (uint32_t l = 0; l < L; ++l) {
                CK(cudaMemsetAsync(ix_ctr_.p + 4, 0, 8, stream_));
                launch(idx_compact_kernel, grid_for(n_, 256), 256, ix_sel_.p, n_, l, ix_list_.p + pos, ix_ctr_.p + 4);
                unsigned long long m = 0;
                CK(cudaMemcpyAsync(&m, ix_ctr_.p + 4, 8, cudaMemcpyDeviceToHost, stream_));
                CK(cudaStreamSynchronize(stream_));
                l_beg[l] = pos;
                pos += static_cast<int64_t>(m);
                l_beg[l + 1] = pos;
            }
        }
        for (uint32_t c0 = 0; c0 < k_; c0 += KT) {
            const uint32_t kt = std::min<uint32_t>(KT, k_ - c0);
            bool built = false;
            for (uint32_t l = 0; l < L; ++l) {
                const int64_t nl = l_beg[l + 1] - l_beg[l];
                if (nl == 0) continue;
                if (!built) {
                    build_postings(ct_.p, ld_, c0, kt);  // general postings of the tile
                    built = true;
                }
                const uint32_t* jl = ix_jlen_.p + static_cast<size_t>(l) * k_;
                const uint32_t* mv = ix_mval_.p + static_cast<size_t>(l) * nnz_c;
                CK(cudaMemsetAsync(ix_lcnt_.p, 0, sizeof(uint32_t) * (d_ + 1), stream_));
                launch(idx_lam_count_kernel, static_cast<unsigned>(ceil_div(static_cast<int64_t>(kt) * 32, 256)), 256,
                       keys, ix_cptr_.p, jl, c0, kt, ix_lcnt_.p);
                size_t t2 = 0;
                CK(cub::DeviceScan::ExclusiveSum(nullptr, t2, ix_lcnt_.p, ix_lptr_.p, static_cast<int>(d_ + 1),
                                                 stream_));
                grow(ix_tmp_, t2);
                CK(cub::DeviceScan::ExclusiveSum(ix_tmp_.p, t2, ix_lcnt_.p, ix_lptr_.p, static_cast<int>(d_ + 1),
                                                 stream_));
                ++launches_;
                uint32_t tot = 0;
                CK(cudaMemcpyAsync(&tot, ix_lptr_.p + d_, 4, cudaMemcpyDeviceToHost, stream_));
                CK(cudaStreamSynchronize(stream_));
                grow(ix_lent_, static_cast<size_t>(tot) + 1);
                CK(cudaMemsetAsync(ix_fill_.p, 0, sizeof(uint32_t) * d_, stream_));
                launch(idx_lam_fill_kernel, static_cast<unsigned>(ceil_div(static_cast<int64_t>(kt) * 32, 256)), 256,
                       keys, ix_cptr_.p, jl, mv, c0, kt, ix_lptr_.p, ix_fill_.p, ix_lent_.p);
                IndexQueryArgs q{};
                q.indptr = indptr_.p;
                q.idx = idx_.p;
                q.gptr = pptr_.p;
                q.gpairs = pairs_.p;
                q.lptr = ix_lptr_.p;
                q.lent = ix_lent_.p;
                q.c0 = c0;
                q.kt = kt;
                q.list = ix_list_.p + l_beg[l];
                q.n_list = nl;
                q.a_start = a_start_.p;
                q.unchanged = unchanged_.p;
                q.rescan = ix_rescan_.p;
                q.counters = ix_ctr_.p;
                const unsigned grid = static_cast<unsigned>(
                    std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(sms_) * std::max(1, per_sm),
                                                           ceil_div(nl, warps))));
                qk<<<grid, warps * 32, smem, stream_>>>(q);
                ++launches_;
                CK_LAUNCH();
            }
        }
        unsigned long long ctr[4] = {0, 0, 0, 0};
        CK(cudaMemcpyAsync(ctr, ix_ctr_.p, sizeof(ctr), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        float build_ms = 0.f;
        CK(cudaEventElapsedTime(&build_ms, ev_[6], ev_[7]));
        st->index_active = 1;
        st->index_build_seconds = build_ms * 1e-3;
        st->index_queries = ctr[0];
        st->candidates_total = ctr[2];
        st->dot_products = st->dot_products - ctr[1] + ctr[3];
    }

    void full_assign(sskm_iteration_stats* st) {
        CK(cudaEventRecord(ev_[2], stream_));
        snapshot_start();
        // the bound screen streams documents in index order (consecutive CSR rows:
        // measured 1.75 -> 1.40 ms per c1 screen against the cluster order the
        // tile scans prefer)
        const uint32_t* order = bound_active() ? nullptr : cluster_order();
        reset_scalars();
        uint64_t n_exact = 0;
        if (screen_enabled_) {
            // (the closing kernels ride along with the screen when the last full
            // scan left no document for the exact scan: bound_assign)
            speculate_finish_ = speculate_ok_ && last_full_n_exact_ == 0 && order == nullptr;
            if (!screen_any(ct_.p, ld_, k_, nullptr, nullptr, order, n_, kInitFull)) resolve<kInitFull>(order, n_);
            speculate_finish_ = false;
            pull_scalars_unless_fresh();
            n_exact = hs_->n_exact;
            last_full_n_exact_ = n_exact;
            if (n_exact > 0) scan_tiles<kInitFull>(ct_.p, ld_, k_, nullptr, exact_.p, static_cast<int64_t>(n_exact));
        } else {
            scan_tiles<kInitFull>(ct_.p, ld_, k_, nullptr, order, n_);
        }
        if (!bound_active()) ub_valid_ = false;
        finish_assign(st);
        cache_trusted_ = true;
        st->n_unchanged_centroids = iteration_ <= 1 ? 0 : n_unchanged_;
        st->dot_products = static_cast<uint64_t>(k_) * static_cast<uint64_t>(n_);
        st->gpu_dot_products = dots_;
        st->n_changed = k_;
        st->n_rescan = 0;
        st->n_exact = n_exact;
        timing(st);
    }

    void ncc_assign(sskm_iteration_stats* st) {
        CK(cudaEventRecord(ev_[2], stream_));
        snapshot_start();
        ensure_cc(false);
        // the bound screen streams documents in index order (consecutive CSR rows:
        // measured 1.75 -> 1.40 ms per c1 screen against the cluster order the
        // tile scans prefer)
        const uint32_t* order = bound_active() ? nullptr : cluster_order();
        reset_scalars();
        uint64_t n_exact = 0, n_rescan = 0;
        // With ncc_epsilon = 0 and a cache this engine produced, the NCC result
        // equals the full scan bit for bit; when many centroids
        // changed the full screened scan is the cheaper way to get it.
        const bool full_equiv = cfg_.ncc_epsilon == 0.0 && cache_trusted_ && screen_enabled_ &&
                                static_cast<double>(n_chg_) >= ncc_full_frac_ * k_;
        if (n_chg_ > 0 && full_equiv) {
            if (!screen_any(ct_.p, ld_, k_, nullptr, nullptr, order, n_, kInitFull)) resolve<kInitFull>(order, n_);
            pull_scalars_unless_fresh();
            n_exact = hs_->n_exact;
            if (n_exact > 0) scan_tiles<kInitFull>(ct_.p, ld_, k_, nullptr, exact_.p, static_cast<int64_t>(n_exact));
            CK(cudaMemsetAsync(&scal_.p->n_rescan, 0, 8, stream_));
            launch(ncc_rescan_count_kernel, grid_for(n_, 256), 256, a_start_.p, sims_start_.p, sims_.p, unchanged_.p,
                   n_, &scal_.p->n_rescan);
            CK_LAUNCH();
            pull_scalars();
            n_rescan = hs_->n_rescan;
        } else if (n_chg_ > 0) {
            ensure_cc(true);
            if (screen_enabled_) {
                if (!screen_any(cc_.p, ld_cc_, n_chg_, chg_ids_.p, a_start_.p, order, n_, kInitNcc))
                    resolve<kInitNcc>(order, n_);
                pull_scalars_unless_fresh();
                n_exact = hs_->n_exact;
                if (n_exact > 0)
                    scan_tiles<kInitNcc>(cc_.p, ld_cc_, n_chg_, chg_ids_.p, exact_.p, static_cast<int64_t>(n_exact));
            } else {
                scan_tiles<kInitNcc>(cc_.p, ld_cc_, n_chg_, chg_ids_.p, order, n_);
            }
            pull_scalars();
            n_rescan = hs_->n_rescan;
            if (n_rescan > 0) {
                // pass B over all centroids for the rescan documents (engine.cpp:303-305)
                if (screen_enabled_) {
                    CK(cudaMemsetAsync(&scal_.p->n_exact, 0, 8, stream_));
                    if (!screen_any(ct_.p, ld_, k_, nullptr, a_.p, rescan_.p, static_cast<int64_t>(n_rescan), kInitRescan))
                        resolve<kInitRescan>(rescan_.p, static_cast<int64_t>(n_rescan));
                    pull_scalars_unless_fresh();
                    const uint64_t nx = hs_->n_exact;
                    n_exact += nx;
                    if (nx > 0) scan_tiles<kInitRescan>(ct_.p, ld_, k_, nullptr, exact_.p, static_cast<int64_t>(nx));
                } else {
                    scan_tiles<kInitRescan>(ct_.p, ld_, k_, nullptr, rescan_.p, static_cast<int64_t>(n_rescan));
                }
            }
        }
        if (!(n_chg_ > 0 && full_equiv)) ub_valid_ = false;  // per-document bounds not refreshed for every document
        last_full_equiv_ = n_chg_ > 0 && full_equiv;
        last_n_rescan_ = n_rescan;
        finish_assign(st);
        cache_trusted_ = true;
        // dot accounting of the reference (engine.cpp:253-306): every document
        // evaluates the changed list (minus its own centroid, which a
        // changed-own document evaluates as its refresh), plus the unchanged
        // list when the refreshed scan did not beat the cache.
        const uint64_t n_unch = k_ - n_chg_;
        st->n_unchanged_centroids = static_cast<uint32_t>(n_unch);
        st->dot_products = static_cast<uint64_t>(n_) * n_chg_ + n_rescan * n_unch;
        st->gpu_dot_products = dots_;
        st->n_changed = n_chg_;
        st->n_rescan = n_rescan;
        st->n_exact = n_exact;
        timing(st);
    }

    // ------------------------------------------------------------ access --
    void get_state(uint32_t* a, double* sims, uint8_t* unchanged) {
        need_state();
        if (a) CK(cudaMemcpyAsync(a, a_.p, n_ * 4, cudaMemcpyDeviceToHost, stream_));
        if (sims) CK(cudaMemcpyAsync(sims, sims_.p, n_ * 8, cudaMemcpyDeviceToHost, stream_));
        if (unchanged) CK(cudaMemcpyAsync(unchanged, unchanged_.p, k_, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    void set_state(const uint32_t* a, const double* sims, uint32_t iteration) {
        counts_fresh_ = false;
        need_config();
        if (!state_) {
            reset_sums();
            CK(cudaMemsetAsync(unchanged_.p, 0, k_, stream_));
            CK(cudaMemsetAsync(ct_.p, 0, static_cast<uint64_t>(d_) * ld_ * 4, stream_));
            state_ = true;
        }
        if (a) {
            for (int64_t i = 0; i < n_; ++i)
                if (a[i] >= k_) throw InvalidArgument("assignment out of range");
            CK(cudaMemcpyAsync(a_.p, a, n_ * 4, cudaMemcpyHostToDevice, stream_));
        }
        if (sims) CK(cudaMemcpyAsync(sims_.p, sims, n_ * 8, cudaMemcpyHostToDevice, stream_));
        iteration_ = iteration;
        cache_trusted_ = false;  // externally supplied cache: follow the reference's NCC literally
        ub_valid_ = false;
        CK(cudaStreamSynchronize(stream_));
    }

    void get_centroids(float* ct) {
        need_state();
        CK(cudaMemcpy2DAsync(ct, k_ * sizeof(float), ct_.p, ld_ * sizeof(float), k_ * sizeof(float), d_,
                             cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    // Test hook: rebuilds the single-pass high postings of the current Cᵀ at the
    // kept lists' θ and compares them row by row with the lists maintained in
    // place (as sets of (column, value) pairs, zero pairs ignored; the kept L_t
    // must bound the fresh one). Returns the number of differing rows, or -1 when no
    // maintained lists are held.
    int64_t check_postings() {
        need_state();
        if (!hp_valid_) return -1;
        const uint32_t kt = k_;
        std::vector<uint4> h_old(d_), h_new(d_);
        std::vector<uint2> p_old(pairs_.n);
        CK(cudaMemcpyAsync(h_old.data(), hptr_.p, d_ * sizeof(uint4), cudaMemcpyDeviceToHost, stream_));
        CK(cudaMemcpyAsync(p_old.data(), pairs_.p, pairs_.n * sizeof(uint2), cudaMemcpyDeviceToHost, stream_));
        DevBuf<uint4> h2;
        DevBuf<uint2> p2;
        DevBuf<unsigned long long> c2;
        h2.alloc(d_);
        p2.alloc(pairs_.n * 2 + 1024);
        c2.alloc(2);
        CK(cudaMemsetAsync(c2.p, 0, 16, stream_));
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ceil_div(d_, 8), static_cast<uint64_t>(sms_) * 32));
        launch(hipost_build_kernel, grid, 256, static_cast<const float*>(ct_.p), (uint64_t)ld_, d_, 0u, kt, hp_theta_,
               h2.p, p2.p, static_cast<unsigned long long>(p2.n), c2.p, c2.p + 1, 0);
        CK_LAUNCH();
        std::vector<uint2> p_new(p2.n);
        CK(cudaMemcpyAsync(h_new.data(), h2.p, d_ * sizeof(uint4), cudaMemcpyDeviceToHost, stream_));
        CK(cudaMemcpyAsync(p_new.data(), p2.p, p2.n * sizeof(uint2), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        int64_t bad = 0;
        for (uint32_t t = 0; t < d_; ++t) {
            std::vector<std::pair<uint32_t, uint32_t>> a, b;
            for (uint32_t q = 0; q < h_old[t].y; ++q) {
                const uint2 e = p_old[h_old[t].x + q];
                if (e.x != kNone && e.y != 0u) a.emplace_back(e.x, e.y);  // zero pairs: entries no longer high
            }
            for (uint32_t q = 0; q < h_new[t].y; ++q) b.emplace_back(p_new[h_new[t].x + q].x, p_new[h_new[t].x + q].y);
            std::sort(a.begin(), a.end());
            std::sort(b.begin(), b.end());
            const bool lbound = __builtin_bit_cast(float, h_old[t].z) >= __builtin_bit_cast(float, h_new[t].z);
            if (a != b || !lbound) ++bad;
        }
        return bad;
    }

    // Row / column slices of Cᵀ, gathered on the device in bounded chunks.
    void get_centroid_rows(uint32_t n_rows, const uint32_t* rows, float* out) {
        need_state();
        for (uint32_t r = 0; r < n_rows; ++r)
            if (rows[r] >= d_) throw InvalidArgument("row out of range");
        const uint32_t per = static_cast<uint32_t>(std::max<uint64_t>(1, (uint64_t(64) << 20) / k_));
        DevBuf<uint32_t> dids;
        DevBuf<float> tmp;
        dids.alloc(per);
        tmp.alloc(static_cast<size_t>(per) * k_);
        for (uint32_t r0 = 0; r0 < n_rows; r0 += per) {
            const uint32_t n = std::min(per, n_rows - r0);
            CK(cudaMemcpyAsync(dids.p, rows + r0, n * 4, cudaMemcpyHostToDevice, stream_));
            launch(gather_rows_kernel, grid_for(static_cast<int64_t>(n) * k_, 256), 256, ct_.p, (uint64_t)ld_, k_,
                   dids.p, n, tmp.p);
            CK_LAUNCH();
            CK(cudaMemcpyAsync(out + static_cast<size_t>(r0) * k_, tmp.p, static_cast<size_t>(n) * k_ * 4,
                               cudaMemcpyDeviceToHost, stream_));
            CK(cudaStreamSynchronize(stream_));
        }
    }

    void get_centroid_cols(uint32_t n_cols, const uint32_t* cols, float* out) {
        need_state();
        for (uint32_t c = 0; c < n_cols; ++c)
            if (cols[c] >= k_) throw InvalidArgument("column out of range");
        if (n_cols == 0) return;
        DevBuf<uint32_t> dids;
        DevBuf<float> tmp;
        dids.alloc(n_cols);
        tmp.alloc(static_cast<size_t>(d_) * n_cols);
        CK(cudaMemcpyAsync(dids.p, cols, n_cols * 4, cudaMemcpyHostToDevice, stream_));
        launch(gather_cols_kernel, grid_for(static_cast<int64_t>(d_) * n_cols, 256), 256, ct_.p, (uint64_t)ld_, d_,
               dids.p, n_cols, tmp.p, (uint64_t)n_cols);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(out, tmp.p, static_cast<size_t>(d_) * n_cols * 4, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    // Teacher forcing: replaces Cᵀ; the sums no longer describe it, so they are
    // rebuilt from scratch by the next update.
    void set_centroids(const float* ct) {
        need_config();
        hp_valid_ = false;
        if (!state_) set_state(nullptr, nullptr, iteration_);
        CK(cudaMemsetAsync(ct_.p, 0, static_cast<uint64_t>(d_) * ld_ * 4, stream_));
        CK(cudaMemcpy2DAsync(ct_.p, ld_ * sizeof(float), ct, k_ * sizeof(float), k_ * sizeof(float), d_,
                             cudaMemcpyHostToDevice, stream_));
        std::vector<double> nrm(k_, 0.0);
        for (uint64_t t = 0; t < d_; ++t)
            for (uint32_t j = 0; j < k_; ++j) {
                const double c = ct[t * k_ + j];
                nrm[j] += c * c;
            }
        cmax_ = 1e-300;
        for (double q : nrm) cmax_ = std::max(cmax_, std::sqrt(q) * (1.0 + 1e-12));
        reset_sums();
        have_cc_ = have_ids_ = false;
        cache_trusted_ = false;
        ub_valid_ = false;
        CK(cudaStreamSynchronize(stream_));
    }

    void set_unchanged(const uint8_t* flags) {
        need_state();
        CK(cudaMemcpyAsync(unchanged_.p, flags, k_, cudaMemcpyHostToDevice, stream_));
        have_cc_ = have_ids_ = false;
        cache_trusted_ = false;
        CK(cudaStreamSynchronize(stream_));
    }

    const std::vector<uint32_t>& repaired() const { return repaired_; }
    uint32_t iteration() const { return iteration_; }
    uint32_t k() const { return k_; }
    int64_t n() const { return n_; }
    uint32_t d() const { return d_; }
    const sskm_run_config& config() const { return cfg_; }

    // -------------------------------------------------- multi-GPU pieces --
    void local_counts(int64_t* out) {
        need_state();
        local_counts_device();
        CK(cudaMemcpyAsync(out, counts_.p, k_ * 8, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    void move_doc(int64_t global_doc, uint32_t cluster) {
        counts_fresh_ = false;
        need_state();
        const int64_t i = global_doc - doc_offset_;
        if (i < 0 || i >= n_ || cluster >= k_) throw InvalidArgument("move_doc out of range");
        CK(cudaMemcpyAsync(a_.p + i, &cluster, 4, cudaMemcpyHostToDevice, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    // Locally moved documents (cluster differs from the one their row is
    // summed into), their row lengths and packed-row offsets — on the device.
    void moved_prepare(int64_t* n_moved, int64_t* nnz_moved) {
        need_state();
        reset_scalars();
        launch(moved_kernel, grid_for(n_, 256), 256, a_.p, a_sum_.p, n_, moved_.p, &scal_.p->n_moved);
        mv_len_.alloc(n_ + 1);
        mv_off_.alloc(n_ + 1);
        mv_old_.alloc(n_);
        mv_new_.alloc(n_);
        launch(moved_meta_kernel, grid_for(n_ + 1, 256), 256, moved_.p, &scal_.p->n_moved, indptr_.p, a_.p, a_sum_.p,
               mv_len_.p, mv_old_.p, mv_new_.p);
        CK_LAUNCH();
        pull_scalars();
        mv_n_ = static_cast<int64_t>(hs_->n_moved);
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, mv_len_.p, mv_off_.p, static_cast<int>(mv_n_ + 1), stream_));
        scan_tmp_.alloc(tmp);
        CK(cub::DeviceScan::ExclusiveSum(scan_tmp_.p, tmp, mv_len_.p, mv_off_.p, static_cast<int>(mv_n_ + 1), stream_));
        ++launches_;
        int64_t nnz = 0;
        CK(cudaMemcpyAsync(&nnz, mv_off_.p + mv_n_, 8, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        mv_nnz_ = nnz;
        *n_moved = mv_n_;
        *nnz_moved = nnz;
    }

    // Packs the prepared rows into caller-owned DEVICE buffers.
    void moved_pack(uint32_t* old_c, uint32_t* new_c, int32_t* lens, int32_t* idx, float* val) {
        need_state();
        if (mv_n_ > 0) {
            CK(cudaMemcpyAsync(old_c, mv_old_.p, mv_n_ * 4, cudaMemcpyDeviceToDevice, stream_));
            CK(cudaMemcpyAsync(new_c, mv_new_.p, mv_n_ * 4, cudaMemcpyDeviceToDevice, stream_));
            launch(pack_rows_kernel, grid_for(mv_n_ * 32, 256), 256, moved_.p, mv_n_, indptr_.p, idx_.p, val_.p,
                   mv_off_.p, lens, idx, val);
            CK_LAUNCH();
        }
        CK(cudaStreamSynchronize(stream_));
    }

    // The first m local repair candidates in the reference's donor order
    // (lowest cached sim, then lowest document index): sims, global ids and
    // current clusters (host arrays).
    int64_t local_candidates(int64_t m, double* sims, int64_t* gids, uint32_t* clusters) {
        need_state();
        m = std::min<int64_t>(m, n_);
        sort_sim_candidates();
        std::vector<uint32_t> docs(m), cur(m);
        fetch_candidates(static_cast<uint64_t>(m), docs.data(), cur.data());
        std::vector<double> all(n_);
        CK(cudaMemcpyAsync(all.data(), sims_.p, n_ * 8, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        for (int64_t q = 0; q < m; ++q) {
            sims[q] = all[docs[q]];
            gids[q] = static_cast<int64_t>(docs[q]) + doc_offset_;
            clusters[q] = cur[q];
        }
        return m;
    }

    // Multi-GPU seed init: centroid j = row j of a k-row CSR (host arrays) —
    // the seed documents gathered from whichever shard owns them.
    void init_from_rows(const int64_t* rptr, const int32_t* ridx, const float* rval) {
        counts_fresh_ = false;
        need_config();
        hp_valid_ = false;
        const int64_t nnz = rptr[k_];
        DevBuf<int64_t> dp;
        DevBuf<int32_t> di;
        DevBuf<float> dv;
        dp.alloc(k_ + 1);
        di.alloc(std::max<int64_t>(nnz, 1));
        dv.alloc(std::max<int64_t>(nnz, 1));
        CK(cudaMemcpyAsync(dp.p, rptr, (k_ + 1) * 8, cudaMemcpyHostToDevice, stream_));
        if (nnz) {
            CK(cudaMemcpyAsync(di.p, ridx, nnz * 4, cudaMemcpyHostToDevice, stream_));
            CK(cudaMemcpyAsync(dv.p, rval, nnz * 4, cudaMemcpyHostToDevice, stream_));
        }
        CK(cudaMemsetAsync(ct_.p, 0, static_cast<uint64_t>(d_) * ld_ * sizeof(float), stream_));
        launch(scatter_rows_kernel, grid_for(static_cast<int64_t>(k_) * 32, 256), 256, dp.p, di.p, dv.p, k_, ct_.p,
               (uint64_t)ld_);
        CK_LAUNCH();
        double m = 0.0;
        for (uint32_t j = 0; j < k_; ++j) {
            double q = 0.0;
            for (int64_t e = rptr[j]; e < rptr[j + 1]; ++e) q += static_cast<double>(rval[e]) * rval[e];
            m = std::max(m, std::sqrt(q));
        }
        cmax_ = std::max(m, 1e-300) * (1.0 + 1e-12);
        seed_assign_state();
        sskm_iteration_stats st{};
        full_assign(&st);
        CK(cudaStreamSynchronize(stream_));
    }

    double local_sims_sum() {
        need_state();
        launch(local_sum_kernel, kObjBlocks, 256, sims_.p, n_, obj_part_.p);
        launch(sum_parts_kernel, 1, 256, obj_part_.p, kObjBlocks, &scal_.p->objective);
        CK_LAUNCH();
        pull_scalars();
        return hs_->objective;
    }

private:
    static constexpr int kObjBlocks = 512;

    void need_config() const {
        if (!corpus_) throw InvalidArgument("no corpus uploaded");
        if (k_ == 0) throw InvalidArgument("context not configured");
    }
    void need_state() const {
        need_config();
        if (!state_) throw InvalidArgument("no clustering state: initialise from seeds or k-means++ first");
    }

    unsigned grid_for(int64_t threads, int block) const {
        const int64_t b = (threads + block - 1) / block;
        const int64_t cap = static_cast<int64_t>(sms_) * 32;
        return static_cast<unsigned>(std::max<int64_t>(1, std::min(b, cap)));
    }

    void reset_scalars() {
        CK(cudaMemsetAsync(scal_.p, 0, sizeof(Scalars), stream_));
    }
    void pull_scalars() {
        CK(cudaMemcpyAsync(hs_, scal_.p, sizeof(Scalars), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }
    // The bound screen pulls the scalars with its own counters (one sync); the
    // call right after a screen then has nothing to wait for.
    void pull_scalars_unless_fresh() {
        if (!scalars_fresh_) pull_scalars();
        scalars_fresh_ = false;
    }

    // All per-iteration scratch is sized once here, so no cudaMalloc (and its
    // implicit device synchronisation) ever runs inside an iteration.
    void prealloc() {
        keys_.alloc(2 * n_);
        vals_.alloc(2 * n_);
        order_.alloc(2 * n_);
        keys32_.alloc(n_);
        sb_.alloc(n_);
        ss_.alloc(n_);
        sa_.alloc(n_);
        exact_.alloc(n_);
        pcnt_.alloc(d_ + 1);
        pptr_.alloc(d_ + 1);
        moves_.alloc(2 * static_cast<size_t>(k_));
        // drift bound (skip_kernel)
        ub_.alloc(static_cast<size_t>(n_) * kUbGroups);
        ub_it_.alloc(n_);
        skip_list_.alloc(n_);
        skip_ctr_.alloc(4);
        btake_.alloc(n_);
        bctr_.alloc(8);
        hptr_.alloc(d_);
        hpctr_.alloc(2);
        size_t t1 = 0, t2 = 0, t3 = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, keys_.p, keys_.p + n_, vals_.p, vals_.p + n_,
                                           static_cast<int>(n_), 0, 64, stream_));
        CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, a_.p, keys32_.p, order_.p, order_.p + n_,
                                           static_cast<int>(n_), 0, 32, stream_));
        CK(cub::DeviceScan::ExclusiveSum(nullptr, t3, pcnt_.p, pptr_.p, static_cast<int>(d_ + 1), stream_));
        sort_tmp_.alloc(std::max(t1, t2));
        scan_tmp_.alloc(t3);
        // postings: start at 10% density of a 2048-cluster tile, grow by 1.5x
        // (SSKM_PAIRS_CAP: a smaller start, to exercise the overflow path)
        size_t cap0 = std::max<size_t>(1, static_cast<size_t>(d_) * std::min<uint32_t>(ld_, 2048) / 10);
        if (const char* e = std::getenv("SSKM_PAIRS_CAP")) cap0 = std::max<size_t>(1, std::strtoull(e, nullptr, 10));
        pairs_.alloc(cap0);
    }

    // Bound on the centroid column norms after a seed init (the screen's δ).
    void seed_cmax(const uint32_t* dseeds) {
        reset_scalars();
        launch(seed_norm_max_kernel, grid_for(k_, 128), 128, indptr_.p, val_.p, dseeds, k_,
               &scal_.p->max_drift_bits);
        CK_LAUNCH();
        pull_scalars();
        double m;
        std::memcpy(&m, &hs_->max_drift_bits, 8);
        cmax_ = std::max(m, 1e-300) * (1.0 + 1e-12);
    }

    void seed_assign_state() {
        ub_valid_ = false;
        launch(fill_u32_kernel, grid_for(n_, 256), 256, a_.p, n_, 0);
        launch(fill_f64_kernel, grid_for(n_, 256), 256, sims_.p, n_, -2.0);
        CK_LAUNCH();
        reset_sums();
        CK(cudaMemsetAsync(unchanged_.p, 0, k_, stream_));
        iteration_ = 0;
        dcum_rows_ = 0;
        have_cc_ = have_ids_ = false;
        state_ = true;
    }

    void fill_sum_owner_local() {
        // after a multi-GPU exchange the local rows are summed under their new cluster
        CK(cudaMemcpyAsync(a_sum_.p, a_.p, n_ * 4, cudaMemcpyDeviceToDevice, stream_));
    }

    void launch_counts() {
        if (k_ <= kSmemBins)
            launch(counts_smem_kernel, static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(sms_, ceil_div(n_, 1024)))),
                   1024, a_.p, n_, k_, counts_.p, &scal_.p->bad);
        else
            launch(counts_kernel, grid_for(n_, 256), 256, a_.p, n_, k_, counts_.p, &scal_.p->bad);
    }

    void local_counts_device() {
        CK(cudaMemsetAsync(counts_.p, 0, k_ * 8, stream_));
        reset_scalars();
        launch_counts();
        CK_LAUNCH();
    }

    // Empty-cluster repair for one context (engine.cpp:154-167): ascending
    // empty clusters, each taking the lowest-(sim, index) document among those
    // whose cluster can spare one. One stable radix sort of (sim, doc) keys
    // gives the candidates in the reference's scan order; the sequential rule
    // (sizes shrink as donors leave) is then replayed exactly on the host over
    // the first M candidates, doubling M in the (never observed) case that all
    // of them become ineligible.
    void repair_empty_single() {
        launch(count_empty_kernel, grid_for(k_, 256), 256, counts_.p, k_, &scal_.p->n_empty);
        CK_LAUNCH();
        pull_scalars();
        if (hs_->bad) throw InvalidArgument("assignment out of range");
        CK(cudaMemsetAsync(repaired_flag_.p, 0, k_, stream_));
        const uint32_t n_empty = hs_->n_empty;
        if (n_empty == 0) return;
        std::vector<unsigned long long> counts(k_);
        CK(cudaMemcpyAsync(counts.data(), counts_.p, k_ * 8, cudaMemcpyDeviceToHost, stream_));
        sort_sim_candidates();
        std::vector<uint32_t> moves;  // (doc, cluster) pairs
        std::vector<uint8_t> flag(k_, 0);
        uint64_t m = std::min<uint64_t>(n_, static_cast<uint64_t>(n_empty) * 2 + 256);
        for (;;) {
            std::vector<uint32_t> docs(m), cur(m);
            fetch_candidates(m, docs.data(), cur.data());
            std::vector<unsigned long long> cnt = counts;
            std::vector<uint8_t> used(m, 0);
            std::vector<uint32_t> mv;
            bool ok = true;
            uint64_t pos = 0;  // first candidate not yet used
            for (uint32_t j = 0; j < k_ && ok; ++j) {
                if (cnt[j] != 0) continue;
                uint64_t c = pos;
                while (c < m && (used[c] || cnt[cur[c]] < 2)) ++c;
                if (c == m) {
                    ok = false;
                    break;
                }
                used[c] = 1;
                while (pos < m && used[pos]) ++pos;
                --cnt[cur[c]];
                cur[c] = j;
                cnt[j] = 1;
                mv.push_back(docs[c]);
                mv.push_back(j);
            }
            if (ok) {
                moves.swap(mv);
                break;
            }
            if (m == static_cast<uint64_t>(n_)) throw CudaError("empty-cluster repair found no donor");
            m = std::min<uint64_t>(n_, m * 4);
        }
        for (size_t q = 0; q < moves.size(); q += 2) {
            repaired_.push_back(moves[q + 1]);
            flag[moves[q + 1]] = 1;
        }
        CK(cudaMemcpyAsync(moves_.p, moves.data(), moves.size() * 4, cudaMemcpyHostToDevice, stream_));
        launch(apply_moves_kernel, 1, 256, moves_.p, static_cast<uint32_t>(moves.size() / 2), a_.p);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(repaired_flag_.p, flag.data(), k_, cudaMemcpyHostToDevice, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    void sort_sim_candidates() {
        keys_.alloc(2 * n_);
        vals_.alloc(2 * n_);
        launch(sim_keys_kernel, grid_for(n_, 256), 256, sims_.p, n_, keys_.p, vals_.p);
        CK_LAUNCH();
        size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys_.p, keys_.p + n_, vals_.p, vals_.p + n_,
                                           static_cast<int>(n_), 0, 64, stream_));
        sort_tmp_.alloc(tmp);
        CK(cub::DeviceRadixSort::SortPairs(sort_tmp_.p, tmp, keys_.p, keys_.p + n_, vals_.p, vals_.p + n_,
                                           static_cast<int>(n_), 0, 64, stream_));
        ++launches_;
    }

    // First m candidates in (sim, doc) order and their current clusters.
    void fetch_candidates(uint64_t m, uint32_t* docs, uint32_t* cur) {
        launch(gather_assign_kernel, grid_for(m, 256), 256, vals_.p + n_, static_cast<uint32_t>(m), a_.p,
               vals_.p);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(docs, vals_.p + n_, m * 4, cudaMemcpyDeviceToHost, stream_));
        CK(cudaMemcpyAsync(cur, vals_.p, m * 4, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
    }

    // Renormalise touched columns, drift, unchanged flags, changed list.
    void finish_update(sskm_iteration_stats* st) {
        // touched columns rewritten group by group (bitmap-driven), drift
        // partials reduced in a fixed order, then the NCC flags
        const uint32_t n_rb = static_cast<uint32_t>(ceil_div(d_, kRowBlock));
        const uint32_t n_groups = static_cast<uint32_t>(ceil_div(k_, 32));
        const dim3 wg_grid(static_cast<unsigned>(ceil_div(n_groups, 4)), n_rb);
        const float wg_thr = keep_lists_ && hp_valid_ ? hp_theta_ : 0.f;
#define SSKM_WG_LAUNCH(R)                                                                                         \
    launch(write_groups_kernel<R>, wg_grid, 128, S_.p, ct_.p, (uint64_t)ld_, d_, k_, touched_.p, Q_.p, part_.p, \
           &scal_.p->zero_flag, nz_.p, hptr_.p, pairs_.p, wg_thr, &scal_.p->hp_ovf)
        if (wg_rows_ == 4)
            SSKM_WG_LAUNCH(4);
        else
            SSKM_WG_LAUNCH(2);
#undef SSKM_WG_LAUNCH
        launch(reduce_groups_kernel, static_cast<unsigned>(ceil_div(k_, 32)), 1024, part_.p, n_rb, k_, touched_.p,
               drift_.p, &scal_.p->n_rec);
        launch(flags_kernel, grid_for(k_, 256), 256, k_, iteration_ <= 1 ? 1 : 0, cfg_.ncc_epsilon,
               repaired_flag_.p, drift_.p, unchanged_.p, same_.p, &scal_.p->max_drift_bits,
               &scal_.p->n_unchanged, touched_.p);
        CK_LAUNCH();
        advance_drift_launch();
        ++updates_since_assign_;
        CK(cudaEventRecord(ev_[1], stream_));  // end of the update (timed by the caller)
        pull_scalars();
        const uint32_t n_rec = hs_->n_rec;
        last_n_rec_ = n_rec;
        if (hs_->zero_flag) throw InvalidArgument("cannot normalize zero vector");
        if (hs_->hp_ovf) hp_valid_ = false;
        n_unchanged_ = hs_->n_unchanged;
        // rewritten columns are fp32 roundings of unit vectors: ||c|| <= 1 + 2^-23
        if (n_rec > 0) cmax_ = (n_rec == k_) ? 1.0 + 0x1p-22 : std::max(cmax_, 1.0 + 0x1p-22);
        double max_drift;
        std::memcpy(&max_drift, &hs_->max_drift_bits, 8);
        advance_drift_check(max_drift);
        have_cc_ = have_ids_ = false;
        std::memset(st, 0, sizeof(*st));
        st->iteration = iteration_;
        st->n_unchanged_centroids = n_unchanged_;
        st->max_sq_drift = iteration_ <= 1 ? 0.0 : max_drift;
        st->n_repaired = static_cast<int32_t>(repaired_.size());
        st->n_moved = hs_->n_moved;
        st->n_recomputed = n_rec;
    }

    // Running sums D_g of the updates' max column drift per cluster group (the
    // drift bound's growth, skip_kernel), accumulated on the device from the
    // update's per-column drift; an update the bounds cannot follow (iteration
    // 1, an empty-cluster repair) adds nothing and invalidates them until the
    // next full screen.
    // (Launched behind the update's kernels, ahead of its scalars' round trip;
    // the drift's finiteness is checked on the host afterwards, advance_drift_check.)
    void advance_drift_launch() {
        const bool ok = iteration_ >= 2 && repaired_.empty();
        if (!ok) ub_valid_ = false;
        const size_t rows = static_cast<size_t>(iteration_) + 1;
        if (dcum_.n < rows * kUbGroups) {  // grow, keeping the history (bounds refer to their own iteration's row)
            DevBuf<double> bigger;
            bigger.alloc(std::max<size_t>(4096, 2 * rows) * kUbGroups);
            CK(cudaMemsetAsync(bigger.p, 0, bigger.n * sizeof(double), stream_));
            if (dcum_.n) CK(cudaMemcpyAsync(bigger.p, dcum_.p, dcum_.n * sizeof(double), cudaMemcpyDeviceToDevice, stream_));
            CK(cudaStreamSynchronize(stream_));
            std::swap(dcum_.p, bigger.p);
            std::swap(dcum_.n, bigger.n);
        }
        // rows between the last written one and this one (engines driven through
        // update_apply after a reset) carry the previous sums forward
        for (uint32_t it = dcum_rows_; it < iteration_; ++it)
            launch(group_drift_kernel, 1, 1024, static_cast<const double*>(drift_.p), k_, 0, dcum_.p, it);
        launch(group_drift_kernel, 1, 1024, static_cast<const double*>(drift_.p), k_, ok ? 1 : 0, dcum_.p, iteration_);
        CK_LAUNCH();
        dcum_rows_ = iteration_ + 1;
    }

    void advance_drift_check(double max_sq_drift) {
        if (!(max_sq_drift >= 0.0 && std::isfinite(max_sq_drift))) ub_valid_ = false;
    }

    // The changed-cluster ids and their count; with `cols`, also the compact
    // copy of their columns (only the NCC passes over the changed list read it:
    // the gather reads and writes up to all of Cᵀ, 0.45 ms on c1).
    void ensure_cc(bool cols = true) {
        if (!have_ids_) {
            launch(compact_ids_kernel, 1, 1024, unchanged_.p, k_, 0, chg_ids_.p, &scal_.p->n_chg);
            CK_LAUNCH();
            pull_scalars();
            n_chg_ = hs_->n_chg;
            ld_cc_ = std::max<uint64_t>(128, round_up(n_chg_, 128));
            have_ids_ = true;
        }
        if (cols && !have_cc_) {
            if (n_chg_ > 0) {
                cc_.alloc(static_cast<uint64_t>(d_) * ld_);
                launch(gather_cols_kernel, grid_for(static_cast<int64_t>(d_) * ld_cc_, 256), 256, 
                    ct_.p, ld_, d_, chg_ids_.p, n_chg_, cc_.p, ld_cc_);
                CK_LAUNCH();
            }
            have_cc_ = true;
        }
    }

    void snapshot_start() {
        screen_ms_ = 0.0;
        screen_launches_ = 0;
        bstat_docs_ = bstat_pairs_ = bstat_cand_ = bstat_doc_nnz_ = bstat_cand_nnz_ = bstat_visits_ = bstat_own_ = 0;
        bstat_own_nnz_ = 0;
        bstat_theta_ = 0.0;
        dots_ = 0;
        skip_docs_ = 0;
        skip_ms_ = 0.0;
        second_docs_ = 0;
        second_ms_ = 0.0;
        CK(cudaMemcpyAsync(a_start_.p, a_.p, n_ * 4, cudaMemcpyDeviceToDevice, stream_));
        CK(cudaMemcpyAsync(sims_start_.p, sims_.p, n_ * 8, cudaMemcpyDeviceToDevice, stream_));
    }

    // Documents ordered by their current cluster (stable): consecutive work
    // items of a block then share their cluster's hot Cᵀ rows in L1. Pure
    // scheduling — every document's result is independent of the order.
    const uint32_t* cluster_order() {
        if (!order_enabled_) return nullptr;
        order_.alloc(2 * n_);
        keys32_.alloc(n_);
        launch(iota_kernel, grid_for(n_, 256), 256, order_.p, n_);
        CK_LAUNCH();
        int bits = 1;
        while ((1u << bits) < k_ && bits < 32) ++bits;
        size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, a_.p, keys32_.p, order_.p, order_.p + n_,
                                           static_cast<int>(n_), 0, bits, stream_));
        sort_tmp_.alloc(tmp);
        CK(cub::DeviceRadixSort::SortPairs(sort_tmp_.p, tmp, a_.p, keys32_.p, order_.p, order_.p + n_,
                                           static_cast<int>(n_), 0, bits, stream_));
        ++launches_;
        return order_.p + n_;
    }

    // Column-tile width: the widest of 128 / 64 / 32 whose d × W fp32 slice
    // fits the L2 budget (SSKM_TILE_BYTES, default 64 MiB of the 126 MB L2).
    int tile_v() const {
        const uint64_t budget = tile_bytes_;
        for (int v : {4, 2, 1})
            if (static_cast<uint64_t>(d_) * 32 * v * 4 <= budget) return v;
        return 1;
    }

    template <int INIT>
    void scan_tiles(const float* M, uint64_t ld, uint32_t ncols, const uint32_t* col_ids, const uint32_t* order,
                    int64_t n_work) {
        int v = tile_v();
        while (v > 1 && ncols <= static_cast<uint32_t>(16 * v)) v >>= 1;  // narrow lists: narrow tiles
        const uint32_t W = 32u * v;
        TileArgs p{};
        p.indptr = indptr_.p;
        p.idx = idx_.p;
        p.val = val_.p;
        p.M = M;
        p.ld = ld;
        p.ncols = ncols;
        p.col_ids = col_ids;
        p.order = order;
        p.n_work = n_work;
        p.a = a_.p;
        p.sims = sims_.p;
        p.unchanged = unchanged_.p;
        p.a_start = a_start_.p;
        p.sims_start = sims_start_.p;
        p.CT = ct_.p;
        p.ld_ct = ld_;
        p.rescan_list = rescan_.p;
        p.n_rescan = &scal_.p->n_rescan;
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
            1, std::min<int64_t>(static_cast<int64_t>(sms_) * blocks_per_sm_, ceil_div(n_work, 8))));
        dots_ += static_cast<uint64_t>(n_work) * ncols;  // every (document, column) pair, exact fp64
        // long work lists go tile by tile (the tile's rows stay hot in L2 across
        // the documents); short ones (the screens' leftovers) take every tile in
        // one launch — hundreds of small launches cost more than the locality
        const bool short_list = static_cast<uint64_t>(n_work) <= static_cast<uint64_t>(sms_) * 128;
        if constexpr (INIT != kInitNcc) {
            // short lists: a warp per (document, column span), spans folded after
            const uint32_t tiles = static_cast<uint32_t>(ceil_div(ncols, W));
            if (short_list && tiles > 1) {
                const uint32_t want = static_cast<uint32_t>(
                    std::min<int64_t>(64, std::max<int64_t>(1, ceil_div(static_cast<int64_t>(sms_) * 16, n_work))));
                const uint32_t per = static_cast<uint32_t>(ceil_div(tiles, std::min(tiles, want)));
                const uint32_t n_spans = static_cast<uint32_t>(ceil_div(tiles, per));
                p.span = per * W;
                span_s_.alloc(static_cast<size_t>(n_work) * n_spans);
                span_a_.alloc(static_cast<size_t>(n_work) * n_spans);
                const dim3 g2(static_cast<unsigned>(ceil_div(n_work, 8)), n_spans);
                if (v == 4)
                    assign_span_kernel<4, 16><<<g2, 256, 0, stream_>>>(p, n_spans, span_s_.p, span_a_.p);
                else if (v == 2)
                    assign_span_kernel<2, 16><<<g2, 256, 0, stream_>>>(p, n_spans, span_s_.p, span_a_.p);
                else
                    assign_span_kernel<1, 16><<<g2, 256, 0, stream_>>>(p, n_spans, span_s_.p, span_a_.p);
                ++launches_;
                launch(assign_span_reduce_kernel<INIT>, grid_for(n_work, 256), 256, p, n_spans, span_s_.p, span_a_.p);
                CK_LAUNCH();
                return;
            }
        }
        const uint32_t span = short_list ? ncols : W;
        for (uint32_t c0 = 0; c0 < ncols; c0 += span) {
            p.col0 = c0;
            p.span = span;
            p.first = c0 == 0;
            p.last = c0 + span >= ncols;
            launch_tile<INIT>(v, grid, p);
        }
        CK_LAUNCH();
    }

    // Returns true when the screen also certified (fused resolve).
    // ------------------------------------------------------- bound screen --
    // Exact assignment from the high centroid entries (bound_kernels.cuh).
    void bound_assign(const float* M, uint64_t ld, uint32_t ncols, const uint32_t* col_ids, const uint32_t* order,
                      int64_t n_work, int init) {
        btake_.alloc(n_);
        bctr_.alloc(8);
        // (the drift-bound pass's counters sit right behind the screen's: one memset for both)
        CK(cudaMemsetAsync(bctr_.p, 0, 12 * sizeof(unsigned long long), stream_));
        // more than one 2048-column tile: one pass with hash-table accumulators
        // over every column (SSKM_HASH=0: a pass per tile)
        const bool hash = ncols > 2048 && ncols <= 65534 && hash_enabled_;  // 16-bit table keys (column + 1)
        const uint32_t KT = hash ? ncols : (ncols <= 1024 ? 1024 : 2048);
        // single-pass lists over Cᵀ are kept from pass to pass, maintained in
        // place by the column rewrite; rebuilt (and θ re-tuned) every
        // kRebuildEvery assigns, or when they were invalidated
        const bool lists_here = ncols <= KT && M == ct_.p;
        const bool reuse = keep_lists_ && lists_here && hp_valid_ && assigns_since_build_ + 1 < rebuild_every() &&
                           (theta_adapt_ || theta_ == hp_theta_);
        if (hash && theta_adapt_ && !hash_theta_started_) {  // the first hash pass of this configuration
            for (auto& q : tctl_) q.theta = std::max(q.theta, hash_theta0_);
            hash_theta_started_ = true;
        }
        float thr = reuse ? hp_theta_ : (theta_adapt_ ? tctl_[init].theta : theta_);
        double pass_ms = 0.0, build_ms_inner = 0.0;
        BoundArgs p{};
        p.indptr = indptr_.p;
        p.indptr32 = indptr32_.p;
        p.idx = idx_.p;
        p.val = val_.p;
        p.col_ids = col_ids;
        p.order = order;
        p.n_work = n_work;
        p.CT = ct_.p;
        p.ld_ct = ld_;
        p.xb = xb_.p;
        p.theta = static_cast<double>(thr);
        p.cmax = cmax_;
        p.k = k_;
        p.a = a_.p;
        p.sims = sims_.p;
        p.unchanged = unchanged_.p;
        // the cached similarity of a full-scan document is exact for its
        // cluster when that column is bit-identical to the one the cache was
        // computed against (one update since this engine's last assign)
        p.same = (init == kInitFull && cache_trusted_ && updates_since_assign_ == 1 && iteration_ >= 2) ? same_.p
                                                                                                        : nullptr;
        p.a_start = a_start_.p;
        p.sims_start = sims_start_.p;
        p.take = btake_.p;
        p.exact_list = exact_.p;
        p.n_exact = &scal_.p->n_exact;
        p.n_cand = bctr_.p + 0;
        p.n_pairs = bctr_.p + 1;
        p.n_visits = bctr_.p + 2;
        p.n_own = bctr_.p + 3;
        p.n_doc_nnz = bctr_.p + 4;
        p.n_cand_nnz = bctr_.p + 5;
        p.n_hovf = bctr_.p + 6;
        p.n_own_nnz = bctr_.p + 7;
        // drift bound: single-tile full-scan passes over every document refresh
        // the per-document bounds; with valid bounds, a pre-pass first keeps
        // the documents that provably keep their cluster (skip_kernel)
        const bool full_cover = init == kInitFull && order == nullptr && col_ids == nullptr && n_work == n_;
        bool skipped = false;
        if (full_cover) {
            ub_.alloc(static_cast<size_t>(n_) * kUbGroups);
            ub_it_.alloc(n_);
            p.ub = ub_.p;
            p.ub_it = ub_it_.p;
            p.iter = iteration_;
            if (skip_enabled_ && ub_valid_ && p.same && iteration_ < dcum_rows_) {
                skip_list_.alloc(n_);
                skip_ctr_.alloc(4);  // zeroed with the screen's counters above
                SkipArgs q{};
                q.indptr = indptr_.p;
                q.n = n_;
                q.a = a_.p;
                q.sims = sims_.p;
                q.same = p.same;
                q.ub = ub_.p;
                q.ub_it = ub_it_.p;
                q.dcum = dcum_.p;
                q.iter = iteration_;
                q.xb = xb_.p;
                q.cmax = cmax_;
                q.list = skip_list_.p;
                q.n_list = skip_ctr_.p;
                q.n_kept = skip_ctr_.p + 1;
                CK(cudaEventRecord(ev_[10], stream_));
                launch(skip_kernel, static_cast<unsigned>(ceil_div(n_, kSkipDocsPerBlock)), 256, q);
                CK(cudaEventRecord(ev_[11], stream_));
                CK_LAUNCH();
                p.order = skip_list_.p;
                p.n_work_dev = skip_ctr_.p;
                skipped = true;
            }
        }
        if (col_ids) {  // cluster -> column of M
            bcol_of_.alloc(k_);
            launch(fill_u32_kernel, grid_for(k_, 256), 256, bcol_of_.p, static_cast<int64_t>(k_), kNone);
            launch(scatter_pos_kernel, grid_for(ncols, 256), 256, col_ids, ncols, bcol_of_.p);
            p.col_of = bcol_of_.p;
        }
        for (uint32_t c0 = 0; c0 < ncols; c0 += KT) {
            const uint32_t kt = std::min<uint32_t>(KT, ncols - c0);
            if (c0 > 0) CK(cudaEventRecord(ev_[8], stream_));
            if (reuse) {
                ++assigns_since_build_;
            } else {
                build_hipost(M, ld, c0, kt, thr, ncols > KT || hash, lists_here);  // synchronises (capacity check)
                // hash passes: the tables hold a document's touched clusters, so
                // θ is raised until the expected high pairs per document,
                // Σ_t df_t·|list_t| / N for the lists just built, is within the
                // target (pairs ∝ θ^-1/2 on these corpora; k = 50,000 needs a θ
                // far above the tile screens')
                for (int q = 0; hash && theta_adapt_ && q < 8; ++q) {
                    const double per_doc = expected_pairs_per_doc();
                    const double tgt = tctl_[init].target;
                    if (per_doc <= tgt * 1.4 || thr >= 0.5f) break;
                    thr = std::min(0.5f, static_cast<float>(thr * std::min(2.0, per_doc / tgt)));
                    build_hipost(M, ld, c0, kt, thr, true, lists_here);
                }
                tctl_[init].theta = thr;
                p.theta = static_cast<double>(thr);
            }
            if (c0 > 0) {
                CK(cudaEventRecord(ev_[9], stream_));
                CK(cudaEventSynchronize(ev_[9]));
                float bms = 0.f;
                CK(cudaEventElapsedTime(&bms, ev_[8], ev_[9]));
                build_ms_inner += bms;
            }
            p.hptr = hptr_.p;
            p.pairs = pairs_.p;
            p.c0 = c0;
            p.kt = kt;
            p.first = c0 == 0 ? 1 : 0;
            p.single_tile = ncols <= KT ? 1 : 0;
            p.last = c0 + KT >= ncols ? 1 : 0;
            p.hp_overflow = hpctr_.p + 1;
            // the screen launches are timed as one interval: the event pair
            // brackets every tile's screen, and the postings builds between
            // tiles are timed separately (build_ms) and subtracted
            if (c0 == 0) CK(cudaEventRecord(ev_[6], stream_));
            if (hash)
                bound_launch_hash(p, init);
            else if (KT == 1024)
                bound_launch<1024>(p, init);
            else
                bound_launch<2048>(p, init);
            screen_launches_ += 1;
        }
        CK(cudaEventRecord(ev_[7], stream_));
        if (init == kInitNcc)
            launch(bound_ncc_rescan_kernel, grid_for(n_work, 256), 256, order, n_work, btake_.p, a_start_.p,
                   sims_start_.p, sims_.p, unchanged_.p, rescan_.p, &scal_.p->n_rescan);
        // θ for the next assign: keep the exact-scan share small and the
        // candidate dots near one per document (θ never changes a result)
        // A full-scan pass that left nothing for the exact scan last time: the
        // assign's closing kernels go out now, ahead of the counters' round trip,
        // so the step has one host synchronisation fewer. If this pass does leave
        // documents (the counters say so), the closing kernels simply run again
        // after the exact scan.
        const bool speculate = speculate_finish_ && init == kInitFull && full_cover && !hash;
        if (speculate) {
                finish_assign_launch();
            CK(cudaEventRecord(ev_[3], stream_));
        }
        unsigned long long ctr[8], hp[2], sk[4];
        CK(cudaMemcpyAsync(hblock_, ctr_block_.p, sizeof(CounterBlock), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        std::memcpy(ctr, hblock_->bctr, sizeof(ctr));
        std::memcpy(hp, hblock_->hp, sizeof(hp));
        std::memcpy(sk, hblock_->sk, sizeof(sk));
        if (full_cover) ub_valid_ = true;  // every document: screened (fresh bound) or kept (bound still valid)
        if (skipped) {
            n_work = static_cast<int64_t>(sk[0]);  // the screen's work list
            skip_docs_ += sk[1];
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev_[10], ev_[11]));
            skip_ms_ += ms;
        }
        scalars_fresh_ = true;
        if (hp[0] > pairs_.n) grow_pairs(hp[0]);  // the last tile's lists overflowed: room for the next pass
        if (!reuse) last_hp_overflow_ = hp[1] != 0;
        if (last_hp_overflow_) hp_valid_ = false;
        const uint64_t n_fb = hs_->n_exact;
        finish_speculated_ = speculate && n_fb == 0;
        {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev_[6], ev_[7]));
            pass_ms = static_cast<double>(ms) - build_ms_inner;
            screen_ms_ += pass_ms;
        }
        uint64_t n_fb2 = n_fb;  // documents left for the exact scan
        if (hash && init == kInitFull && lists_here && second_pass_ && n_fb >= second_pass_min_)
            n_fb2 = bound_second_pass(p, thr, n_fb);
        const uint64_t n_list = n_work > 0 ? static_cast<uint64_t>(n_work) - std::min<uint64_t>(n_fb2, n_work) : 0;
        bstat_docs_ += n_list;
        bstat_pairs_ += ctr[1];
        dots_ += ctr[0] + ctr[3];  // exact fp64 dots: candidates and own-cluster dots
        bstat_cand_ += ctr[0];
        bstat_visits_ += ctr[2];
        bstat_own_ += ctr[3];
        bstat_own_nnz_ += ctr[7];
        bstat_doc_nnz_ += ctr[4];
        bstat_cand_nnz_ += ctr[5];
        bstat_theta_ = static_cast<double>(thr);
        if (debug_)
            std::fprintf(stderr,
                         "[sskm] bound init=%d theta=%.5g work=%lld exact=%llu cand=%llu pairs=%llu own=%llu "
                         "cache=%d\n",
                         init, static_cast<double>(thr), static_cast<long long>(n_work),
                         static_cast<unsigned long long>(n_fb), static_cast<unsigned long long>(ctr[0]),
                         static_cast<unsigned long long>(ctr[1]), static_cast<unsigned long long>(ctr[3]),
                         p.same != nullptr);
        // θ for the next pass of this kind: hill-climb the measured screen time
        // per work item (θ trades high pairs against candidate dots, and the
        // balance differs per corpus); back off when documents fall through to
        // the exact scan. θ never changes a result.
        // θ follows the failures, per period of kRebuildEvery passes (θ only
        // changes at a rebuild): lower (tighter low-part bounds) when documents
        // fall through to the exact scan; in hash passes, a lower pairs target
        // when tables overflow. Otherwise θ stays: on these corpora the step
        // time is flat over a wide θ range once the lists are kept (measured,
        // DESIGN.md §3.1), and comparing costs across converging iterations
        // misleads a hill climb.
        if (theta_adapt_ && n_work > 0) {
            ThetaCtl& c = tctl_[init];
            c.acc_fb += static_cast<double>(n_fb - std::min<uint64_t>(n_fb, ctr[6]));
            c.acc_hovf += static_cast<double>(ctr[6]);
            c.acc_work += static_cast<double>(n_work);
            if (!lists_here || ++c.passes >= rebuild_every()) {
                // (a second pass makes a fallen-through document ~5 screens dear instead
                // of an exact scan over every column: more of them are tolerated)
                const bool sp = hash && init == kInitFull && second_pass_;
                if (c.acc_hovf > (sp ? 3e-3 : 1e-4) * c.acc_work) {
                    c.target *= 0.7;
                    c.theta *= 1.3f;
                } else if (c.acc_fb > (sp ? 2e-2 : 2e-3) * c.acc_work) {
                    c.target *= 1.4;
                    c.theta *= 0.7f;
                }
                c.target = std::min(1024.0, std::max(8.0, c.target));
                c.theta = std::min(0.5f, std::max(1e-5f, c.theta));
                c.acc_fb = c.acc_work = c.acc_hovf = 0.0;
                c.passes = 0;
            }
        }
    }

    static constexpr int kHashSlots = 1024;  // per-warp hash accumulators (4 KB keys + 4 KB sums)

    // Σ_t df_t · (high-list length of t) / N for the lists just built: the high
    // pairs an average document accumulates. df_ (document frequencies) once.
    double expected_pairs_per_doc() {
        if (!df_ready_) {
            df_.alloc(d_);
            CK(cudaMemsetAsync(df_.p, 0, d_ * sizeof(uint32_t), stream_));
            launch(doc_freq_kernel, grid_for(nnz_, 256), 256, idx_.p, nnz_, df_.p);
            CK_LAUNCH();
            df_ready_ = true;
        }
        CK(cudaMemsetAsync(&scal_.p->n_moved, 0, 8, stream_));
        launch(pairs_expect_kernel, grid_for(d_, 256), 256, hptr_.p, df_.p, d_, &scal_.p->n_moved);
        CK_LAUNCH();
        unsigned long long tot = 0;
        CK(cudaMemcpyAsync(&tot, &scal_.p->n_moved, 8, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        return static_cast<double>(tot) / static_cast<double>(std::max<int64_t>(1, n_));
    }

    // Second pass of a hash-accumulator screen (configs 2 and 4). Documents the
    // first pass could not settle — own similarity below the bound on the
    // clusters they share no high entry with (Σ|x_t|·L_t is loose at the large θ
    // that keeps k = 50,000 clusters' pairs within the tables), or a full table —
    // used to take the exact scan over every column (c4: ~80k documents, half the
    // iteration). They are screened again against lists at a much lower θ
    // (tighter low-part bounds, ~4× the pairs) with 4096-slot tables; only what
    // that leaves goes to the exact scan. The second lists are rebuilt per pass
    // in their own buffers (one read of Cᵀ); the kept first-pass lists stay.
    uint64_t bound_second_pass(const BoundArgs& p1, float thr1, uint64_t n_fb) {
        constexpr int HT2 = 4096;
        const float thr2 = std::max(1e-5f, thr1 * second_pass_ratio_);
        exact2_.alloc(n_);
        CK(cudaMemcpyAsync(exact2_.p, exact_.p, n_fb * sizeof(uint32_t), cudaMemcpyDeviceToDevice, stream_));
        CK(cudaMemsetAsync(&scal_.p->n_exact, 0, 8, stream_));
        CK(cudaMemsetAsync(bctr_.p, 0, 8 * sizeof(unsigned long long), stream_));
        hptr2_.alloc(d_);
        hpctr2_.alloc(2);
        if (pairs2_.n == 0) pairs2_.alloc(std::max<size_t>(pairs_.n, 1u << 20));
        CK(cudaMemsetAsync(hpctr2_.p, 0, 2 * sizeof(unsigned long long), stream_));
        CK(cudaEventRecord(ev_[8], stream_));
        const unsigned grid_b = static_cast<unsigned>(std::min<uint64_t>(ceil_div(d_, 8), static_cast<uint64_t>(sms_) * 32));
        launch(hipost_build_kernel, grid_b, 256, static_cast<const float*>(ct_.p), static_cast<uint64_t>(ld_), d_, 0u, k_,
               thr2, hptr2_.p, pairs2_.p, std::min<unsigned long long>(pairs2_.n, 0xFFFFFFFFull), hpctr2_.p,
               hpctr2_.p + 1, 0);
        CK_LAUNCH();
        BoundArgs p = p1;
        p.order = exact2_.p;
        p.n_work = static_cast<int64_t>(n_fb);
        p.n_work_dev = nullptr;
        p.hptr = hptr2_.p;
        p.pairs = pairs2_.p;
        p.theta = static_cast<double>(thr2);
        p.hp_overflow = hpctr2_.p + 1;
        p.first = 1;
        p.single_tile = 1;
        p.last = 1;
        CK(cudaEventRecord(ev_[6], stream_));
        bound_launch_k(bound_screen_kernel<2048, kInitFull, HT2>, BoundSmem<2048, HT2>::per_warp, p);
        CK(cudaEventRecord(ev_[7], stream_));
        screen_launches_ += 1;
        unsigned long long ctr[8] = {0, 0, 0, 0, 0, 0, 0, 0}, hp[2] = {0, 0};
        CK(cudaMemcpyAsync(ctr, bctr_.p, sizeof(ctr), cudaMemcpyDeviceToHost, stream_));
        CK(cudaMemcpyAsync(hp, hpctr2_.p, sizeof(hp), cudaMemcpyDeviceToHost, stream_));
        CK(cudaMemcpyAsync(hs_, scal_.p, sizeof(Scalars), cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        if (hp[0] > pairs2_.n) pairs2_.alloc(static_cast<size_t>(std::min<unsigned long long>(hp[0], 0xFFFFFFFFull)) * 5 / 4 + 1);
        float ms = 0.f, bms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_[6], ev_[7]));
        CK(cudaEventElapsedTime(&bms, ev_[8], ev_[6]));
        screen_ms_ += ms;
        second_ms_ += ms + bms;
        second_docs_ += n_fb;
        bstat_pairs_ += ctr[1];
        dots_ += ctr[0] + ctr[3];
        bstat_cand_ += ctr[0];
        bstat_visits_ += ctr[2];
        bstat_own_ += ctr[3];
        bstat_own_nnz_ += ctr[7];
        bstat_doc_nnz_ += ctr[4];
        bstat_cand_nnz_ += ctr[5];
        if (debug_)
            std::fprintf(stderr,
                         "[sskm] bound second pass theta=%.5g work=%llu exact=%llu cand=%llu pairs=%llu hovf=%llu "
                         "lists=%llu pairs (cap %zu, dropped=%llu) build %.2f ms screen %.2f ms\n",
                         static_cast<double>(thr2), static_cast<unsigned long long>(n_fb),
                         static_cast<unsigned long long>(hs_->n_exact), ctr[0], ctr[1], ctr[6], hp[0], pairs2_.n, hp[1],
                         static_cast<double>(bms), static_cast<double>(ms));
        return hs_->n_exact;
    }

    void bound_launch_hash(const BoundArgs& p, int init) {
        using SM = BoundSmem<2048, kHashSlots>;
        if (init == kInitFull)
            bound_launch_k(bound_screen_kernel<2048, kInitFull, kHashSlots>, SM::per_warp, p);
        else if (init == kInitNcc)
            bound_launch_k(bound_screen_kernel<2048, kInitNcc, kHashSlots>, SM::per_warp, p);
        else
            bound_launch_k(bound_screen_kernel<2048, kInitRescan, kHashSlots>, SM::per_warp, p);
    }

    template <int KT>
    void bound_launch(const BoundArgs& p, int init) {
        if (init == kInitFull)
            bound_launch_k(bound_screen_kernel<KT, kInitFull>, BoundSmem<KT>::per_warp, p);
        else if (init == kInitNcc)
            bound_launch_k(bound_screen_kernel<KT, kInitNcc>, BoundSmem<KT>::per_warp, p);
        else
            bound_launch_k(bound_screen_kernel<KT, kInitRescan>, BoundSmem<KT>::per_warp, p);
    }

    template <typename K>
    void bound_launch_k(K k, size_t per_warp, const BoundArgs& p) {
        // warps per block: the most resident warps per SM (shared memory bounds
        // the 2048-cluster tiles, registers the 1024-cluster ones); chosen once
        // per kernel
        const void* key = reinterpret_cast<const void*>(k);
        auto it = launch_cfg_.find(key);
        if (it == launch_cfg_.end()) it = launch_cfg_.emplace(key, pick_bound_cfg(k, per_warp)).first;
        const int warps = it->second.first, per_sm = it->second.second;
        const size_t smem = static_cast<size_t>(warps) * per_warp;
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
            1, std::min<int64_t>(static_cast<int64_t>(sms_) * per_sm, ceil_div(p.n_work, warps))));
        k<<<grid, warps * 32, smem, stream_>>>(p);
        ++launches_;
        CK_LAUNCH();
    }

    template <typename K>
    std::pair<int, int> pick_bound_cfg(K k, size_t per_warp) {
        int warps = 1, per_sm = 1, best = 0;
        // the attribute is per device and function, and engines of a
        // multi-device context (several may share a device) pick their
        // configurations concurrently: it is only ever raised to one common
        // ceiling, never lowered under another engine's launch
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(200u << 10)));
        for (int w : {8, 4, 2}) {
            const size_t sm = static_cast<size_t>(w) * per_warp;
            if (sm > (200u << 10)) continue;
            int b = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, w * 32, sm));
            if (b * w > best) {
                best = b * w;
                warps = w;
                per_sm = std::max(1, b);
            }
        }
        const size_t smem = static_cast<size_t>(warps) * per_warp;
        if (debug_)
            std::fprintf(stderr, "[sskm] bound launch: %d warps/block, %d blocks/SM, %zu B smem/block\n", warps, per_sm,
                         smem);
        return {warps, per_sm};
    }

    // High postings (|value| >= thr) of the columns [c0, c0 + kt) of M into
    // hptr_ / pairs_ in one pass over M; grows the pair buffer and rebuilds
    // when the previous capacity was exceeded.
    // High postings of the tile [c0, c0 + kt) of M. With `check`, wait for the
    // pair count and rebuild in a grown buffer when it overflowed (multi-tile
    // passes, whose first tile bounds the later tiles' clusters by θ·‖x‖₁);
    // without, an overflow only loosens the bound (the dropped lists' weights
    // are covered by L_t) and the host grows the buffer after the pass.
    // `slack`: the single-tile lists over Cᵀ, built with room to be maintained
    // in place by the column rewrite until the next rebuild.
    void build_hipost(const float* M, uint64_t ld, uint32_t c0, uint32_t kt, float thr, bool check,
                      bool slack = false) {
        hptr_.alloc(d_);
        hpctr_.alloc(2);
        hp_valid_ = false;
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ceil_div(d_, 8), static_cast<uint64_t>(sms_) * 32));
        for (int attempt = 0; attempt < 2; ++attempt) {
            CK(cudaMemsetAsync(hpctr_.p, 0, 2 * sizeof(unsigned long long), stream_));
            // the screen addresses pairs with 32-bit offsets: lists past 2^32 are
            // dropped (exact, looser bound) rather than truncated
            launch(hipost_build_kernel, grid, 256, M, ld, d_, c0, kt, thr, hptr_.p, pairs_.p,
                   std::min<unsigned long long>(pairs_.n, 0xFFFFFFFFull), hpctr_.p, hpctr_.p + 1, slack ? 1 : 0);
            CK_LAUNCH();
            if (slack) {
                hp_valid_ = true;  // withdrawn after the pass if a list was dropped
                hp_theta_ = thr;
                assigns_since_build_ = 0;
            }
            if (!check) return;
            unsigned long long total = 0;
            CK(cudaMemcpyAsync(&total, hpctr_.p, 8, cudaMemcpyDeviceToHost, stream_));
            CK(cudaStreamSynchronize(stream_));
            if (total <= pairs_.n) return;
            grow_pairs(total);
        }
    }

    void grow_pairs(unsigned long long total) {
        if (total >= (1ull << 32)) throw std::runtime_error("bound screen: high postings exceed 2^32 pairs");
        hp_valid_ = false;
        pairs_.alloc(static_cast<size_t>(total) * 3 / 2 + 1);
    }

    bool bound_active() const { return screen_enabled_ && bound_enabled_ && bound_ok_ && iteration_ >= 1; }

    bool screen_any(const float* M, uint64_t ld, uint32_t ncols, const uint32_t* col_ids, const uint32_t* skip,
                    const uint32_t* order, int64_t n_work, int init) {
        // the bound screen needs a real assignment to start from: not the
        // seed assignment (iteration 0), whose state is all cluster 0
        if (bound_active()) {
            bound_assign(M, ld, ncols, col_ids, order, n_work, init);
            return true;  // candidates resolved exactly in the kernel; the exact list holds the rest
        }
        // postings move 8 B per nonzero centroid weight at ~4 TB/s, the dense
        // screen 4 B per weight mostly from L2 at ~12 TB/s: above ~15% density
        // (long documents, few clusters: c3) the dense screen wins (measured)
        if (screen_kind_ == 2 && last_density_ > dense_above_ && (++dense_assigns_ % 5) == 0) {
            // re-measure the density every few dense assigns (one count pass over tile 0)
            const uint32_t kt = std::min<uint32_t>(ncols, 2048);
            CK(cudaMemsetAsync(pcnt_.p + d_, 0, 4, stream_));
            launch(postings_count_kernel, grid_for(static_cast<int64_t>(d_) * 32, 256), 256, M, ld, d_, 0u, kt,
                   pcnt_.p, 0.f);
            size_t tmp = scan_tmp_.n;
            CK(cub::DeviceScan::ExclusiveSum(scan_tmp_.p, tmp, pcnt_.p, pptr_.p, static_cast<int>(d_ + 1), stream_));
            uint32_t total = 0;
            CK(cudaMemcpyAsync(&total, pptr_.p + d_, 4, cudaMemcpyDeviceToHost, stream_));
            CK(cudaStreamSynchronize(stream_));
            last_density_ = static_cast<double>(total) / (static_cast<double>(d_) * kt);
        }
        const bool use_postings = screen_kind_ == 1 || (screen_kind_ == 2 && last_density_ <= dense_above_);
        if (use_postings) {
            postings_screen(M, ld, ncols, col_ids, skip, order, n_work, fuse_resolve_ ? init : -1);
            return fuse_resolve_;
        }
        screen_tiles(M, ld, ncols, col_ids, skip, order, n_work);
        return false;
    }

    // Inverted-index screen, one cluster tile at a time: build the tile's
    // postings from the dense columns, then run the warp-per-document screen.
    // Postings of the columns [c0, c0 + kt) of M into pptr_ / pairs_: per-term
    // counts, exclusive scan, bank-interleaved fill. Returns the pair count.
    uint32_t build_postings(const float* M, uint64_t ld, uint32_t c0, uint32_t kt, float thr = 0.f) {
        hp_valid_ = false;  // the pair buffer is shared with the high postings
        pcnt_.alloc(d_ + 1);
        pptr_.alloc(d_ + 1);
        CK(cudaMemsetAsync(pcnt_.p + d_, 0, 4, stream_));
        launch(postings_count_kernel, grid_for(static_cast<int64_t>(d_) * 32, 256), 256, M, ld, d_, c0, kt, pcnt_.p,
               thr);
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, pcnt_.p, pptr_.p, static_cast<int>(d_ + 1), stream_));
        scan_tmp_.alloc(tmp);
        CK(cub::DeviceScan::ExclusiveSum(scan_tmp_.p, tmp, pcnt_.p, pptr_.p, static_cast<int>(d_ + 1), stream_));
        ++launches_;
        uint32_t total = 0;
        CK(cudaMemcpyAsync(&total, pptr_.p + d_, 4, cudaMemcpyDeviceToHost, stream_));
        CK(cudaStreamSynchronize(stream_));
        if (total > pairs_.n) pairs_.alloc(static_cast<size_t>(total) * 3 / 2 + 1);
        launch(postings_fill_kernel, grid_for(static_cast<int64_t>(d_) * 32, 256), 256, M, ld, d_, c0, kt, pptr_.p,
               pairs_.p, thr);
        return total;
    }

    void postings_screen(const float* M, uint64_t ld, uint32_t ncols, const uint32_t* col_ids, const uint32_t* skip,
                         const uint32_t* order, int64_t n_work, int fuse) {
        dots_ += static_cast<uint64_t>(n_work) * (ncols + 1);  // fp32 screen dots + the certified exact one
        sb_.alloc(n_);
        ss_.alloc(n_);
        sa_.alloc(n_);
        pcnt_.alloc(d_ + 1);
        pptr_.alloc(d_ + 1);
        // tile pairs are addressed with 32-bit offsets: d · KT < 2^32
        const uint32_t KT = post_tile_width(ncols);
        if (static_cast<uint64_t>(d_) * KT >= (1ull << 32)) throw InvalidArgument("vocabulary too large for postings");
        PostingsArgs p{};
        p.indptr = indptr_.p;
        p.idx = idx_.p;
        p.val = val_.p;
        p.col_ids = col_ids;
        p.order = order;
        p.n_work = n_work;
        p.skip_id = skip;
        p.sb = sb_.p;
        p.ss = ss_.p;
        p.sa = sa_.p;
        p.r = resolve_args(order, n_work);
        for (uint32_t c0 = 0; c0 < ncols; c0 += KT) {
            const uint32_t kt = std::min<uint32_t>(KT, ncols - c0);
            const uint32_t total = build_postings(M, ld, c0, kt);
            p.pptr = pptr_.p;
            p.pairs = pairs_.p;
            if (c0 == 0) last_density_ = static_cast<double>(total) / (static_cast<double>(d_) * kt);
            p.c0 = c0;
            p.kt = kt;
            p.first = c0 == 0;
            postings_total_ += total;
            CK(cudaEventRecord(ev_[6], stream_));
            const int f = c0 + KT >= ncols ? fuse : -1;
            if (KT == 256)
                postings_launch<256>(p, n_work, f);
            else if (KT == 512)
                postings_launch<512>(p, n_work, f);
            else if (KT == 1024)
                postings_launch<1024>(p, n_work, f);
            else
                postings_launch<2048>(p, n_work, f);
            CK(cudaEventRecord(ev_[7], stream_));
            CK(cudaEventSynchronize(ev_[7]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ev_[6], ev_[7]));
            screen_ms_ += ms;
            screen_launches_ += 1;
        }
        CK_LAUNCH();
    }

    // Σ over document nonzeros of the posting-list length of their term, for
    // the last built tile set: the (cluster, value) pairs the screen streams.
public:
    uint64_t postings_work() {
        need_state();
        reset_scalars();
        uint64_t total = 0;
        const uint32_t KT = post_tile_width(k_);
        for (uint32_t c0 = 0; c0 < k_; c0 += KT) {
            const uint32_t kt = std::min<uint32_t>(KT, k_ - c0);
            CK(cudaMemsetAsync(pcnt_.p + d_, 0, 4, stream_));
            launch(postings_count_kernel, grid_for(static_cast<int64_t>(d_) * 32, 256), 256, ct_.p, (uint64_t)ld_, d_,
                   c0, kt, pcnt_.p, 0.f);
            CK(cudaMemsetAsync(&scal_.p->n_moved, 0, 8, stream_));
            launch(postings_work_kernel, grid_for(nnz_, 256), 256, idx_.p, nnz_, pcnt_.p, &scal_.p->n_moved);
            CK_LAUNCH();
            pull_scalars();
            total += hs_->n_moved;
        }
        return total;
    }

private:
    // Cluster-tile width of the postings screen: the per-warp accumulator is
    // KT floats of shared memory, so narrower tiles buy occupancy (the screen
    // is latency-bound) at the price of one more CSR pass per tile.
    uint32_t post_tile_width(uint32_t ncols) const {
        if (ncols <= 256) return 256;
        if (ncols <= 512 || post_kt_max_ <= 512) return 512;
        if (ncols <= 1024 || post_kt_max_ <= 1024) return 1024;
        return 2048;
    }

    template <int KT>
    void postings_launch(const PostingsArgs& p, int64_t n_work, int fuse) {
        if (fuse == kInitFull)
            postings_launch_s<KT, 32, kInitFull>(p, n_work);
        else if (fuse == kInitNcc)
            postings_launch_s<KT, 32, kInitNcc>(p, n_work);
        else if (fuse == kInitRescan)
            postings_launch_s<KT, 32, kInitRescan>(p, n_work);
        else
            postings_launch_s<KT, 32, -1>(p, n_work);  // split-warp lists (SUB < 32) measured slower: not built
    }

    template <int KT, int SUB, int FUSE>
    void postings_launch_s(const PostingsArgs& p, int64_t n_work) {
        auto k = postings_screen_kernel<KT, SUB, FUSE>;
        const size_t per_warp = static_cast<size_t>(32 / SUB) * KT * sizeof(float);
        const int warps = static_cast<int>(std::max<size_t>(1, std::min<size_t>(post_warps_, (200u << 10) / per_warp)));
        const size_t smem = static_cast<size_t>(warps) * per_warp;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, warps * 32, smem));
        per_sm = std::max(1, per_sm);
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
            1, std::min<int64_t>(static_cast<int64_t>(sms_) * per_sm, ceil_div(n_work, warps))));
        k<<<grid, warps * 32, smem, stream_>>>(p);
        ++launches_;
    }

    void screen_tiles(const float* M, uint64_t ld, uint32_t ncols, const uint32_t* col_ids, const uint32_t* skip,
                      const uint32_t* order, int64_t n_work) {
        dots_ += static_cast<uint64_t>(n_work) * (ncols + 1);  // fp32 screen dots + the certified exact one
        sb_.alloc(n_);
        ss_.alloc(n_);
        sa_.alloc(n_);
        int v = tile_v();
        while (v > 1 && ncols <= static_cast<uint32_t>(16 * v)) v >>= 1;
        const uint32_t W = 32u * v;
        ScreenArgs p{};
        p.indptr = indptr_.p;
        p.idx = idx_.p;
        p.val = val_.p;
        p.M = M;
        p.ld = ld;
        p.ncols = ncols;
        p.col_ids = col_ids;
        p.order = order;
        p.n_work = n_work;
        p.skip_id = skip;
        p.sb = sb_.p;
        p.ss = ss_.p;
        p.sa = sa_.p;
        for (uint32_t c0 = 0; c0 < ncols; c0 += W) {
            p.col0 = c0;
            p.first = c0 == 0;
            if (v == 4)
                screen_launch<4>(p, n_work);
            else if (v == 2)
                screen_launch<2>(p, n_work);
            else
                screen_launch<1>(p, n_work);
        }
        CK_LAUNCH();
    }

    // One resident wave: blocks = SMs × occupancy, each a contiguous chunk of
    // the cluster-ordered work list.
    template <class K>
    unsigned resident_grid(K kernel, int64_t n_work) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
        per_sm = std::max(1, std::min(per_sm, screen_blocks_per_sm_));
        return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(sms_) * per_sm,
                                                                            ceil_div(n_work, 8))));
    }

    template <int V>
    void screen_launch(const ScreenArgs& p, int64_t n_work) {
        auto k = screen_tile_kernel<V, 16>;
        launch(k, resident_grid(k, n_work), 256, p);
    }

    ResolveArgs resolve_args(const uint32_t* order, int64_t n_work) {
        ResolveArgs r{};
        r.indptr = indptr_.p;
        r.idx = idx_.p;
        r.val = val_.p;
        r.CT = ct_.p;
        r.ld_ct = ld_;
        r.order = order;
        r.n_work = n_work;
        r.cmax = cmax_;
        r.xnorm2 = xnorm2_.p;
        r.nonneg = nonneg_ ? 1 : 0;
        r.sb = sb_.p;
        r.ss = ss_.p;
        r.sa = sa_.p;
        r.unchanged = unchanged_.p;
        r.a_start = a_start_.p;
        r.sims_start = sims_start_.p;
        r.a = a_.p;
        r.sims = sims_.p;
        r.exact_list = exact_.p;
        r.n_exact = &scal_.p->n_exact;
        r.rescan_list = rescan_.p;
        r.n_rescan = &scal_.p->n_rescan;
        return r;
    }

    template <int INIT>
    void resolve(const uint32_t* order, int64_t n_work) {
        launch(resolve_kernel<INIT>, grid_for(n_work * 32, 256), 256, resolve_args(order, n_work));
        CK_LAUNCH();
    }

    template <int INIT, int U>
    void launch_tile_u(int v, unsigned grid, const TileArgs& p) {
        if (v == 4)
            launch(assign_tile_kernel<4, INIT, U>, grid, 256, p);
        else if (v == 2)
            launch(assign_tile_kernel<2, INIT, U>, grid, 256, p);
        else
            launch(assign_tile_kernel<1, INIT, U>, grid, 256, p);
    }

    template <int INIT>
    void launch_tile(int v, unsigned grid, const TileArgs& p) {
        launch_tile_u<INIT, 16>(v, grid, p);
    }

    // The assign's closing kernels: reassignment count and objective, then the
    // cluster sizes of the new assignment, so that the next update's empty-
    // cluster check needs no round trip of its own (engine.cpp:154).
    void finish_assign_launch() {
        // (one kernel zeroes the cluster sizes and the four scalars these kernels
        // add into: five memsets' worth of launches less on the host's path)
        launch(zero_closing_kernel, grid_for(k_, 256), 256, counts_.p, k_, scal_.p);
        launch(finish_assign_kernel, kObjBlocks, 256, a_.p, a_start_.p, sims_.p, n_, obj_part_.p,
                                                              &scal_.p->reassigned);
        launch(sum_parts_kernel, 1, 256, obj_part_.p, kObjBlocks, &scal_.p->objective);
        launch_counts();
        launch(count_empty_kernel, grid_for(k_, 256), 256, counts_.p, k_, &scal_.p->n_empty);
        CK_LAUNCH();
    }

    void finish_assign(sskm_iteration_stats* st) {
        if (!finish_speculated_) {
            finish_assign_launch();
            CK(cudaEventRecord(ev_[3], stream_));
            pull_scalars();
        }
        finish_speculated_ = false;
        st->n_reassigned = hs_->reassigned;
        st->objective = hs_->objective;
        updates_since_assign_ = 0;
        counts_fresh_ = hs_->n_empty == 0 && hs_->bad == 0;  // anything else takes the update's own check
    }

    void reset_scalars_keep_rescan() {
        CK(cudaMemsetAsync(&scal_.p->reassigned, 0, 8, stream_));
        CK(cudaMemsetAsync(&scal_.p->objective, 0, 8, stream_));
    }

    void timing(sskm_iteration_stats* st) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
        st->assign_ms = ms;
        st->assign_kernel_ms = ms;  // (its own event pair was two launches on the host's path: folded into assign_ms)
        st->screen_ms = screen_ms_;
        st->screen_launches = screen_launches_;
        st->centroid_density = last_density_;
        st->bound_docs = bstat_docs_;
        st->bound_pairs = bstat_pairs_;
        st->bound_candidates = bstat_cand_;
        st->bound_doc_nnz = bstat_doc_nnz_;
        st->bound_cand_nnz = bstat_cand_nnz_;
        st->bound_theta = bstat_theta_;
        st->bound_visits = bstat_visits_;
        st->bound_own_dots = bstat_own_;
        st->bound_own_nnz = bstat_own_nnz_;
        st->skip_docs = skip_docs_;
        st->second_pass_docs = static_cast<uint32_t>(std::min<uint64_t>(second_docs_, 0xFFFFFFFFull));
        st->skip_ms = skip_ms_;
    }

    int device_;
    int sms_ = 148;
    cudaStream_t stream_{};
    cudaEvent_t ev_[12]{};
    static constexpr int kUserEvents = 256;
    cudaEvent_t user_ev_[kUserEvents]{};
    uint64_t launches_ = 0;
    uint64_t tile_bytes_ = 64ull << 20;
    bool order_enabled_ = true;
    int blocks_per_sm_ = 2;
    int screen_blocks_per_sm_ = 8;
    bool screen_enabled_ = true;
    double cmax_ = 1.0;
    DevBuf<CounterBlock> ctr_block_;
    CounterBlock* hblock_ = nullptr;
    DevBuf<Scalars> scal_;  // window of ctr_block_ (as bctr_, hpctr_, skip_ctr_)
    Scalars* hs_ = nullptr;

    bool corpus_ = false, state_ = false, have_cc_ = false, have_ids_ = false;
    int64_t n_ = 0, n_total_ = 0, doc_offset_ = 0, nnz_ = 0;
    uint32_t d_ = 0, k_ = 0, ld_ = 0;
    int K_ = 0;
    uint32_t iteration_ = 0, n_unchanged_ = 0, n_chg_ = 0;
    uint64_t ld_cc_ = 128;
    sskm_run_config cfg_{};
    std::vector<double> lambdas_;
    std::vector<uint32_t> repaired_;

    DevBuf<int64_t> indptr_;
    DevBuf<int32_t> idx_;
    DevBuf<float> val_;
    DevBuf<float2> xb_;
    DevBuf<uint32_t> indptr32_;
    bool bound_ok_ = false;  // nnz < 2^32 on this device
    DevBuf<uint8_t> btake_, same_;
    DevBuf<uint32_t> bcol_of_;
    DevBuf<uint4> hptr_;
    DevBuf<unsigned long long> bctr_, hpctr_;
    // ncc+index accounting (index_account)
    DevBuf<uint32_t> ix_cnt_, ix_mval_, ix_jlen_, ix_lcnt_, ix_lptr_, ix_fill_, ix_list_;
    DevBuf<uint64_t> ix_off_, ix_cptr_, ix_keys_;
    DevBuf<unsigned long long> ix_ctr_;
    DevBuf<double> ix_lam_;
    DevBuf<uint8_t> ix_sel_, ix_rescan_;
    DevBuf<uint2> ix_lent_;
    DevBuf<char> ix_tmp_;
    bool last_full_equiv_ = false;
    uint64_t last_n_rescan_ = 0;
    DevBuf<float> ct_, cc_;
    DevBuf<long long> S_;
    DevBuf<uint32_t> a_, a_sum_, a_start_, moved_, rescan_, chg_ids_;
    DevBuf<double> sims_start_, xnorm2_;
    DevBuf<float> sb_, ss_;
    DevBuf<uint32_t> pcnt_, pptr_;
    DevBuf<uint2> pairs_;
    DevBuf<unsigned char> scan_tmp_;
    int64_t postings_total_ = 0;
    double screen_ms_ = 0.0;
    uint32_t screen_launches_ = 0;
    int screen_kind_ = 2;  // 0 dense, 1 postings, 2 by measured density
    uint32_t post_kt_max_ = 1024;
    int post_warps_ = 8;
    bool cache_trusted_ = false;
    bool scalars_fresh_ = false;
    // the assign's closing kernels launched ahead of the screen's counters (bound_assign)
    bool speculate_ok_ = true, speculate_finish_ = false, finish_speculated_ = false;
    uint64_t last_full_n_exact_ = 1;
    bool counts_fresh_ = false;  // the last assign's cluster sizes: none empty, nothing since changed an assignment
    std::map<const void*, std::pair<int, int>> launch_cfg_;
    void* stage_[2] = {nullptr, nullptr};  // pinned upload staging (h2d)
    double h2d_wait_ms_ = 0.0, h2d_copy_ms_ = 0.0;
    cudaEvent_t stage_ev_[2]{};
    bool stage_used_[2] = {false, false};
    bool stage_failed_ = false;  // pinned staging unavailable: pageable copies  // bound screen: (warps per block, blocks per SM)
    bool last_hp_overflow_ = false;  // the last pass ran with dropped postings lists (looser bound)  // hs_ was pulled by the last bound-screen pass
    bool fuse_resolve_ = false;
    bool bound_enabled_ = true;   // bound screen (SSKM_BOUND=0: the full postings / dense screens)
    bool theta_adapt_ = true;
    bool debug_ = false;  // SSKM_DEBUG=1: per-assign screen counters on stderr
    float theta_ = 0.004f;        // fixed high/low split of the centroid weights (SSKM_THETA)
    struct ThetaCtl {
        float theta = 0.004f;   // adaptive split, per pass kind (full, NCC pass A, rescan)
        double target = 192.0;  // hash passes: high pairs per document
        double acc_fb = 0.0, acc_work = 0.0, acc_hovf = 0.0;  // the current period
        uint32_t passes = 0;
    };
    ThetaCtl tctl_[3];
    // per-assign bound-screen totals (stats)
    uint64_t bstat_docs_ = 0, bstat_pairs_ = 0, bstat_cand_ = 0, bstat_doc_nnz_ = 0, bstat_cand_nnz_ = 0,
             bstat_visits_ = 0, bstat_own_ = 0;
    uint64_t bstat_own_nnz_ = 0;
    uint32_t updates_since_assign_ = 0;  // updates since the last assign (the same_ flags' validity)
    double bstat_theta_ = 0.0;
    uint64_t dots_ = 0;
    // drift bound (skip_kernel)
    DevBuf<__half> ub_;        // [n][32]: per document and cluster group
    DevBuf<uint32_t> ub_it_, skip_list_;
    DevBuf<double> dcum_;
    DevBuf<unsigned long long> skip_ctr_;
    uint32_t dcum_rows_ = 0;   // rows of dcum_ ([iteration][32]) written so far
    bool ub_valid_ = false;     // every document's bound is valid for the current assignments
    // high postings kept across passes (single cluster tile over Cᵀ)
    static constexpr uint32_t kRebuildEvery = 4;
    int wg_rows_ = 2;  // SSKM_WG_ROWS: marked rows per round of the column rewrite (2, or 4 for A/B runs)
    uint32_t rebuild_late_ = 16;  // SSKM_REBUILD_LATE: the period once few columns change per update
    // The kept lists are rebuilt for fresh, tight L_t (maintenance only ever
    // raises them) and to re-tune θ: every 4 assigns while the centroids still
    // move a lot, less often once an update rewrites under a third of the columns.
    uint32_t rebuild_every() const { return last_n_rec_ * 3 < k_ ? rebuild_late_ : kRebuildEvery; }
    uint32_t last_n_rec_ = 0xFFFFFFFFu / 4;
    bool hp_valid_ = false;     // hptr_/pairs_ hold exactly Cᵀ's entries >= hp_theta_
    bool keep_lists_ = true;    // SSKM_KEEP_LISTS=0: rebuild the high postings every assign
    float theta0_ = 0.004f, hash_theta0_ = 0.02f;
    bool theta0_set_ = false, hash_theta_started_ = false;
    float hp_theta_ = 0.f;
    uint32_t assigns_since_build_ = 0;
    double last_update_ms_ = 0.0;  // the last update's device time (θ tuning)
    uint64_t kpp_host_rounds_ = 0;  // k-means++ rounds the host had to replay (last seeding)
    bool skip_enabled_ = true;  // SSKM_SKIP=0: screen every document
    // SSKM_INDEX_ACCOUNTING=0: `ncc+index` runs at the NCC step's speed and reports the NCC
    // counters (index_active = 0) instead of replaying the reference's index for its counters
    bool index_accounting_ = true;
    // second pass of the hash screens (bound_second_pass)
    bool second_pass_ = true;          // SSKM_SECOND_PASS=0: fallen-through documents go straight to the exact scan
    float second_pass_ratio_ = 0.5f;  // θ of the second lists relative to the first pass's (measured on c4)
    uint64_t second_pass_min_ = 512;   // fewer fallen-through documents than this: not worth the lists
    DevBuf<uint4> hptr2_;
    DevBuf<uint2> pairs2_;
    DevBuf<unsigned long long> hpctr2_;
    DevBuf<uint32_t> exact2_;
    DevBuf<double> span_s_;   // exact scan of short lists: per (document, column span) maxima
    DevBuf<uint32_t> span_a_;
    double second_ms_ = 0.0;
    uint64_t second_docs_ = 0;
    bool hash_enabled_ = true;  // SSKM_HASH=0: multi-tile passes instead of one hash-accumulator pass
    DevBuf<uint32_t> df_;       // document frequency per term (hash-pass θ)
    bool df_ready_ = false;
    uint64_t skip_docs_ = 0;
    double skip_ms_ = 0.0;  // dots the kernels evaluated in the current assign (gpu_dot_products)
    bool nonneg_ = true;
    double last_density_ = 0.0;
    double dense_above_ = 0.15;
    uint64_t dense_assigns_ = 0;
    double ncc_full_frac_ = 0.0;  // SSKM_NCC_FULL_FRAC: NCC passes over the changed list only below this changed share (measured: the full screened scan with the drift bound is never slower)
    DevBuf<uint32_t> sa_, exact_;
    DevBuf<uint32_t> order_, keys32_;
    DevBuf<double> sims_, drift_, part_, obj_part_;
    DevBuf<unsigned long long> Q_;  // exact Σ_t S[t][j]² per column (128-bit: lo, hi)
    DevBuf<unsigned int> nz_;       // a bit per (term, cluster): S or Cᵀ may be nonzero there
    DevBuf<uint8_t> unchanged_, touched_, repaired_flag_;
    DevBuf<unsigned long long> counts_, keys_;
    DevBuf<uint32_t> vals_, moves_, mv_old_, mv_new_;
    DevBuf<int64_t> mv_len_, mv_off_;
    int64_t mv_n_ = 0, mv_nnz_ = 0;
    DevBuf<unsigned char> sort_tmp_;
};

}  // namespace sskm_b200

#include "multi.cuh"

// ====================================================================== C-ABI
using sskm_b200::Engine;
using sskm_b200::MultiEngine;

struct sskm_ctx {
    std::unique_ptr<Engine> eng;
};

struct sskm_multi {
    std::unique_ptr<MultiEngine> m;
};

namespace {
thread_local std::string g_err;
// sskm_cluster_csr keeps one engine per device; the map lock is held only for
// the lookup, each engine's own lock for its run (runs on different devices
// proceed in parallel)
struct CachedEngine {
    std::mutex mu;
    std::unique_ptr<Engine> eng;
};
std::mutex g_cache_mu;
std::map<int, std::shared_ptr<CachedEngine>> g_engine_cache;

}  // namespace

namespace sskm_b200 {
void set_last_error(const char* msg) { g_err = msg; }
}  // namespace sskm_b200

namespace {
template <class F>
int guard(F&& f) {
    try {
        f();
        return SSKM_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SSKM_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SSKM_ERUNTIME;
    } catch (...) {
        g_err = "unknown error";
        return SSKM_ERUNTIME;
    }
}

Engine& E(sskm_ctx* c) {
    if (!c || !c->eng) throw sskm_b200::InvalidArgument("null context");
    CK(cudaSetDevice(c->eng->device()));  // the calling thread may have another current device
    return *c->eng;
}

MultiEngine& M(sskm_multi* c) {
    if (!c || !c->m) throw sskm_b200::InvalidArgument("null context");
    return *c->m;
}

std::vector<int> device_list(int32_t n, const int32_t* devs) {
    if (n <= 0 || !devs) throw sskm_b200::InvalidArgument("device list must not be empty");
    return std::vector<int>(devs, devs + n);
}

template <class Step, class Cfg>
void run_loop(Step&& step, const Cfg& cfg, sskm_iteration_stats* stats, uint32_t cap, uint32_t* n_iters,
              int32_t* stop_reason, double* objective);

bool stop_after(const sskm_iteration_stats& st, double conv, int32_t* reason) {
    if (st.n_reassigned == 0) {
        *reason = SSKM_STOP_NO_REASSIGNMENTS;
        return true;
    }
    if (st.iteration > 1 && st.max_sq_drift < conv) {
        *reason = SSKM_STOP_CENTROID_DRIFT;
        return true;
    }
    return false;
}

// run() loop (engine.cpp:357-424) over any step function.
template <class Step, class Cfg>
void run_loop(Step&& step_fn, const Cfg& cfg, sskm_iteration_stats* stats, uint32_t cap, uint32_t* n_iters,
              int32_t* stop_reason, double* objective) {
    int32_t reason = SSKM_STOP_MAX_ITERATIONS;
    uint32_t t = 0;
    double obj = 0.0;
    for (uint32_t iter = 1; iter <= cfg.max_iters; ++iter) {
        sskm_iteration_stats st{};
        step_fn(&st);
        if (stats && t < cap) stats[t] = st;
        ++t;
        obj = st.objective;
        if (stop_after(st, cfg.conv_sq_dist, &reason)) break;
    }
    if (n_iters) *n_iters = t;
    if (stop_reason) *stop_reason = reason;
    if (objective) *objective = obj;
}

void step(Engine& e, sskm_iteration_stats* st) {
    const auto t0 = std::chrono::steady_clock::now();
    e.update(st);
    sskm_iteration_stats a{};
    e.assign(&a);
    st->n_reassigned = a.n_reassigned;
    st->dot_products = a.dot_products;
    st->gpu_dot_products = a.gpu_dot_products;
    st->n_changed = a.n_changed;
    st->n_rescan = a.n_rescan;
    st->objective = a.objective;
    st->assign_ms = a.assign_ms;
    st->assign_kernel_ms = a.assign_kernel_ms;
    st->screen_ms = a.screen_ms;
    st->screen_launches = a.screen_launches;
    st->centroid_density = a.centroid_density;
    st->n_exact = a.n_exact;
    st->index_active = a.index_active;
    st->index_queries = a.index_queries;
    st->candidates_total = a.candidates_total;
    st->index_build_seconds = a.index_build_seconds;
    st->bound_docs = a.bound_docs;
    st->bound_pairs = a.bound_pairs;
    st->bound_candidates = a.bound_candidates;
    st->bound_doc_nnz = a.bound_doc_nnz;
    st->bound_cand_nnz = a.bound_cand_nnz;
    st->bound_theta = a.bound_theta;
    st->bound_visits = a.bound_visits;
    st->bound_own_dots = a.bound_own_dots;
    st->bound_own_nnz = a.bound_own_nnz;
    st->skip_docs = a.skip_docs;
    st->second_pass_docs = a.second_pass_docs;
    st->skip_ms = a.skip_ms;
    st->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

extern "C" {

const char* sskm_last_error(void) { return g_err.c_str(); }

int sskm_validate(const sskm_run_config* cfg, uint64_t n_docs) {
    return guard([&] {
        if (!cfg) throw sskm_b200::InvalidArgument("null config");
        Engine::validate(*cfg, n_docs);
    });
}

int sskm_open(int32_t device, sskm_ctx** out) {
    return guard([&] {
        if (!out) throw sskm_b200::InvalidArgument("null output");
        auto* c = new sskm_ctx();
        try {
            c->eng = std::make_unique<Engine>(device);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int sskm_close(sskm_ctx* ctx) {
    return guard([&] { delete ctx; });
}

int sskm_upload_csr(sskm_ctx* ctx, int64_t n_docs, uint32_t dims, const int64_t* indptr,
                    const int32_t* indices, const float* values, int64_t doc_offset, int64_t n_docs_total) {
    return guard([&] { E(ctx).upload(n_docs, dims, indptr, indices, values, doc_offset, n_docs_total); });
}

int sskm_configure(sskm_ctx* ctx, const sskm_run_config* cfg) {
    return guard([&] {
        if (!cfg) throw sskm_b200::InvalidArgument("null config");
        E(ctx).configure(*cfg);
    });
}

int sskm_init_from_seeds(sskm_ctx* ctx, const uint32_t* seeds) {
    return guard([&] { E(ctx).init_from_seeds(seeds); });
}

int sskm_init_kmeanspp(sskm_ctx* ctx, uint64_t seed, uint32_t* seeds_out) {
    return guard([&] { E(ctx).init_kmeanspp(seed, seeds_out); });
}

int sskm_update(sskm_ctx* ctx, sskm_iteration_stats* st) {
    return guard([&] { E(ctx).update(st); });
}

int sskm_assign(sskm_ctx* ctx, sskm_iteration_stats* st) {
    return guard([&] {
        std::memset(st, 0, sizeof(*st));
        E(ctx).assign(st);
    });
}

int sskm_step(sskm_ctx* ctx, sskm_iteration_stats* st) {
    return guard([&] { step(E(ctx), st); });
}

int sskm_step_n(sskm_ctx* ctx, uint32_t n, sskm_iteration_stats* stats) {
    return guard([&] {
        Engine& e = E(ctx);
        for (uint32_t t = 0; t < n; ++t) {
            sskm_iteration_stats st{};
            step(e, &st);
            if (stats) stats[t] = st;
        }
    });
}

int sskm_run(sskm_ctx* ctx, sskm_iteration_stats* stats, uint32_t cap, uint32_t* n_iters, int32_t* stop_reason) {
    return guard([&] {
        Engine& e = E(ctx);
        int32_t reason = SSKM_STOP_MAX_ITERATIONS;
        uint32_t t = 0;
        for (uint32_t iter = 1; iter <= e.config().max_iters; ++iter) {
            sskm_iteration_stats st{};
            step(e, &st);
            if (stats && t < cap) stats[t] = st;
            ++t;
            if (stop_after(st, e.config().conv_sq_dist, &reason)) break;
        }
        if (n_iters) *n_iters = t;
        if (stop_reason) *stop_reason = reason;
    });
}

int sskm_get_state(sskm_ctx* ctx, uint32_t* a, double* sims, uint8_t* unchanged) {
    return guard([&] { E(ctx).get_state(a, sims, unchanged); });
}

int sskm_set_state(sskm_ctx* ctx, const uint32_t* a, const double* sims, uint32_t iteration) {
    return guard([&] { E(ctx).set_state(a, sims, iteration); });
}

int sskm_set_unchanged(sskm_ctx* ctx, const uint8_t* flags) {
    return guard([&] { E(ctx).set_unchanged(flags); });
}

int sskm_get_centroids(sskm_ctx* ctx, float* ct) {
    return guard([&] { E(ctx).get_centroids(ct); });
}

int sskm_get_centroid_rows(sskm_ctx* ctx, uint32_t n_rows, const uint32_t* rows, float* out) {
    return guard([&] { E(ctx).get_centroid_rows(n_rows, rows, out); });
}

int sskm_get_centroid_cols(sskm_ctx* ctx, uint32_t n_cols, const uint32_t* cols, float* out) {
    return guard([&] { E(ctx).get_centroid_cols(n_cols, cols, out); });
}

int sskm_debug_check_postings(sskm_ctx* ctx, int64_t* bad_rows) {
    return guard([&] { *bad_rows = E(ctx).check_postings(); });
}

int sskm_set_centroids(sskm_ctx* ctx, const float* ct) {
    return guard([&] { E(ctx).set_centroids(ct); });
}

int sskm_get_repaired(sskm_ctx* ctx, uint32_t* repaired, uint32_t* n_repaired) {
    return guard([&] {
        const auto& r = E(ctx).repaired();
        if (repaired) std::memcpy(repaired, r.data(), r.size() * 4);
        *n_repaired = static_cast<uint32_t>(r.size());
    });
}

int sskm_get_iteration(sskm_ctx* ctx, uint32_t* iteration) {
    return guard([&] { *iteration = E(ctx).iteration(); });
}

int sskm_cluster_csr(const sskm_run_config* cfg, int64_t n_docs, uint32_t dims, const int64_t* indptr,
                     const int32_t* indices, const float* values, const uint32_t* seeds, uint32_t* assignments,
                     double* sims, float* ct, sskm_iteration_stats* stats, uint32_t stats_cap,
                     uint32_t* n_iters, int32_t* stop_reason, double* objective) {
    return guard([&] {
        if (!cfg) throw sskm_b200::InvalidArgument("null config");
        Engine::validate(*cfg, n_docs > 0 ? static_cast<uint64_t>(n_docs) : 0);
        // one persistent engine per device: its HBM buffers are reused by the
        // next call instead of being freed (cudaFree synchronises and costs
        // ~0.1-0.5 s for the c1 working set)
        std::shared_ptr<CachedEngine> slot;
        {
            std::lock_guard<std::mutex> lock(g_cache_mu);
            auto& s = g_engine_cache[cfg->device];
            if (!s) s = std::make_shared<CachedEngine>();
            slot = s;
        }
        std::lock_guard<std::mutex> run_lock(slot->mu);
        if (!slot->eng) slot->eng = std::make_unique<Engine>(cfg->device);
        Engine& e = *slot->eng;
        CK(cudaSetDevice(cfg->device));
        e.upload(n_docs, dims, indptr, indices, values, 0, n_docs);
        e.configure(*cfg);
        if (seeds) {
            e.init_from_seeds(seeds);
        } else {
            e.init_kmeanspp(cfg->seed, nullptr);
        }
        int32_t reason = SSKM_STOP_MAX_ITERATIONS;
        uint32_t t = 0;
        double obj = 0.0;
        for (uint32_t iter = 1; iter <= cfg->max_iters; ++iter) {
            sskm_iteration_stats st{};
            step(e, &st);
            if (stats && t < stats_cap) stats[t] = st;
            ++t;
            obj = st.objective;
            if (stop_after(st, cfg->conv_sq_dist, &reason)) break;
        }
        e.get_state(assignments, sims, nullptr);
        if (ct) e.get_centroids(ct);
        if (n_iters) *n_iters = t;
        if (stop_reason) *stop_reason = reason;
        if (objective) *objective = obj;
    });
}

// ------------------------------------------------------- multi-device --
int sskm_multi_open(int32_t n_devices, const int32_t* devices, sskm_multi** out) {
    return guard([&] {
        if (!out) throw sskm_b200::InvalidArgument("null output");
        auto* c = new sskm_multi();
        try {
            c->m = std::make_unique<MultiEngine>(device_list(n_devices, devices));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int sskm_multi_close(sskm_multi* ctx) {
    return guard([&] { delete ctx; });
}

int sskm_multi_upload_csr(sskm_multi* ctx, int64_t n_docs, uint32_t dims, const int64_t* indptr,
                          const int32_t* indices, const float* values) {
    return guard([&] { M(ctx).upload(n_docs, dims, indptr, indices, values); });
}

int sskm_multi_configure(sskm_multi* ctx, const sskm_run_config* cfg) {
    return guard([&] {
        if (!cfg) throw sskm_b200::InvalidArgument("null config");
        M(ctx).configure(*cfg);
    });
}

int sskm_multi_init_from_seeds(sskm_multi* ctx, const uint32_t* seeds) {
    return guard([&] { M(ctx).init_from_seeds(seeds); });
}

int sskm_multi_step(sskm_multi* ctx, sskm_iteration_stats* st) {
    return guard([&] { M(ctx).step(st); });
}

int sskm_multi_run(sskm_multi* ctx, sskm_iteration_stats* stats, uint32_t cap, uint32_t* n_iters,
                   int32_t* stop_reason) {
    return guard([&] {
        MultiEngine& m = M(ctx);
        run_loop([&](sskm_iteration_stats* st) { m.step(st); }, m.config(), stats, cap, n_iters, stop_reason,
                 nullptr);
    });
}

int sskm_multi_get_state(sskm_multi* ctx, uint32_t* assignments, double* sims) {
    return guard([&] { M(ctx).get_state(assignments, sims); });
}

int sskm_multi_get_centroids(sskm_multi* ctx, float* ct) {
    return guard([&] { M(ctx).get_centroids(ct); });
}

int sskm_multi_launch_count(sskm_multi* ctx, uint64_t* n) {
    return guard([&] { *n = M(ctx).launches(); });
}

int sskm_cluster_csr_multi(const sskm_run_config* cfg, int32_t n_devices, const int32_t* devices, int64_t n_docs,
                           uint32_t dims, const int64_t* indptr, const int32_t* indices, const float* values,
                           const uint32_t* seeds, uint32_t* assignments, double* sims, float* ct,
                           sskm_iteration_stats* stats, uint32_t stats_cap, uint32_t* n_iters, int32_t* stop_reason,
                           double* objective) {
    return guard([&] {
        if (!cfg) throw sskm_b200::InvalidArgument("null config");
        Engine::validate(*cfg, n_docs > 0 ? static_cast<uint64_t>(n_docs) : 0);
        if (!seeds) throw sskm_b200::InvalidArgument("a multi-device run needs init_seeds (k-means++ runs on one device)");
        MultiEngine m(device_list(n_devices, devices));
        m.upload(n_docs, dims, indptr, indices, values);
        m.configure(*cfg);
        m.init_from_seeds(seeds);
        run_loop([&](sskm_iteration_stats* st) { m.step(st); }, *cfg, stats, stats_cap, n_iters, stop_reason,
                 objective);
        m.get_state(assignments, sims);
        if (ct) m.get_centroids(ct);
    });
}

int sskm_release_cache(void) {
    return guard([&] {
        std::lock_guard<std::mutex> lock(g_cache_mu);
        g_engine_cache.clear();
    });
}

int sskm_local_counts(sskm_ctx* ctx, int64_t* counts) {
    return guard([&] { E(ctx).local_counts(counts); });
}

int sskm_move_doc(sskm_ctx* ctx, int64_t global_doc, uint32_t cluster) {
    return guard([&] { E(ctx).move_doc(global_doc, cluster); });
}

int sskm_moved_prepare(sskm_ctx* ctx, int64_t* n_moved, int64_t* nnz_moved) {
    return guard([&] { E(ctx).moved_prepare(n_moved, nnz_moved); });
}

int sskm_moved_pack(sskm_ctx* ctx, uint32_t* old_c, uint32_t* new_c, int32_t* lens, int32_t* idx, float* val) {
    return guard([&] { E(ctx).moved_pack(old_c, new_c, lens, idx, val); });
}

int sskm_local_candidates(sskm_ctx* ctx, int64_t m, double* sims, int64_t* gids, uint32_t* clusters,
                          int64_t* m_out) {
    return guard([&] { *m_out = E(ctx).local_candidates(m, sims, gids, clusters); });
}

int sskm_init_from_rows(sskm_ctx* ctx, const int64_t* row_ptr, const int32_t* idx, const float* val) {
    return guard([&] { E(ctx).init_from_rows(row_ptr, idx, val); });
}

int sskm_update_apply(sskm_ctx* ctx, int64_t n_moved, const uint32_t* old_c, const uint32_t* new_c,
                      const int64_t* row_ptr, const int32_t* idx, const float* val, const uint32_t* repaired,
                      uint32_t n_repaired, sskm_iteration_stats* st) {
    return guard([&] { E(ctx).update_apply(n_moved, old_c, new_c, row_ptr, idx, val, repaired, n_repaired, st); });
}

int sskm_timer_record(sskm_ctx* ctx, int32_t slot) {
    return guard([&] { E(ctx).timer_record(slot); });
}

int sskm_timer_elapsed(sskm_ctx* ctx, int32_t a, int32_t b, double* ms) {
    return guard([&] { *ms = E(ctx).timer_elapsed(a, b); });
}

int sskm_launch_count(sskm_ctx* ctx, uint64_t* n) {
    return guard([&] { *n = E(ctx).launches(); });
}

int sskm_synchronize(sskm_ctx* ctx) {
    return guard([&] { E(ctx).synchronize(); });
}

int sskm_postings_work(sskm_ctx* ctx, uint64_t* pairs) {
    return guard([&] { *pairs = E(ctx).postings_work(); });
}

int sskm_local_sims_sum(sskm_ctx* ctx, double* sum) {
    return guard([&] { *sum = E(ctx).local_sims_sum(); });
}

}  // extern "C"
