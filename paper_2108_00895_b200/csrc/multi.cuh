// Multi-device context: one host process drives several GPUs of one node
// (SURVEY §8b `sskm_cuda_open(n_dev, devs)`, §8e). Documents are sharded in
// contiguous equal ranges, one Engine per device; Cᵀ and the exact integer
// cluster sums are replicated. The exchange of an iteration needs no
// collective library and no gather: each device applies the moved rows of
// EVERY shard to its own sums with the delta kernel reading the peers' CSR
// rows and moved lists directly over NVLink (peer access), ordered by CUDA
// events across the devices' streams. Integer sums are associative, so every
// device holds bit-identical sums, renormalises bit-identical centroids and
// derives identical NCC flags — the assignments, sims and centroids equal a
// single-GPU run bit for bit. Per iteration (engine.cpp:357-407):
//
//   1. local cluster sizes → host, summed (k · 8 B per device); empty clusters
//      (rare) are repaired by replaying the reference's sequential rule
//      (engine.cpp:154-167) over the merged donor candidates of all shards;
//   2. moved list per shard (device-resident);
//   3. every device: rows of every shard's moved documents into its sums
//      (peer reads); 4. once all devices are done: column rewrite + flags;
//   5. assign, local to each shard; counters summed, objective partials summed
//      in device order.
//
// A worker thread per device issues each phase, so the devices' host-side
// synchronisations overlap; phases are separated by a host join.
#pragma once

#include <condition_variable>
#include <exception>
#include <functional>
#include <thread>

namespace sskm_b200 {

// Persistent workers, one per device; run(f) calls f(r) on worker r for every
// r and returns when all are done (the first exception is rethrown).
class DevicePool {
public:
    explicit DevicePool(const std::vector<int>& devices) : devs_(devices) {
        if (devs_.size() > 1)
            for (size_t r = 0; r < devs_.size(); ++r) th_.emplace_back([this, r] { loop(r); });
    }
    ~DevicePool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(const std::function<void(size_t)>& f) {
        if (devs_.size() == 1) {  // inline on the caller
            CK(cudaSetDevice(devs_[0]));
            f(0);
            return;
        }
        {
            std::lock_guard<std::mutex> l(mu_);
            task_ = &f;
            pending_ = devs_.size();
            err_ = nullptr;
            ++gen_;
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> l(mu_);
        done_cv_.wait(l, [this] { return pending_ == 0; });
        task_ = nullptr;
        if (err_) std::rethrow_exception(err_);
    }

private:
    void loop(size_t r) {
        uint64_t seen = 0;
        cudaSetDevice(devs_[r]);
        for (;;) {
            const std::function<void(size_t)>* f;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                f = task_;
            }
            std::exception_ptr e;
            try {
                CK(cudaSetDevice(devs_[r]));
                (*f)(r);
            } catch (...) {
                e = std::current_exception();
            }
            {
                std::lock_guard<std::mutex> l(mu_);
                if (e && !err_) err_ = e;
                if (--pending_ == 0) done_cv_.notify_all();
            }
        }
    }
    std::vector<int> devs_;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t)>* task_ = nullptr;
    size_t pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
    std::exception_ptr err_;
};

// The sequential repair rule of compute_centroids (engine.cpp:154-167) over
// donor candidates in the reference's scan order (lowest sim, ties to the
// lowest document index): each empty cluster j, ascending, takes the first
// unused candidate whose current cluster still has >= 2 members. cur[] is the
// candidates' current clusters. Returns false when the candidates run out.
inline bool replay_repair(std::vector<unsigned long long> cnt, const std::vector<int64_t>& docs,
                          std::vector<uint32_t> cur, std::vector<std::pair<int64_t, uint32_t>>& moves) {
    const size_t m = docs.size();
    std::vector<uint8_t> used(m, 0);
    size_t pos = 0;
    moves.clear();
    for (uint32_t j = 0; j < cnt.size(); ++j) {
        if (cnt[j] != 0) continue;
        size_t c = pos;
        while (c < m && (used[c] || cnt[cur[c]] < 2)) ++c;
        if (c == m) return false;
        used[c] = 1;
        while (pos < m && used[pos]) ++pos;
        --cnt[cur[c]];
        cur[c] = j;
        cnt[j] = 1;
        moves.emplace_back(docs[c], j);
    }
    return true;
}

class MultiEngine {
public:
    explicit MultiEngine(const std::vector<int>& devices) : devs_(devices) {
        if (devices.empty()) throw InvalidArgument("no devices");
        for (int d : devices) engs_.push_back(std::make_unique<Engine>(d));
        // peer access between distinct devices (the delta kernels read peers' shards)
        for (int a : devices)
            for (int b : devices) {
                if (a == b) continue;
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, a, b));
                if (!ok) throw CudaError("multi-device context: no peer access between devices");
                CK(cudaSetDevice(a));
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) {
                    (void)cudaGetLastError();
                } else {
                    CK(e);
                }
            }
        for (size_t r = 0; r < devs_.size(); ++r) {
            CK(cudaSetDevice(devs_[r]));
            cudaEvent_t e1, e2;
            CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
            ev_moved_.push_back(e1);
            ev_delta_.push_back(e2);
        }
        pool_ = std::make_unique<DevicePool>(devs_);
    }
    ~MultiEngine() {
        pool_.reset();
        for (size_t r = 0; r < devs_.size(); ++r) {
            cudaSetDevice(devs_[r]);
            cudaEventDestroy(ev_moved_[r]);
            cudaEventDestroy(ev_delta_[r]);
        }
    }

    size_t size() const { return engs_.size(); }
    Engine& engine(size_t r) { return *engs_[r]; }

    void upload(int64_t n, uint32_t dims, const int64_t* indptr, const int32_t* indices, const float* values) {
        if (n <= 0) throw InvalidArgument("empty corpus");
        if (indptr[0] != 0) throw InvalidArgument("indptr[0] must be 0");
        const size_t p = engs_.size();
        if (static_cast<int64_t>(p) > n) throw InvalidArgument("more devices than documents");
        n_ = n;
        off_.assign(p + 1, 0);
        for (size_t r = 0; r <= p; ++r) off_[r] = n * static_cast<int64_t>(r) / static_cast<int64_t>(p);
        pool_->run([&](size_t r) {
            const int64_t b = off_[r], e = off_[r + 1];
            std::vector<int64_t> ptr(indptr + b, indptr + e + 1);
            for (auto& x : ptr) x -= indptr[b];
            engs_[r]->upload(e - b, dims, ptr.data(), indices + indptr[b], values + indptr[b], b, n);
        });
        configured_ = false;
    }

    void configure(const sskm_run_config& c) {
        pool_->run([&](size_t r) { engs_[r]->configure(c); });
        cfg_ = c;
        lambdas_.assign(c.lambdas, c.lambdas + c.n_lambdas);
        cfg_.lambdas = lambdas_.data();
        k_ = c.k;
        configured_ = true;
    }

    const sskm_run_config& config() const { return cfg_; }

    // BASELINE init: the k seed rows gathered from their shards, then every
    // device builds Cᵀ from them and runs its shard's seed assignment.
    void init_from_seeds(const uint32_t* seeds) {
        need_config();
        std::vector<std::vector<uint32_t>> local(engs_.size());
        std::vector<std::vector<uint32_t>> which(engs_.size());
        for (uint32_t j = 0; j < k_; ++j) {
            const int64_t g = seeds[j];
            if (g < 0 || g >= n_) throw InvalidArgument("seed out of range");
            const size_t r = owner(g);
            local[r].push_back(static_cast<uint32_t>(g - off_[r]));
            which[r].push_back(j);
        }
        std::vector<std::vector<int64_t>> rp(engs_.size());
        std::vector<std::vector<int32_t>> ri(engs_.size());
        std::vector<std::vector<float>> rv(engs_.size());
        pool_->run([&](size_t r) { engs_[r]->get_rows(local[r], rp[r], ri[r], rv[r]); });
        std::vector<int64_t> len(k_, 0);
        std::vector<std::pair<size_t, size_t>> src(k_);
        for (size_t r = 0; r < engs_.size(); ++r)
            for (size_t q = 0; q < which[r].size(); ++q) {
                len[which[r][q]] = rp[r][q + 1] - rp[r][q];
                src[which[r][q]] = {r, q};
            }
        std::vector<int64_t> ptr(k_ + 1, 0);
        for (uint32_t j = 0; j < k_; ++j) ptr[j + 1] = ptr[j] + len[j];
        std::vector<int32_t> idx(std::max<int64_t>(ptr[k_], 1));
        std::vector<float> val(std::max<int64_t>(ptr[k_], 1));
        for (uint32_t j = 0; j < k_; ++j) {
            const auto [r, q] = src[j];
            std::copy(ri[r].begin() + rp[r][q], ri[r].begin() + rp[r][q + 1], idx.begin() + ptr[j]);
            std::copy(rv[r].begin() + rp[r][q], rv[r].begin() + rp[r][q + 1], val.begin() + ptr[j]);
        }
        pool_->run([&](size_t r) { engs_[r]->init_from_rows(ptr.data(), idx.data(), val.data()); });
        state_ = true;
    }

    void step(sskm_iteration_stats* st) {
        need_state();
        const auto t0 = std::chrono::steady_clock::now();
        const size_t p = engs_.size();
        // 1. cluster sizes
        std::vector<std::vector<unsigned long long>> cnt(p, std::vector<unsigned long long>(k_));
        pool_->run([&](size_t r) { engs_[r]->mp_begin(cnt[r].data()); });
        std::vector<unsigned long long> tot(k_, 0);
        for (size_t r = 0; r < p; ++r)
            for (uint32_t j = 0; j < k_; ++j) tot[j] += cnt[r][j];
        std::vector<std::vector<uint32_t>> moves(p);
        std::vector<uint32_t> repaired;
        if (std::find(tot.begin(), tot.end(), 0ull) != tot.end()) repair(tot, moves, repaired);
        // 2-4. moved lists, peer deltas, column rewrite
        pool_->run([&](size_t r) { engs_[r]->mp_moved(moves[r], repaired, ev_moved_[r]); });
        std::vector<Engine::PeerView> views;
        for (auto& e : engs_) views.push_back(e->peer_view());
        pool_->run([&](size_t r) { engs_[r]->mp_delta(views, ev_moved_, ev_delta_[r]); });
        std::vector<sskm_iteration_stats> su(p), sa(p);
        pool_->run([&](size_t r) { engs_[r]->mp_finish(ev_delta_, &su[r]); });
        // 5. assign
        pool_->run([&](size_t r) {
            std::memset(&sa[r], 0, sizeof(sa[r]));
            engs_[r]->assign(&sa[r]);
        });
        combine(su, sa, st);
        st->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }

    void get_state(uint32_t* a, double* sims) {
        need_state();
        pool_->run([&](size_t r) {
            engs_[r]->get_state(a ? a + off_[r] : nullptr, sims ? sims + off_[r] : nullptr, nullptr);
        });
    }

    void get_centroids(float* ct) {
        need_state();
        CK(cudaSetDevice(devs_[0]));
        engs_[0]->get_centroids(ct);
    }

    uint64_t launches() const {
        uint64_t t = 0;
        for (auto& e : engs_) t += e->launches();
        return t;
    }

private:
    size_t owner(int64_t g) const {
        size_t r = static_cast<size_t>(std::upper_bound(off_.begin(), off_.end(), g) - off_.begin()) - 1;
        return std::min(r, engs_.size() - 1);
    }
    void need_config() const {
        if (!configured_) throw InvalidArgument("context not configured");
    }
    void need_state() const {
        need_config();
        if (!state_) throw InvalidArgument("no clustering state: initialise from seeds first");
    }

    // Empty clusters: the first m donor candidates of every shard (local
    // (sim, doc) order = global order within a shard), merged by (sim, global
    // id) and replayed; m grows when the candidates run out.
    void repair(const std::vector<unsigned long long>& tot, std::vector<std::vector<uint32_t>>& moves,
                std::vector<uint32_t>& repaired) {
        const size_t p = engs_.size();
        int64_t n_empty = 0;
        for (auto c : tot) n_empty += c == 0;
        int64_t m = std::min<int64_t>(n_, 2 * n_empty + 256);
        for (;;) {
            struct Cand {
                double sim;
                int64_t gid;
                uint32_t cur;
            };
            std::vector<std::vector<Cand>> per(p);
            pool_->run([&](size_t r) {
                const int64_t mr = std::min<int64_t>(m, off_[r + 1] - off_[r]);
                std::vector<double> s(std::max<int64_t>(mr, 1));
                std::vector<int64_t> g(std::max<int64_t>(mr, 1));
                std::vector<uint32_t> c(std::max<int64_t>(mr, 1));
                const int64_t got = engs_[r]->local_candidates(mr, s.data(), g.data(), c.data());
                for (int64_t q = 0; q < got; ++q) per[r].push_back({s[q] + 0.0, g[q], c[q]});
            });
            std::vector<Cand> all;
            for (auto& v : per) all.insert(all.end(), v.begin(), v.end());
            std::sort(all.begin(), all.end(), [](const Cand& x, const Cand& y) {
                return x.sim < y.sim || (x.sim == y.sim && x.gid < y.gid);
            });
            if (static_cast<int64_t>(all.size()) > m) all.resize(m);
            std::vector<int64_t> docs;
            std::vector<uint32_t> cur;
            for (auto& c : all) {
                docs.push_back(c.gid);
                cur.push_back(c.cur);
            }
            std::vector<std::pair<int64_t, uint32_t>> mv;
            if (replay_repair(tot, docs, cur, mv)) {
                for (auto& [g, j] : mv) {
                    const size_t r = owner(g);
                    moves[r].push_back(static_cast<uint32_t>(g - off_[r]));
                    moves[r].push_back(j);
                    repaired.push_back(j);
                }
                return;
            }
            if (m >= n_) throw CudaError("empty-cluster repair found no donor");
            m = std::min<int64_t>(n_, m * 4);
        }
    }

    static void combine(const std::vector<sskm_iteration_stats>& su, const std::vector<sskm_iteration_stats>& sa,
                        sskm_iteration_stats* st) {
        *st = su[0];  // update results are identical on every device
        st->n_moved = 0;
        st->update_ms = 0.0;
        for (auto& u : su) {
            st->n_moved += u.n_moved;
            st->update_ms = std::max(st->update_ms, u.update_ms);
        }
        const sskm_iteration_stats& a0 = sa[0];
        st->n_changed = a0.n_changed;
        st->centroid_density = a0.centroid_density;
        st->bound_theta = a0.bound_theta;
        st->index_active = a0.index_active;
        st->n_reassigned = st->dot_products = st->gpu_dot_products = st->n_rescan = st->n_exact = 0;
        st->index_queries = st->candidates_total = 0;
        st->bound_docs = st->bound_pairs = st->bound_candidates = st->bound_doc_nnz = st->bound_cand_nnz = 0;
        st->bound_visits = st->bound_own_dots = 0;
        st->objective = 0.0;
        st->assign_ms = st->assign_kernel_ms = st->screen_ms = st->index_build_seconds = 0.0;
        st->screen_launches = 0;
        for (auto& a : sa) {  // device order: a fixed association
            st->n_reassigned += a.n_reassigned;
            st->dot_products += a.dot_products;
            st->gpu_dot_products += a.gpu_dot_products;
            st->n_rescan += a.n_rescan;
            st->n_exact += a.n_exact;
            st->index_queries += a.index_queries;
            st->candidates_total += a.candidates_total;
            st->bound_docs += a.bound_docs;
            st->bound_pairs += a.bound_pairs;
            st->bound_candidates += a.bound_candidates;
            st->bound_doc_nnz += a.bound_doc_nnz;
            st->bound_cand_nnz += a.bound_cand_nnz;
            st->bound_visits += a.bound_visits;
            st->bound_own_dots += a.bound_own_dots;
            st->objective += a.objective;
            st->assign_ms = std::max(st->assign_ms, a.assign_ms);
            st->assign_kernel_ms = std::max(st->assign_kernel_ms, a.assign_kernel_ms);
            st->screen_ms = std::max(st->screen_ms, a.screen_ms);
            st->index_build_seconds = std::max(st->index_build_seconds, a.index_build_seconds);
            st->screen_launches = std::max(st->screen_launches, a.screen_launches);
        }
    }

    std::vector<int> devs_;
    std::vector<std::unique_ptr<Engine>> engs_;
    std::unique_ptr<DevicePool> pool_;
    std::vector<cudaEvent_t> ev_moved_, ev_delta_;
    std::vector<int64_t> off_;
    std::vector<double> lambdas_;
    sskm_run_config cfg_{};
    int64_t n_ = 0;
    uint32_t k_ = 0;
    bool configured_ = false, state_ = false;
};

}  // namespace sskm_b200
