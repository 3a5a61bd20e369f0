"""CPU: the multi-GPU driver's host logic over torch.distributed/gloo at
world_size 2. A numpy shard engine with the engine's exchange
semantics (fixed-point replicated sums, per-document assign) stands in for the
GPU so that sharding, the all-gather of moved rows, the cross-rank
empty-cluster repair replay and the statistics reductions are exercised; the
2-rank trajectory must equal the 1-rank trajectory bit for bit, and both must
agree with the reference oracle."""
import math
import os
import socket

import numpy as np
import pytest
import torch

from paper_2108_00895_b200 import distributed as D
from paper_2108_00895_b200 import synthetic as S
from paper_2108_00895_b200.api import IterationStats

NONE = 0xFFFFFFFF


class NumpyShard:
    def __init__(self, shard, offset, n_total, k):
        self.m, self.off, self.n_total, self.k = shard, offset, n_total, k
        self.d = shard.dims
        self.K = 62 - int(math.ceil(math.log2(max(n_total, 2))))
        self.S = np.zeros((self.d, k), np.int64)
        self.CT = np.zeros((self.d, k), np.float32)
        n = shard.n_docs
        self.a = np.zeros(n, np.int64)
        self.a_sum = np.full(n, -1, np.int64)
        self.sims = np.full(n, -2.0)
        self.iteration = 0

    def rows(self, gids):
        out = []
        for g in gids:
            i = int(g) - self.off
            b, e = self.m.indptr[i], self.m.indptr[i + 1]
            out.append((self.m.indices[b:e].copy(), self.m.values[b:e].copy()))
        return out

    def local_counts(self):
        return np.bincount(self.a, minlength=self.k).astype(np.int64)

    def local_candidates(self, m):
        o = np.lexsort((np.arange(len(self.sims)), self.sims + 0.0))[:m]
        return self.sims[o], o.astype(np.int64) + self.off, self.a[o].astype(np.uint32)

    def move_doc(self, gid, c):
        self.a[int(gid) - self.off] = c

    def moved_pack(self):
        mv = np.nonzero(self.a != self.a_sum)[0]
        lens = np.diff(self.m.indptr)[mv]
        idx = np.concatenate([self.m.indices[self.m.indptr[i]:self.m.indptr[i + 1]] for i in mv]) if len(mv) else []
        val = np.concatenate([self.m.values[self.m.indptr[i]:self.m.indptr[i + 1]] for i in mv]) if len(mv) else []
        t = lambda x, dt: torch.as_tensor(np.asarray(x, dt))  # noqa: E731
        return (t(self.a_sum[mv], np.int32), t(self.a[mv], np.int32), t(lens, np.int32), t(idx, np.int32),
                t(val, np.float32))

    def update_apply(self, old, new, lens, idx, val, repaired):
        old, new, lens = old.numpy().astype(np.int64), new.numpy().astype(np.int64), lens.numpy()
        idx, val = idx.numpy(), val.numpy()
        touched = np.zeros(self.k, bool)
        p = 0
        for o, nw, ln in zip(old, new, lens):
            t, x = idx[p:p + ln], val[p:p + ln]
            q = np.rint(np.ldexp(x.astype(np.float64), self.K)).astype(np.int64)
            self.S[t, nw] += q
            touched[nw] = True
            if o != -1:
                self.S[t, o] -= q
                touched[o] = True
            p += ln
        self.a_sum = self.a.copy()
        self.iteration += 1
        drift = np.zeros(self.k)
        for j in np.nonzero(touched)[0]:
            v = self.S[:, j].astype(np.float64)
            inv = 1.0 / math.sqrt(float(np.dot(v, v)))
            c = (v * inv).astype(np.float32)
            drift[j] = float(np.sum((c.astype(np.float64) - self.CT[:, j].astype(np.float64)) ** 2))
            self.CT[:, j] = c
        max_drift = 0.0 if self.iteration <= 1 else float(drift.max())
        return IterationStats(iteration=self.iteration, max_sq_drift=max_drift, n_repaired=len(repaired),
                              n_recomputed=int(touched.sum()))

    def init_from_rows(self, rptr, idx, val):
        self.CT[:] = 0
        for j in range(self.k):
            self.CT[idx[rptr[j]:rptr[j + 1]], j] = val[rptr[j]:rptr[j + 1]]
        self.a[:] = 0
        self.sims[:] = -2.0
        self.a_sum[:] = -1
        self.S[:] = 0
        self.iteration = 0
        self.assign()

    def assign(self):
        a0 = self.a.copy()
        ct = self.CT.astype(np.float64)
        for i in range(self.m.n_docs):
            b, e = self.m.indptr[i], self.m.indptr[i + 1]
            acc = np.zeros(self.k)
            for t, x in zip(self.m.indices[b:e], self.m.values[b:e]):
                acc = acc + float(x) * ct[t]  # ascending-term fp64 accumulation
            j = int(np.argmax(acc))  # first max = lowest id on ties
            self.a[i], self.sims[i] = (j, acc[j]) if acc[j] > -2.0 else (0, -2.0)
        obj = 0.0
        for s in self.sims:
            obj += s
        return IterationStats(n_reassigned=int(np.sum(self.a != a0)), objective=obj,
                              n_unchanged_centroids=0, gpu_dot_products=self.k * self.m.n_docs,
                              dot_products=self.k * self.m.n_docs)


def corpus_with_duplicate_seeds():
    m = S.generate(240, 400, 4, 20.0, seed=5)
    rows = [(m.indices[m.indptr[i]:m.indptr[i + 1]], m.values[m.indptr[i]:m.indptr[i + 1]]) for i in range(m.n_docs)]
    rows[150] = rows[3]  # seed 150 duplicates seed 3 -> its cluster starts empty (repair)
    ptr = np.zeros(len(rows) + 1, np.int64)
    ptr[1:] = np.cumsum([len(r[0]) for r in rows])
    from paper_2108_00895_b200.api import CorpusMatrix
    return CorpusMatrix.from_csr(ptr, np.concatenate([r[0] for r in rows]), np.concatenate([r[1] for r in rows]),
                                 m.dims), np.array([3, 150, 20, 200, 90, 160], np.uint32)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data, seeds = corpus_with_duplicate_seeds()
        shard, off = D.shard_corpus(data, rank, world)
        comm = D.Comm(rank, world, torch.device("cpu"))
        km = D.DistributedKMeans(NumpyShard(shard, off, data.n_docs, len(seeds)), comm, data.n_docs, len(seeds),
                                 conv_sq_dist=1e-300)
        km.init_from_seeds(seeds)
        trace = []
        for _ in range(6):
            st = km.step()
            a = comm.all_gather_var(torch.as_tensor(km.s.a))
            s = comm.all_gather_var(torch.as_tensor(km.s.sims))
            trace.append((torch.cat(a).numpy(), torch.cat(s).numpy(), km.s.CT.copy(),
                          (st.n_reassigned, st.n_repaired, st.n_moved, st.max_sq_drift, st.objective, st.dot_products)))
        if rank == 0:
            q.put(trace)
    finally:
        dist.destroy_process_group()


def _run(world):
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.fixture(scope="module")
def traces():
    return _run(1), _run(2)


def test_two_ranks_equal_one_rank_bitwise(traces):
    one, two = traces
    assert len(one) == len(two)
    for (a1, s1, c1, st1), (a2, s2, c2, st2) in zip(one, two):
        assert np.array_equal(a1, a2)
        assert np.array_equal(s1, s2)
        assert np.array_equal(c1, c2)  # integer sums: centroids independent of the rank count
        assert st1[:3] == st2[:3] and st1[3] == st2[3] and st1[5] == st2[5]
        assert st1[4] == pytest.approx(st2[4], rel=1e-12)


def test_cross_rank_repair_happened(traces):
    one, _ = traces
    assert one[0][3][1] == 1  # the duplicated seed's cluster was refilled on iteration 1


def test_matches_oracle_trajectory(traces):
    from oracle import oracle as O

    data, seeds = corpus_with_duplicate_seeds()
    c = O.Corpus(data.indptr, data.indices, data.values.astype(np.float64), data.dims)
    r = O.run_seeded(c, len(seeds), seeds, conv_sq_dist=1e-300, max_iters=6, kind="port", record=True)
    one, _ = traces
    for (a, s, _, _), (ra, rs, _) in zip(one, r["trace"]):
        assert np.mean(a == ra) >= 0.99
        np.testing.assert_allclose(s[a == ra], rs[a == ra], atol=1e-6)


def test_replay_repair_needs_longer_lists_when_truncated():
    counts = np.array([0, 3, 2], np.int64)
    # rank 0 returned a truncated list whose candidates are all ineligible
    cand0 = (np.array([0.1]), np.array([5]), np.array([2], np.uint32))
    cand1 = (np.array([0.2, 0.3]), np.array([7, 8]), np.array([2, 1], np.uint32))
    assert D.replay_repair(np.array([0, 3, 1]), [cand0, cand1], [10, 2], 1) is None
    moves = D.replay_repair(counts, [cand0, cand1], [1, 2], 1)
    assert moves == [(5, 2, 0)]


def test_single_rank_collectives_are_identities():
    """A collective over one rank is the identity: Comm(world=1) answers without
    touching torch.distributed (no process group exists here) and in the shapes
    the multi-rank paths return."""
    c = D.Comm(0, 1, torch.device("cpu"))
    x = np.arange(5, dtype=np.int64)
    assert np.array_equal(c.all_reduce_i64(x), x)
    assert c.all_reduce_f64_max(2.5) == 2.5
    assert c.all_gather_f64(1.25) == [1.25]
    t = torch.arange(7, dtype=torch.int32)
    (g,) = c.all_gather_var(t)
    assert torch.equal(g, t)
    a, b = c.all_gather_var_multi([t, t.float()])
    assert len(a) == 1 and torch.equal(a[0], t) and torch.equal(b[0], t.float())
    v = c.all_gather_f64_vec(np.array([1.0, 2.0]))
    assert v.shape == (1, 2) and v[0, 1] == 2.0
    assert c.all_gather_object({"k": 1}) == [{"k": 1}]
