"""GPU: the document-sharded driver with the real CUDA engine.

Two ranks share one B200 through torch.distributed/gloo (collectives on the
CPU, so no kernel ever waits on another rank); their trajectory must equal a
single-GPU Engine run bit for bit — assignments, sims, centroids and the
reference's statistics — including the cross-rank empty-cluster repair.
"""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import distributed as D
from paper_2108_00895_b200 import synthetic as S

pytestmark = pytest.mark.gpu

ITERS = 6


def corpus_and_seeds():
    m = S.generate(6000, 4096, 12, 50.0, seed=17)
    rows = [(m.indices[m.indptr[i]:m.indptr[i + 1]], m.values[m.indptr[i]:m.indptr[i + 1]]) for i in range(m.n_docs)]
    rows[4000] = rows[10]  # duplicated seed on the other shard -> cross-rank repair on iteration 1
    ptr = np.zeros(len(rows) + 1, np.int64)
    ptr[1:] = np.cumsum([len(r[0]) for r in rows])
    data = P.CorpusMatrix.from_csr(ptr, np.concatenate([r[0] for r in rows]), np.concatenate([r[1] for r in rows]),
                                   m.dims)
    seeds = S.init_seeds(data.n_docs, 24, 0)
    seeds[0], seeds[1] = 10, 4000
    return data, seeds


def _cfg(mode):
    # ncc+index: a low activation threshold so the replayed index is active
    return dict(mode=mode, conv_sq_dist=1e-300, index_activation_threshold=2 if mode == "ncc+index" else 100)


def _stats(st):
    return (st.n_reassigned, st.n_repaired, st.dot_products, st.index_queries, st.candidates_total,
            bool(st.index_active), st.max_sq_drift, st.objective)


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data, seeds = corpus_and_seeds()
        shard, off = D.shard_corpus(data, rank, world)
        gs = D.GPUShard(shard, off, data.n_docs, len(seeds), device=0, **_cfg(mode))
        comm = D.Comm(rank, world, torch.device("cpu"))
        km = D.DistributedKMeans(gs, comm, data.n_docs, len(seeds), mode=mode, conv_sq_dist=1e-300)
        km.init_from_seeds(seeds)
        trace = []
        for _ in range(ITERS):
            st = km.step()
            a, s, _ = gs.get_state()
            ag = torch.cat(comm.all_gather_var(torch.as_tensor(a.astype(np.int64)))).numpy()
            sg = torch.cat(comm.all_gather_var(torch.as_tensor(s))).numpy()
            trace.append((ag, sg, gs.get_centroids(), _stats(st)))
        if rank == 0:
            q.put(trace)
    finally:
        dist.destroy_process_group()


def run_sharded(world, mode):
    import torch.multiprocessing as mp

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("mode", ["baseline", "ncc", "ncc+index"])
def test_two_shards_equal_single_gpu(mode):
    data, seeds = corpus_and_seeds()
    eng = P.Engine(0)
    eng.upload(data)
    eng.configure(len(seeds), **_cfg(mode))
    eng.init_from_seeds(seeds)
    single = []
    for _ in range(ITERS):
        st = eng.step()
        a, s, _ = eng.get_state()
        single.append((a.astype(np.int64), s, eng.get_centroids(), _stats(st)))
    eng.close()
    two = run_sharded(2, mode)
    assert single[0][3][1] == 1  # repair happened (duplicated seed on the other shard)
    for t, ((a1, s1, c1, x1), (a2, s2, c2, x2)) in enumerate(zip(single, two)):
        assert np.array_equal(a1, a2), t
        assert np.array_equal(s1, s2), t
        assert np.array_equal(c1, c2), t
        assert x1[:7] == x2[:7], (t, x1, x2)
        assert x2[7] == pytest.approx(x1[7], rel=1e-12)
    if mode == "ncc+index":
        assert any(x[5] for _, _, _, x in single)
