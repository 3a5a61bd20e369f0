"""GPU: the multi-device context (sskm_multi_*, cluster(devices=...)).

One host thread drives the listed devices; every device applies every shard's
moved rows to its own exact sums through peer memory. Listing device 0 twice
gives two shards (two engines, two streams) on one B200: the peer reads are
then same-device reads and no kernel ever waits on another, but the whole
sharded path runs — cross-shard delta application, cross-shard repair,
device-ordered counters. Its trajectory must equal a single-GPU run bit for bit.
"""
import numpy as np
import pytest

import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
from tests.test_gpu_distributed import ITERS, _cfg, _stats, corpus_and_seeds

pytestmark = pytest.mark.gpu


def single_trace(data, seeds, mode, iters=ITERS):
    eng = P.Engine(0)
    eng.upload(data)
    eng.configure(len(seeds), **_cfg(mode))
    eng.init_from_seeds(seeds)
    out = []
    for _ in range(iters):
        st = eng.step()
        a, s, _ = eng.get_state()
        out.append((a, s, eng.get_centroids(), _stats(st)))
    eng.close()
    return out


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("mode", ["baseline", "ncc", "ncc+index"])
def test_multi_device_equals_single(devices, mode):
    data, seeds = corpus_and_seeds()
    single = single_trace(data, seeds, mode)
    m = P.MultiEngine(devices)
    m.upload(data)
    m.configure(len(seeds), **_cfg(mode))
    m.init_from_seeds(seeds)
    assert single[0][3][1] == 1  # iteration 1 repairs a cluster (its seed is duplicated on another shard)
    for t in range(ITERS):
        st = m.step()
        a, s = m.get_state()
        a1, s1, c1, x1 = single[t]
        assert np.array_equal(a, a1), t
        assert np.array_equal(s, s1), t
        assert np.array_equal(m.get_centroids(), c1), t
        x = _stats(st)
        assert x[:7] == x1[:7], (t, x, x1)
        assert x[7] == pytest.approx(x1[7], rel=1e-12)
    assert m.launch_count() > 0
    m.close()


def test_cluster_devices_bitwise():
    """cluster(devices=[0]) and devices=[0, 0] equal cluster(device=0) bit for bit."""
    m = S.generate(8000, 4096, 16, 50.0, seed=5)
    seeds = S.init_seeds(m.n_docs, 32, 0)
    kw = dict(mode="ncc", init_seeds=seeds, conv_sq_dist=1e-300, max_iters=12, return_centroids=True)
    r0 = P.cluster(m, 32, **kw)
    for devs in ([0], [0, 0]):
        r = P.cluster(m, 32, devices=devs, **kw)
        assert np.array_equal(r.assignments, r0.assignments)
        assert np.array_equal(r.sims, r0.sims)
        assert np.array_equal(r.centroids, r0.centroids)
        assert len(r.iterations) == len(r0.iterations) and r.stop_reason == r0.stop_reason
        assert [it.dot_products for it in r.iterations] == [it.dot_products for it in r0.iterations]
        assert r.objective == pytest.approx(r0.objective, rel=1e-12)
        if devs == [0]:
            assert r.objective == r0.objective


def test_multi_errors():
    with pytest.raises(ValueError, match="init_seeds"):
        P.cluster(S.generate(300, 256, 4, 10.0, seed=1), 4, devices=[0])
    with pytest.raises(ValueError):
        P.MultiEngine([])
