"""Simulation (c1, baseline): how many documents a per-cluster-GROUP drift bound would keep
out of the screen. Per sampled document: U[g] = bound on its similarity to the clusters of
group g (j % G) from its last screen, grown by ||x||·(max drift of the group's clusters) per
update; the document skips when its exact own similarity beats every group's bound.
G = 1 is the engine's current global bound."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S

cfg = S.CONFIGS["c1"]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
data = S.corpus(cfg)
k = cfg.k
eng = P.Engine(0)
eng.upload(data)
eng.configure(k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, k, 0))
rng = np.random.default_rng(3)
docs = np.sort(rng.choice(data.n_docs, 3000, replace=False))
X = np.zeros((len(docs), data.dims), np.float32)
xn = np.zeros(len(docs))
for q, i in enumerate(docs):
    b, e = data.indptr[i], data.indptr[i + 1]
    X[q, data.indices[b:e]] = data.values[b:e]
    xn[q] = np.linalg.norm(data.values[b:e].astype(np.float64))
GS = [1, 16, 32, 64, 128, 1000]
SLACK = 0.015
state = {G: dict(U=None, acc=None) for G in GS}
prev = eng.get_centroids().astype(np.float64)
a_prev = None
n = len(docs)
for it in range(1, iters + 1):
    eng.step()
    ct = eng.get_centroids()
    d = np.sqrt(((ct.astype(np.float64) - prev) ** 2).sum(0))
    prev = ct.astype(np.float64)
    sims = (X @ ct).astype(np.float64)
    a_all, _, _ = eng.get_state()
    a = a_all[docs].astype(np.int64)
    out = {"it": it, "dmax": float(d.max())}
    for G in GS:
        st = state[G]
        grp = np.arange(k) % G
        if st["U"] is None or it <= 2:
            full = np.ones(n, bool)
            own_only = np.zeros(n, bool)
        else:
            dg = np.zeros(G)
            np.maximum.at(dg, grp, d)
            # exclude the own cluster's drift from its group? (its column is handled by the own dot):
            st["acc"] += xn[:, None] * dg[None, :] * (1 + 1e-9)
            s_own = sims[np.arange(n), a_prev]
            bound = (st["U"] + st["acc"]).max(1)
            ok = s_own > bound
            changed_own = d[a_prev] > 0
            full = ~ok
            own_only = ok & changed_own
        # screened documents refresh their bounds from the current similarities
        if full.any():
            if st["U"] is None:
                st["U"] = np.zeros((n, G)); st["acc"] = np.zeros((n, G))
            idx = np.where(full)[0]
            sm = sims[idx].copy()
            sm[np.arange(len(idx)), a[idx]] = -1.0
            U = np.full((len(idx), G), 0.0)
            for g in range(G):
                cols = np.where(grp == g)[0]
                U[:, g] = np.maximum(sm[:, cols].max(1), 0.0) + SLACK
            st["U"][idx] = U
            st["acc"][idx] = 0.0
        # a document that moved gets no bound (the engine sets U = inf): force a screen next time
        if a_prev is not None:
            mv = a != a_prev
            st["U"][mv] = 9.0
        out[f"G{G}"] = {"full": round(float(full.mean()), 3), "own_only": round(float(own_only.mean()), 3)}
    a_prev = a
    print(json.dumps(out), flush=True)
