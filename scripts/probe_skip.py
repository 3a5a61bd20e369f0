"""Probe (c1, baseline): how many documents a per-document upper bound on the
best OTHER similarity, kept from the last screen and grown by the centroid
drift, would let the next assign skip. The bound is the one the bound screen
certifies: max over clusters j != own of (high part of x·c_j) + min(Σ|x_t|·L_t,
θ·‖x‖₁), for several θ. Prints, per θ, quantiles of (own − U) and the skip
fraction against the next iteration's max drift."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S

cfg = S.CONFIGS["c1"]
data = S.corpus(cfg)
k = cfg.k
eng = P.Engine(0)
eng.upload(data)
eng.configure(k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, k, 0))
rng = np.random.default_rng(5)
docs = np.sort(rng.choice(data.n_docs, 3000, replace=False))
for it in range(1, 31):
    eng.step()
    if it not in (5, 10, 20, 29):
        continue
    ct = eng.get_centroids().astype(np.float64)
    a, s, _ = eng.get_state()
    eng_next = None
    # drift to the next iteration
    eng.step()
    ct2 = eng.get_centroids().astype(np.float64)
    dmax = float(np.sqrt(((ct2 - ct) ** 2).sum(0)).max())
    a2, s2, _ = eng.get_state()
    res = {"it": it, "dmax_next": dmax}
    for theta in (0.002, 0.005, 0.01, 0.02, 0.05):
        hi = np.where(np.abs(ct) >= theta, ct, 0.0)
        lo_abs = np.where(np.abs(ct) < theta, np.abs(ct), 0.0)
        L = lo_abs.max(1)
        margins = []
        for i in docs:
            b, e = data.indptr[i], data.indptr[i + 1]
            t = data.indices[b:e]
            x = data.values[b:e].astype(np.float64)
            h = x @ hi[t, :]
            h[a[i]] = -np.inf
            lowb = min(float(np.abs(x) @ L[t]), theta * float(np.abs(x).sum()))
            U = h.max() + lowb
            margins.append(s[i] - U)
        m = np.array(margins)
        res[f"theta={theta}"] = {"q10_50_90": [float(v) for v in np.quantile(m, [0.1, 0.5, 0.9])],
                                 "skip_next": float(np.mean(m > dmax)),
                                 "skip_next_q99drift": None}
    print(json.dumps(res), flush=True)
