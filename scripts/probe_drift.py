"""Probe (c1, baseline): per iteration, the drift distribution of the centroid
columns and, for a document sample, the gap between the best and second-best
exact similarity — how many documents a drift bound (Hamerly-style) could skip.
Also prints the per-iteration screen statistics (theta, pairs, candidates)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
stats_only = "--stats-only" in sys.argv
data = S.corpus(cfg)
k = cfg.k
eng = P.Engine(0)
eng.upload(data)
eng.configure(k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, k, 0))
rng = np.random.default_rng(3)
docs = np.sort(rng.choice(data.n_docs, 4000 if not stats_only else 1, replace=False))
X = np.zeros((len(docs), data.dims if not stats_only else 1), np.float32)
xn = np.zeros(len(docs))
for q, i in enumerate(docs if not stats_only else []):
    b, e = data.indptr[i], data.indptr[i + 1]
    X[q, data.indices[b:e]] = data.values[b:e]
    xn[q] = np.linalg.norm(data.values[b:e].astype(np.float64))
prev = eng.get_centroids() if not stats_only else None
for it in range(1, iters + 1):
    t0 = time.perf_counter()
    st = eng.step()
    if stats_only:
        print(json.dumps({"it": it, "ms": st.update_ms + st.assign_ms, "upd": st.update_ms, "asg": st.assign_ms,
                          "screen": st.screen_ms, "theta": st.bound_theta, "moved": st.n_moved, "own": st.bound_own_dots,
                          "reassigned": st.n_reassigned, "recomputed": st.n_recomputed, "exact": st.n_exact,
                          "skip_docs": st.skip_docs, "skip_ms": st.skip_ms,
                          "launches": st.screen_launches, "wall": time.perf_counter() - t0,
                          "pairs": st.bound_pairs, "doc_nnz": st.bound_doc_nnz, "visits": st.bound_visits,
                          "cand": st.bound_candidates, "cand_nnz": st.bound_cand_nnz,
                          "alg_bytes": 8 * st.bound_pairs + 16 * st.bound_doc_nnz + 36 * st.bound_visits
                                       + 4 * st.bound_cand_nnz + 4 * st.bound_own_nnz + 68 * st.bound_visits}), flush=True)
        continue
    ct = eng.get_centroids()
    d = np.sqrt(((ct.astype(np.float64) - prev) ** 2).sum(0))
    prev = ct.astype(np.float64)
    sims = X @ ct  # fp32 approx is fine for the gap distribution
    top2 = -np.partition(-sims, 1, axis=1)[:, :2]
    gap = top2[:, 0] - top2[:, 1]
    a, s, _ = eng.get_state()
    dmax = d.max()
    q = np.quantile(d, [0.5, 0.9, 0.99])
    skip1 = np.mean(gap > 2 * xn * dmax)  # next iteration: own can drop by dmax and another rise by dmax
    out = {"it": it, "ms": st.update_ms + st.assign_ms, "upd": st.update_ms, "asg": st.assign_ms, "screen": st.screen_ms,
           "theta": st.bound_theta, "pairs_per_doc": st.bound_pairs / data.n_docs,
           "cand_per_doc": st.bound_candidates / data.n_docs, "own": st.bound_own_dots, "moved": st.n_moved,
           "reassigned": st.n_reassigned, "skip_docs": st.skip_docs, "skip_ms": st.skip_ms, "recomputed": st.n_recomputed, "exact": st.n_exact,
           "drift_max": float(dmax), "drift_q50_90_99": [float(x) for x in q],
           "gap_q10_50": [float(x) for x in np.quantile(gap, [0.1, 0.5])], "skip_frac_dmax": float(skip1)}
    for qq in (0.5, 0.9, 0.99):
        out[f"skip_frac_drift_q{int(qq*100)}"] = float(np.mean(gap > 2 * xn * np.quantile(d, qq)))
    print(json.dumps(out), flush=True)
