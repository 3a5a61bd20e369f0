"""Per-config timing probe: a few iterations of each BASELINE config on 1 GPU."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
name, mode, iters = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = S.CONFIGS[name]
t0 = time.time(); data = S.corpus(cfg); tg = time.time() - t0
eng = P.Engine(0)
t0 = time.time(); eng.upload(data); eng.configure(cfg.k, mode=mode, conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, cfg.k, 0)); ti = time.time() - t0
print(json.dumps(dict(config=name, mode=mode, n=data.n_docs, nnz=data.nnz, gen_s=round(tg, 1), init_s=round(ti, 2))), flush=True)
for it in range(1, iters + 1):
    eng.timer_record(0); st = eng.step(); eng.timer_record(1)
    print(json.dumps(dict(iter=it, ms=round(eng.timer_elapsed(0, 1), 2), update_ms=round(st.update_ms, 2),
                          assign_ms=round(st.assign_ms, 2), screen_ms=round(st.screen_ms, 2), tiles=st.screen_launches,
                          n_changed=st.n_changed, density=round(st.centroid_density, 4), n_reassigned=st.n_reassigned, n_exact=st.n_exact,
                          n_rescan=st.n_rescan, n_repaired=st.n_repaired, dots=st.dot_products,
                          bound=dict(theta=round(st.bound_theta, 5), pairs=st.bound_pairs, cands=st.bound_candidates,
                                     own=st.bound_own_dots, docs=st.bound_docs),
                          **({} if not st.index_active else dict(idx_build_ms=round(st.index_build_seconds * 1e3, 2), idx_queries=st.index_queries, idx_cands=st.candidates_total)))), flush=True)
if os.environ.get("PROBE_PAIRS"):
    pairs = eng.postings_work()
    print(json.dumps(dict(postings_pairs=pairs, mean_dfc_per_entry=pairs / data.nnz,
                          density_weighted_ratio=pairs / (data.nnz * cfg.k))), flush=True)
