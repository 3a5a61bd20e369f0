"""Centroid density on a config: per-term cluster counts df_c(t) and the work a
postings (sparse-centroid) screen would do vs the dense scan."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
data = S.corpus(cfg)
eng = P.Engine(0); eng.upload(data)
eng.configure(cfg.k, mode="ncc", conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, cfg.k, 0))
for it in range(1, 13):
    st = eng.step()
    if it in (1, 2, 3, 5, 8, 12):
        ct = eng.get_centroids()
        dfc = np.count_nonzero(ct, axis=1).astype(np.int64)  # clusters per term
        work = int(dfc[data.indices].sum())
        dense = data.nnz * cfg.k
        print(json.dumps(dict(iter=it, density=float(np.count_nonzero(ct)) / ct.size, postings_work_ratio=work / dense,
                              mean_dfc_per_doc_entry=work / data.nnz, n_changed=st.n_changed, n_reassigned=st.n_reassigned,
                              assign_ms=st.assign_ms, update_ms=st.update_ms)), flush=True)
