"""Distribution of the high-list lengths a document's terms see (c1, baseline, iteration 10):
for each length c, the share of document nonzeros whose term has c high pairs, and the share of
all (doc-weighted) pairs in lists of at most c."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
data = S.corpus(cfg)
eng = P.Engine(0); eng.upload(data)
eng.configure(cfg.k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, cfg.k, 0))
for it in range(10): st = eng.step()
theta = st.bound_theta
ct = eng.get_centroids()
cnt = (np.abs(ct) >= theta).sum(1).astype(np.int64)
df = np.bincount(data.indices, minlength=data.dims).astype(np.int64)
nnz = df.sum(); pairs = (df * cnt).sum()
print(json.dumps({"theta": theta, "pairs_per_doc": pairs / data.n_docs, "nnz_per_doc": nnz / data.n_docs}))
edges = [0, 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 64, 128, 10**9]
for lo, hi in zip(edges[:-1], edges[1:]):
    m = (cnt >= lo) & (cnt < hi)
    print(f"len [{lo},{hi}): nnz share {df[m].sum()/nnz:.3f}  pair share {(df[m]*cnt[m]).sum()/pairs:.3f}")
for P2 in (1, 2, 4):
    rem = (df * np.maximum(cnt - P2, 0)).sum()
    print(f"direct {P2}: remainder pairs/doc {rem/data.n_docs:.1f} ({rem/pairs:.3f} of all)")
