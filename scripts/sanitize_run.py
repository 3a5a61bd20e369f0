"""A small run of every kernel family under compute-sanitizer (tests/test_gpu_sanitizer.py):
seed assignment (postings screen), bound screen (one tile and the hash pass), drift
bound, kept postings, NCC passes, the ncc+index replay and the multi-device delta."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S

for n, d, kt, k, mode in [(3000, 2048, 12, 24, "baseline"), (3000, 2048, 12, 24, "ncc+index"),
                          (4000, 4096, 60, 2100, "baseline")]:
    m = S.generate(n, d, kt, 40.0, seed=2)
    seeds = S.init_seeds(m.n_docs, k, 0)
    r = P.cluster(m, k, mode=mode, init_seeds=seeds, conv_sq_dist=1e-300, max_iters=6,
                  index_activation_threshold=2)
    print(mode, k, len(r.iterations), r.objective)
mm = P.MultiEngine([0, 0])
m = S.generate(3000, 2048, 12, 40.0, seed=3)
mm.upload(m)
mm.configure(24, mode="ncc", conv_sq_dist=1e-300, max_iters=6)
mm.init_from_seeds(S.init_seeds(m.n_docs, 24, 0))
for _ in range(5):
    mm.step()
print("multi ok")
