"""One c1 setup + a few baseline iterations, for ncu captures of the assign tiles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
data = S.corpus(cfg)
eng = P.Engine(0)
eng.upload(data)
eng.configure(cfg.k, mode=os.environ.get("SSKM_MODE", "baseline"), conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, cfg.k, 0))
for _ in range(iters):
    st = eng.step()
print("ok", st.assign_kernel_ms)
