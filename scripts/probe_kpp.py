"""k-means++ seeding time (device-resident rounds) on a BASELINE corpus."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
data = S.corpus(cfg)
eng = P.Engine(0)
eng.upload(data)
eng.configure(cfg.k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6)
t0 = time.perf_counter()
seeds = eng.init_kmeanspp(0)
print(json.dumps({"config": cfg.name, "k": cfg.k, "n": data.n_docs, "kmeanspp_s": time.perf_counter() - t0,
                  "env_host": os.environ.get("SSKM_KPP_HOST", "0"), "first_seeds": seeds[:5].tolist()}), flush=True)
