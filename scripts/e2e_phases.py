"""Wall-clock phases of the public cluster() path on c1 (upload, configure, seeding, iterations, download)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
cfg = S.CONFIGS["c1"]
data = S.corpus(cfg)
seeds = S.init_seeds(data.n_docs, cfg.k, 0)
for rep in range(2):
    t = [time.perf_counter()]
    eng = P.Engine(0); eng.upload(data); eng.synchronize(); t.append(time.perf_counter())
    eng.configure(cfg.k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6); eng.synchronize(); t.append(time.perf_counter())
    eng.init_from_seeds(seeds); eng.synchronize(); t.append(time.perf_counter())
    for _ in range(30): eng.step()
    eng.synchronize(); t.append(time.perf_counter())
    a, s_, _ = eng.get_state(); t.append(time.perf_counter())
    eng.close()
    names = ["upload", "configure", "seed", "30 iterations", "download"]
    print(json.dumps({n: round((t[i + 1] - t[i]) * 1e3, 2) for i, n in enumerate(names)}), flush=True)
