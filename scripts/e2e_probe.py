import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
cfg = S.CONFIGS["c1"]; data = S.corpus(cfg); seeds = S.init_seeds(data.n_docs, cfg.k, 0)
for rep in range(3):
    t = {}; t0 = time.perf_counter()
    e = P.Engine(0); t["open"] = time.perf_counter() - t0
    t1 = time.perf_counter(); e.upload(data); t["upload"] = time.perf_counter() - t1
    t1 = time.perf_counter(); e.configure(cfg.k, conv_sq_dist=1e-300, max_iters=30); t["configure"] = time.perf_counter() - t1
    t1 = time.perf_counter(); e.init_from_seeds(seeds); t["init"] = time.perf_counter() - t1
    t1 = time.perf_counter(); its, stop = e.run(); t["run30"] = time.perf_counter() - t1
    t1 = time.perf_counter(); a, s, _ = e.get_state(); t["download"] = time.perf_counter() - t1
    t1 = time.perf_counter(); e.close(); t["close"] = time.perf_counter() - t1
    print(json.dumps({k: round(v, 4) for k, v in t.items()}), flush=True)
