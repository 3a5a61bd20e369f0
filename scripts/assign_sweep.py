"""Sweep assign-kernel scheduling knobs on c1 (baseline full scans); prints ms/iteration."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
data = S.corpus(cfg)
seeds = S.init_seeds(data.n_docs, cfg.k, 0)
variants = [dict(SSKM_SCREEN="0", SSKM_TILE_BYTES=str(128 << 20), SSKM_ORDER="1", SSKM_UNROLL="16")]
variants += [dict(SSKM_SCREEN="1", SSKM_SCREEN_KIND="1", SSKM_ORDER=str(o), SSKM_FUSE_RESOLVE=str(f)) for o in (0, 1) for f in (0, 1)]
ref_a = None
for v in variants:
    os.environ.update(v)
    eng = P.Engine(0)
    eng.upload(data)
    eng.configure(cfg.k, mode="baseline", conv_sq_dist=1e-300, max_iters=10**6)
    eng.init_from_seeds(seeds)
    for _ in range(3):
        eng.step()
    eng.timer_record(0)
    sts = [eng.step() for _ in range(5)]
    eng.timer_record(1)
    ms = eng.timer_elapsed(0, 1) / 5
    a, s, _ = eng.get_state()
    same = None
    if ref_a is None:
        ref_a, ref_s = a, s
    else:
        same = bool(np.array_equal(a, ref_a) and np.array_equal(s, ref_s))
    print(json.dumps(dict(v, n_exact=int(np.mean([x.n_exact for x in sts])), ms_iter=round(ms, 3), assign_kernel_ms=round(float(np.mean([x.assign_kernel_ms for x in sts])), 3),
                          update_ms=round(float(np.mean([x.update_ms for x in sts])), 3), screen_ms=round(float(np.mean([x.screen_ms for x in sts])), 3), same_as_first=same)), flush=True)
    eng.close()
