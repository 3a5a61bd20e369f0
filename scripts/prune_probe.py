"""Probe: how many candidates survive a value-split bound on real c1 centroids.
A_high = X @ C_high (entries >= theta), UB = A_high + theta*||x||_1 (nonneg data),
LB = rowmax(A_high); candidates = #{j : UB_j >= LB}. Also the high-pair fraction."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2108_00895_b200 as P
from paper_2108_00895_b200 import synthetic as S
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = S.CONFIGS[name]
data = S.corpus(cfg)
eng = P.Engine(0); eng.upload(data); eng.configure(cfg.k, conv_sq_dist=1e-300, max_iters=10**6)
eng.init_from_seeds(S.init_seeds(data.n_docs, cfg.k, 0))
for _ in range(4): eng.step()
ct = torch.from_numpy(eng.get_centroids()).cuda()          # d x k fp32
a_cur, s_cur, _ = eng.get_state()
nsub = min(data.n_docs, 200000)
ip = data.indptr[:nsub + 1]
X = torch.sparse_csr_tensor(torch.from_numpy(ip.astype(np.int64)), torch.from_numpy(data.indices[:ip[-1]].astype(np.int64)),
                            torch.from_numpy(data.values[:ip[-1]]), size=(nsub, data.dims)).cuda()
x1 = torch.from_numpy(np.add.reduceat(np.abs(data.values[:ip[-1]]), ip[:-1]).astype(np.float32)).cuda()
nnz_t = torch.from_numpy(np.diff(ip).astype(np.float32)).cuda()
A = (X @ ct)                                             # full fp32 sims
best = A.max(1).values
total_pairs = float((ct != 0).sum())
cnt_x = torch.bincount(torch.from_numpy(data.indices[:ip[-1]].astype(np.int64)).cuda(), minlength=data.dims).float()
nz_per_term = (ct != 0).sum(1).float()
P_full = float((cnt_x * nz_per_term).sum())
for theta in [0.005, 0.01, 0.02, 0.03, 0.05, 0.08]:
    hi = torch.where(ct >= theta, ct, torch.zeros_like(ct))
    Ah = X @ hi
    lb = Ah.max(1).values
    # per-document bound of the low part: theta * ||x||_1 (fp slack ignored in the probe)
    ub = Ah + (theta * x1)[:, None]
    cand = (ub >= lb[:, None]).sum(1).float()
    P_hi = float((cnt_x * (hi != 0).sum(1).float()).sum())
    # tighter: low part bound min(theta*||x||_1, ||x|| * ||c_low||) with ||x|| = 1
    cl = torch.sqrt(((ct - hi) ** 2).sum(0))
    ub2 = Ah + torch.minimum((theta * x1)[:, None], cl[None, :])
    cand2 = (ub2 >= lb[:, None]).sum(1).float()
    print(json.dumps(dict(config=name, theta=theta, hi_pair_frac=round(P_hi / P_full, 4),
                          cand_mean=round(float(cand.mean()), 2), cand_p50=float(cand.median()),
                          cand_p99=float(torch.quantile(cand, 0.99)), cand2_mean=round(float(cand2.mean()), 2),
                          cand2_p99=float(torch.quantile(cand2, 0.99)))), flush=True)
