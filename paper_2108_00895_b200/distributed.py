"""Document-sharded multi-GPU clustering over torch.distributed (NCCL on B200s,
gloo for CPU tests and for several ranks sharing one GPU).

One process per GPU. Documents are sharded in contiguous equal ranges; the
dense centroid matrix Cᵀ and the fixed-point cluster sums are replicated.
Every iteration exchanges only what the reference's loop makes necessary
(engine.cpp:357-416):

  update  1. all-reduce of the local cluster sizes (int64[k]);
          2. empty clusters: every rank contributes its first m documents in
             donor order (lowest cached sim, then lowest global index,
             engine.cpp:156-161); the merged list is replayed through the
             sequential repair rule identically on every rank, and the owner
             rank applies each move;
          3. all-gather of the rows of documents that moved (delta path,
             SURVEY §8e): every rank applies all of them to its replicated
             integer sums, so all ranks hold bit-identical sums and
             renormalise bit-identical centroids with no centroid exchange.
  assign  local; all-reduce of the integer counters, all-gather of the
          objective partials summed in rank order.

Integer sums make the centroids bitwise independent of the number of ranks;
assignments and sims are per-document and identical to a single-GPU run.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from . import _lib
from .api import CorpusMatrix, Engine, IterationStats, make_config
from ._lib import STOP_REASONS, check


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous equal ranges: rank r owns [r·N/p, (r+1)·N/p)."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def shard_corpus(data: CorpusMatrix, rank: int, world: int):
    b, e = shard_range(data.n_docs, rank, world)
    p0, p1 = data.indptr[b], data.indptr[e]
    m = CorpusMatrix.from_csr(data.indptr[b:e + 1] - p0, data.indices[p0:p1], data.values[p0:p1], data.dims)
    return m, b


class GPUShard:
    """The per-rank engine (one CUDA context) behind the driver's interface."""

    def __init__(self, shard: CorpusMatrix, doc_offset: int, n_total: int, k: int, device: int = 0, **cfg):
        import torch

        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.eng = Engine(device)
        self.eng.upload(shard, doc_offset=doc_offset, n_docs_total=n_total)
        self.eng.configure(k, device=device, **cfg)
        self.shard, self.offset, self.k = shard, doc_offset, k
        self.lib = self.eng.lib

    # -- update pieces
    def local_counts(self) -> np.ndarray:
        out = np.zeros(self.k, np.int64)
        check(self.lib.sskm_local_counts(self.eng.h, out))
        return out

    def local_candidates(self, m: int):
        m = int(min(m, self.shard.n_docs))
        s = np.zeros(max(m, 1), np.float64)
        g = np.zeros(max(m, 1), np.int64)
        c = np.zeros(max(m, 1), np.uint32)
        got = C.c_int64()
        check(self.lib.sskm_local_candidates(self.eng.h, m, s, g, c, C.byref(got)))
        n = got.value
        return s[:n], g[:n], c[:n]

    def move_doc(self, gid: int, cluster: int):
        check(self.lib.sskm_move_doc(self.eng.h, int(gid), int(cluster)))

    def moved_pack(self):
        torch = self.torch
        n, nnz = C.c_int64(), C.c_int64()
        check(self.lib.sskm_moved_prepare(self.eng.h, C.byref(n), C.byref(nnz)))
        n, nnz = n.value, nnz.value
        old = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        new = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        lens = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=self.dev)
        val = torch.empty(max(nnz, 1), dtype=torch.float32, device=self.dev)
        check(self.lib.sskm_moved_pack(self.eng.h, old.data_ptr(), new.data_ptr(), lens.data_ptr(), idx.data_ptr(),
                                       val.data_ptr()))
        return old[:n], new[:n], lens[:n], idx[:nnz], val[:nnz]

    def update_apply(self, old, new, lens, idx, val, repaired) -> IterationStats:
        torch = self.torch
        old, new, lens, idx, val = (t.to(self.dev) for t in (old, new, lens, idx, val))
        rptr = torch.zeros(len(lens) + 1, dtype=torch.int64, device=self.dev)
        if len(lens):
            rptr[1:] = torch.cumsum(lens.to(torch.int64), 0)
        rep = np.ascontiguousarray(repaired, np.uint32) if len(repaired) else np.zeros(1, np.uint32)
        # the engine runs on its own non-blocking stream: the gathered rows
        # (produced on torch's / NCCL's stream) must be complete before it reads
        torch.cuda.synchronize(self.dev)
        keep = (old, new, rptr, idx, val)  # noqa: F841 (alive across the call; it synchronises before returning)
        st = _lib.sskm_iteration_stats()
        check(self.lib.sskm_update_apply(self.eng.h, len(lens), old.data_ptr(), new.data_ptr(), rptr.data_ptr(),
                                         idx.data_ptr(), val.data_ptr(), rep, len(repaired), C.byref(st)))
        return IterationStats.from_c(st)

    def init_from_rows(self, rptr, idx, val):
        check(self.lib.sskm_init_from_rows(self.eng.h, np.ascontiguousarray(rptr, np.int64),
                                           np.ascontiguousarray(idx, np.int32) if len(idx) else np.zeros(1, np.int32),
                                           np.ascontiguousarray(val, np.float32) if len(val) else np.zeros(1, np.float32)))

    def assign(self) -> IterationStats:
        return self.eng.assign()

    def get_state(self):
        return self.eng.get_state()

    def get_centroids(self):
        return self.eng.get_centroids()

    def rows(self, gids):
        """Host CSR rows of local documents (seed gathering)."""
        out = []
        for g in gids:
            i = int(g) - self.offset
            b, e = self.shard.indptr[i], self.shard.indptr[i + 1]
            out.append((self.shard.indices[b:e].copy(), self.shard.values[b:e].copy()))
        return out


@dataclass
class Comm:
    """torch.distributed with tensors staged on `dev` (cuda for NCCL, cpu for gloo)."""
    rank: int
    world: int
    dev: object
    group: object = None

    def _d(self):
        import torch.distributed as dist
        return dist

    def all_reduce_i64(self, x: np.ndarray, op="sum") -> np.ndarray:
        if self.world == 1:  # a collective over one rank is the identity: no device round trip
            return np.ascontiguousarray(x, np.int64)
        import torch
        dist = self._d()
        t = torch.as_tensor(np.ascontiguousarray(x, np.int64)).to(self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()

    def all_reduce_f64_max(self, x: float) -> float:
        if self.world == 1:
            return float(x)
        import torch
        dist = self._d()
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def all_gather_f64(self, x: float) -> list:
        if self.world == 1:
            return [float(x)]
        import torch
        dist = self._d()
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [float(o.item()) for o in out]

    def all_gather_var(self, t):
        """All-gather of a 1-D tensor of per-rank length; rank-ordered list."""
        if self.world == 1:
            return [t]
        import torch
        dist = self._d()
        src_dev = t.device
        t = t.to(self.dev)
        n = torch.tensor([t.numel()], dtype=torch.int64, device=self.dev)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        mx = max(max(ns), 1)
        buf = torch.zeros(mx, dtype=t.dtype, device=self.dev)
        buf[: t.numel()] = t
        outs = [torch.zeros_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return [o[:c].to(src_dev) for o, c in zip(outs, ns)]

    def all_gather_var_multi(self, ts):
        """All-gather of several 1-D tensors of per-rank length: one gather of
        all the lengths, then one padded gather per tensor. Returns, per tensor,
        the rank-ordered list."""
        if self.world == 1:
            return [[t] for t in ts]
        import torch
        dist = self._d()
        src = [t.device for t in ts]
        ts = [t.to(self.dev) for t in ts]
        n = torch.tensor([t.numel() for t in ts], dtype=torch.int64, device=self.dev)
        ns = torch.zeros(self.world * len(ts), dtype=torch.int64, device=self.dev)
        dist.all_gather_into_tensor(ns, n, group=self.group)
        ns = ns.view(self.world, len(ts)).cpu().tolist()
        res = []
        for i, t in enumerate(ts):
            mx = max(max(r[i] for r in ns), 1)
            buf = torch.zeros(mx, dtype=t.dtype, device=self.dev)
            buf[: t.numel()] = t
            out = torch.empty(self.world * mx, dtype=t.dtype, device=self.dev)
            dist.all_gather_into_tensor(out, buf, group=self.group)
            out = out.view(self.world, mx)
            res.append([out[r, : ns[r][i]].to(src[i]) for r in range(self.world)])
        return res

    def all_gather_f64_vec(self, x: np.ndarray) -> np.ndarray:
        """[world, len(x)] float64, rank-ordered rows."""
        if self.world == 1:
            return np.ascontiguousarray(x, np.float64).reshape(1, -1)
        import torch
        dist = self._d()
        t = torch.as_tensor(np.ascontiguousarray(x, np.float64)).to(self.dev)
        out = torch.empty(self.world * t.numel(), dtype=torch.float64, device=self.dev)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.view(self.world, -1).cpu().numpy()

    def all_gather_object(self, obj) -> list:
        if self.world == 1:
            return [obj]
        dist = self._d()
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out


def replay_repair(counts: np.ndarray, cand_lists: list, n_locals: list, m: int):
    """Sequential empty-cluster repair (engine.cpp:154-167) over the merged
    candidates of all ranks. Returns [(gid, old, new)] or None when a longer
    candidate list is needed to stay exact."""
    k = len(counts)
    cnt = counts.copy()
    merged = []
    bound = None  # candidates beyond the smallest truncated list's last key are not exact
    for (s, g, c), n_local in zip(cand_lists, n_locals):
        merged += list(zip(s.tolist(), g.tolist(), c.tolist()))
        if len(s) == m and len(s) < n_local:
            last = (s[-1] + 0.0, int(g[-1]))
            bound = last if bound is None or last < bound else bound
    merged.sort(key=lambda x: (x[0] + 0.0, x[1]))  # -0.0 == +0.0, ties -> lowest index
    cur = [c for _, _, c in merged]
    used = [False] * len(merged)
    moves = []
    for j in range(k):
        if cnt[j] != 0:
            continue
        pick = None
        for q, (s, g, _) in enumerate(merged):
            if bound is not None and (s + 0.0, g) > bound:
                return None
            if used[q] or cnt[cur[q]] < 2:
                continue
            pick = q
            break
        if pick is None:
            if bound is None:
                raise RuntimeError("empty-cluster repair found no donor")
            return None
        used[pick] = True
        cnt[cur[pick]] -= 1
        moves.append((merged[pick][1], cur[pick], j))
        cur[pick] = j
        cnt[j] = 1
    return moves


class DistributedKMeans:
    """run() (engine.cpp:345-425) over document shards."""

    def __init__(self, shard, comm: Comm, n_total: int, k: int, mode: str = "baseline", conv_sq_dist: float = 1e-4,
                 max_iters: int = 100):
        self.s, self.comm, self.n_total, self.k = shard, comm, n_total, k
        self.mode, self.conv, self.max_iters = mode, conv_sq_dist, max_iters
        self.iteration = 0
        self.bounds = [shard_range(n_total, r, comm.world) for r in range(comm.world)]

    def owner(self, gid: int) -> int:
        for r, (b, e) in enumerate(self.bounds):
            if b <= gid < e:
                return r
        raise ValueError(gid)

    def init_from_seeds(self, seeds):
        """Centroid j = document seeds[j]: owners contribute the rows."""
        seeds = [int(x) for x in seeds]
        mine = [(j, g) for j, g in enumerate(seeds) if self.owner(g) == self.comm.rank]
        rows = self.s.rows([g for _, g in mine])
        gathered = self.comm.all_gather_object([(j, r) for (j, _), r in zip(mine, rows)])
        by_j = {}
        for part in gathered:
            for j, r in part:
                by_j[j] = r
        rptr = np.zeros(self.k + 1, np.int64)
        idx, val = [], []
        for j in range(self.k):
            ri, rv = by_j[j]
            rptr[j + 1] = rptr[j] + len(ri)
            idx.append(ri)
            val.append(rv)
        self.s.init_from_rows(rptr, np.concatenate(idx) if idx else [], np.concatenate(val) if val else [])
        self.iteration = 0

    def update(self) -> IterationStats:
        counts = self.comm.all_reduce_i64(self.s.local_counts())
        repaired = []
        if np.any(counts == 0):
            n_empty = int(np.sum(counts == 0))
            m = 2 * n_empty + 256
            n_locals = self.comm.all_gather_object(self._n_local())
            while True:
                cl = self.comm.all_gather_object(self.s.local_candidates(m))
                moves = replay_repair(counts, cl, n_locals, m)
                if moves is not None:
                    break
                m *= 4
            for gid, _, new in moves:
                if self.owner(gid) == self.comm.rank:
                    self.s.move_doc(gid, new)
            repaired = [new for _, _, new in moves]
        import torch

        old, new, lens, idx, val = self.s.moved_pack()
        # two payloads: per moved document (old, new, row length), and the rows
        # (term ids and the fp32 weights' bits): one length gather + two gathers
        meta = torch.cat([old, new, lens])
        rows = torch.cat([idx, val.view(torch.int32)])
        g_meta, g_rows = self.comm.all_gather_var_multi([meta, rows])
        parts = [[], [], [], [], []]
        for m_r, r_r in zip(g_meta, g_rows):
            n_r, z_r = m_r.numel() // 3, r_r.numel() // 2
            parts[0].append(m_r[:n_r])
            parts[1].append(m_r[n_r:2 * n_r])
            parts[2].append(m_r[2 * n_r:])
            parts[3].append(r_r[:z_r])
            parts[4].append(r_r[z_r:].view(torch.float32))
        cat = [self._cat(p) for p in parts]
        st = self.s.update_apply(*cat, repaired)
        self.iteration += 1
        st.n_moved = int(len(cat[0]))
        st.iteration = self.iteration
        return st

    def _n_local(self):
        b, e = self.bounds[self.comm.rank]
        return e - b

    @staticmethod
    def _cat(ts):
        import torch
        return torch.cat(list(ts)) if len(ts) > 1 else ts[0]

    def assign(self) -> IterationStats:
        st = self.s.assign()
        # every counter is a sum over documents (the reference's accounting is
        # per document, engine.cpp:244-312), so the global value is the sum of
        # the ranks' local ones — in every mode, the ncc+index replay included
        # one gather: the objective partial and the counters (< 2^53: exact in
        # fp64), summed on the host in rank order
        g = self.comm.all_gather_f64_vec(np.array([st.objective, st.n_reassigned, st.n_rescan, st.n_exact,
                                                   st.gpu_dot_products, st.dot_products, st.index_queries,
                                                   st.candidates_total], np.float64))
        tot = [int(round(sum(float(v) for v in g[:, c]))) for c in range(1, g.shape[1])]
        obj = 0.0
        for o in g[:, 0]:  # rank order: deterministic for a given world size
            obj += float(o)
        return replace(st, n_reassigned=int(tot[0]), n_rescan=int(tot[1]), n_exact=int(tot[2]),
                       gpu_dot_products=int(tot[3]), objective=obj, dot_products=int(tot[4]),
                       index_queries=int(tot[5]), candidates_total=int(tot[6]))

    def step(self) -> IterationStats:
        u = self.update()
        a = self.assign()
        return replace(a, iteration=u.iteration, max_sq_drift=u.max_sq_drift, n_repaired=u.n_repaired,
                       n_moved=u.n_moved, n_recomputed=u.n_recomputed, update_ms=u.update_ms)

    def run(self):
        its, stop = [], 2
        for it in range(1, self.max_iters + 1):
            st = self.step()
            its.append(st)
            if st.n_reassigned == 0:
                stop = 0
                break
            if it > 1 and st.max_sq_drift < self.conv:
                stop = 1
                break
        return its, STOP_REASONS[stop]


def init_process_group_from_env(backend: Optional[str] = None):
    """torch.distributed from torchrun's env (MASTER_ADDR=127.0.0.1 here)."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if "RANK" not in os.environ:  # a single process outside torchrun (bench.py --distributed at N = 1)
        os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"})
    backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
    dist.init_process_group(backend=backend)
    return dist.get_rank(), dist.get_world_size()


def bench_distributed(args, extras=None):
    """bench.py at N > 1 (torchrun, one rank per GPU): strong scaling of config
    args.config over N GPUs. Device time of K steps on every rank's engine
    stream, max over ranks; clocks sampled on each rank's GPU during the timed
    region (rank 0 reports its own); e2e = the same K steps through the shard
    API from host CSR (upload, seeding, steps, download), wall clock max over
    ranks. `extras` (from bench.py): {"clock": ClockSampler class,
    "roofline": fn(stats, data) -> roofline dict}."""
    import json
    import statistics
    import time

    import torch
    import torch.distributed as dist

    from . import synthetic as S

    extras = extras or {}
    rank, world = init_process_group_from_env("nccl")
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    cfg = S.CONFIGS[args.config]
    data = S.corpus(cfg)  # deterministic on every rank; each keeps its shard
    shard, off = shard_corpus(data, rank, world)
    seeds = S.init_seeds(data.n_docs, cfg.k, 0)
    gs = GPUShard(shard, off, data.n_docs, cfg.k, device=local, mode=args.mode, conv_sq_dist=1e-300,
                  max_iters=10 ** 6)
    comm = Comm(rank, world, torch.device("cuda", local))
    km = DistributedKMeans(gs, comm, data.n_docs, cfg.k, mode=args.mode)
    km.init_from_seeds(seeds)
    # the clock sampler runs from before the warm-up (nothing is forked inside the timed region)
    clock = extras["clock"](local).start() if "clock" in extras else None
    for _ in range(max(args.warmup, 3)):
        km.step()
    dist.barrier()
    torch.cuda.synchronize()
    gs.eng.synchronize()
    if clock:
        clock.begin()
    gs.eng.timer_record(0)
    l0 = gs.eng.launch_count()
    stats = [km.step() for _ in range(args.steps)]
    gs.eng.timer_record(1)
    ms = gs.eng.timer_elapsed(0, 1)
    if clock:
        clock.end()
        clock.stop()
    dist.barrier()
    ms_max = comm.all_reduce_f64_max(ms)
    launches = gs.eng.launch_count() - l0
    K = args.steps
    e2e = None
    if not getattr(args, "no_e2e", False):
        del km, gs  # the timed engine's device memory goes back before the e2e engine is built
        import gc

        gc.collect()
        # end to end through the shard API from host CSR: upload, seeding, K steps, download
        dist.barrier()
        t0 = time.perf_counter()
        gs2 = GPUShard(shard, off, data.n_docs, cfg.k, device=local, mode=args.mode, conv_sq_dist=1e-300,
                       max_iters=10 ** 6)
        km2 = DistributedKMeans(gs2, comm, data.n_docs, cfg.k, mode=args.mode)
        km2.init_from_seeds(seeds)
        for _ in range(K):
            km2.step()
        a2, s2, _ = gs2.get_state()
        wall = comm.all_reduce_f64_max(time.perf_counter() - t0)
        h2d = shard.indptr.nbytes + shard.indices.nbytes + shard.values.nbytes + 4 * cfg.k
        e2e = {"value": data.n_docs * cfg.k * K / wall, "unit": "comparisons/s",
               "h2d_bytes_per_step": h2d * world / K, "d2h_bytes_per_step": (a2.nbytes + s2.nbytes) * world / K,
               "wall_s": wall, "iterations": K,
               "note": "every rank: shard upload, seeding, K steps, download of its assignments and sims; "
                       "wall clock, max over ranks; bytes summed over ranks, amortised per step"}
        del km2, gs2
    if rank == 0:
        line = {
            "metric": "effective doc·centroid comparisons/s", "value": data.n_docs * cfg.k * K / (ms_max / 1e3),
            "unit": "comparisons/s", "n_gpus": world, "steps": K, "warmup": max(args.warmup, 3),
            "ms_per_step": ms_max / K, "s_per_iteration": ms_max / K / 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE generator, seed 0)",
            "config": {"workload": f"{cfg.name}: N={data.n_docs}, d={cfg.dims}, k={cfg.k}", "mode": args.mode,
                       "parallelism": f"doc-sharded x{world}, delta all-gather (NCCL)",
                       "l2": "inputs larger than L2"},
            "phase_ms": {"update": statistics.mean(s.update_ms for s in stats),
                         "assign": statistics.mean(s.assign_ms for s in stats),
                         "screen": statistics.mean(s.screen_ms for s in stats)},
            "moved_per_iter": statistics.mean(s.n_moved for s in stats),
            "gpu_launches": launches,
        }
        if "roofline" in extras:
            line["roofline"] = extras["roofline"](stats, data)
        if clock:
            line["clocks"] = clock.summary()
        if e2e:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
