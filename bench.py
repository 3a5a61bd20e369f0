"""Benchmark: effective doc·centroid comparisons/s of full Lloyd iterations on
BASELINE.json config 1 (N=1e6, d=262,144, k=1,000), B200-native vs the
reference's own CPU path.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c1] [--mode baseline]

A step is one Lloyd iteration (compute_centroids + detect_unchanged + assign +
objective) over the whole corpus in `--mode` (default baseline: every iteration
is a full k-scan, the reference's default mode). value = N·k·K / device time of
the K timed steps (CUDA events on the engine's stream; max over ranks), inputs
resident in HBM. e2e = the same metric through the public API
(paper_2108_00895_b200.cluster on host CSR arrays: engine construction, upload,
seeding, K iterations, download of assignments and sims), wall clock.

After the timed steps, rank 0 runs one more iteration teacher-forced against the
compiled reference (oracle/teacher.py) and reports a `parity` block, and times
the reference on the box's host cores (`cpu_baseline`, all three modes).

--impl reference times the reference C++ engine (oracle/_ref, built from the
unmodified sources; the C restatement if absent) on this box's host cores: per
step, compute_centroids over all N documents plus a full-scan assign of a
uniform document sample, extrapolated by N / |sample|. That arm imports only
`corpora` (the input generator) and `oracle/` — nothing of this package.

--gpus N without torchrun re-launches itself under torch.distributed.run with N
ranks (one process per GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective doc·centroid comparisons/s"
UNIT = "comparisons/s"


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    The sampler process is started before the warm-up (forking it at the start
    of the timed region delayed the first timed step's launches by 1-2 ms) and
    polls every 50 ms; `begin()` / `end()` bracket the timed region and the
    summary uses the samples that arrived inside it (plus one period after)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 50  # a 20 ms poll measurably slowed the steps it was watching (driver locks): 1.58 -> 1.61 ms

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []  # (arrival time, line)
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def begin(self):
        self.t0 = time.perf_counter()

    def end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.proc:
            time.sleep(2.5 * self.PERIOD_MS / 1e3)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    # context-manager form: sampler started here, the whole block is the timed region
    def __enter__(self):
        if self.proc is None:
            self.start()
        self.begin()
        return self

    def __exit__(self, *exc):
        self.end()
        self.stop()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def collect(rows):
            sm, mx, reasons = [], [], set()
            for ln in rows:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx.append(float(parts[1]))
                except ValueError:
                    continue
                for name, v in zip(names, parts[4:8]):
                    if v.lower() == "active":
                        reasons.add(name)
            return sm, mx, reasons

        inside = [ln for (t, ln) in self.lines
                  if self.t0 is not None and self.t1 is not None and self.t0 <= t <= self.t1 + 2 * self.PERIOD_MS / 1e3]
        sm, mx, reasons = collect(inside)
        where = "timed region"
        if not sm:  # a region shorter than the polling period: the nearest samples around it
            sm, mx, reasons = collect([ln for _, ln in self.lines])
            where = "around the timed region (shorter than the polling period)"
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "sampled": where, "period_ms": self.PERIOD_MS}


def ncu_traffic():
    """Per-launch DRAM bytes of the bound screen from the committed ncu capture of
    this bench command (profiles/r02_ncu_bound_summary.json)."""
    p = os.path.join(ROOT, "profiles", "r02_ncu_bound_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    return None, None


def workload_config(cfg, data, mode):
    return {"workload": f"{cfg.name}: N={data.n_docs}, d={cfg.dims}, k={cfg.k}, K_true={cfg.k_true}, "
                        f"mean len {cfg.mean_len:g} (sigma {cfg.sigma}), nnz={data.nnz}",
            "mode": mode, "init": "k distinct docs, numpy default_rng(0).choice",
            "l2": (lambda csr, ld: f"inputs larger than L2 (CSR {csr / 1e9:.2f} GB + Ct {cfg.dims * ld * 4 / 1e9:.2f} GB + "
                   f"sums {cfg.dims * ld * 8 / 1e9:.1f} GB >> 126 MB); no flush")(
                       data.nnz * 8 + (data.n_docs + 1) * 8, -(-cfg.k // 128) * 128),
            "parallelism": "doc-sharded"}


# ----------------------------------------------------------------- reference --
def sample_corpus(O, data, docs, remap=False):
    from oracle.teacher import gather_rows

    ptr, idx, val = gather_rows(data, docs)
    return O.Corpus(ptr, idx, val.astype(np.float64), data.dims)


def reference_arm_iteration(data, k, seeds, n_sample=2000, threads=0, steps=1, warmup=0, seed=1):
    """Reference C++ engine on a bounded sample (SURVEY §8d CPU plan): the
    reference's own seed assignment (untimed), then per step compute_centroids
    over all N documents + a full-scan assign of a uniform sample, extrapolated."""
    from oracle import oracle as O

    kind = "ref" if O.ref_available() else "port"
    c = O.Corpus(data.indptr, data.indices, data.values.astype(np.float64), data.dims)
    st = O.Stepper(c, k, "baseline", threads=threads, kind=kind)
    t0 = time.perf_counter()
    st.init_seeds(seeds)  # the reference's own seed assignment (full scan vs seed docs)
    a, sims, _ = st.get_state()
    setup_s = time.perf_counter() - t0
    docs = np.sort(np.random.default_rng(seed).choice(data.n_docs, n_sample, replace=False))
    cs = sample_corpus(O, data, docs)
    sa = O.Stepper(cs, k, "baseline", threads=threads, kind=kind, sample=kind == "ref") if kind == "ref" else \
        O.Stepper(cs, min(k, n_sample), "baseline", threads=threads, kind=kind)
    per_step = []
    for s in range(warmup + steps):
        t1 = time.perf_counter()
        st.compute_centroids(a, sims)  # all N documents (engine.cpp:137-195)
        t_cc = time.perf_counter() - t1
        sa.set_centroids_csr(*st.get_centroids_csr())
        sa.set_state(a[docs], sims[docs], np.zeros(k, np.uint8), 1)
        t2 = time.perf_counter()
        sa.assign()  # full scan, engine.cpp:265-266
        t_as = time.perf_counter() - t2
        t_iter = t_cc + t_as * data.n_docs / n_sample
        if s >= warmup:
            per_step.append((t_iter, t_cc, t_as))
    cores = threads or os.cpu_count()
    return kind, per_step, cores, setup_s, n_sample


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import corpora  # input generator only: no module of this package is imported on this arm

    cfg = corpora.CONFIGS[args.config]
    data = corpora.corpus(cfg)
    seeds = corpora.init_seeds(data.n_docs, cfg.k, 0)
    kind, steps, cores, setup_s, n_s = reference_arm_iteration(
        data, cfg.k, seeds, n_sample=args.ref_sample, steps=args.steps, warmup=min(args.warmup, 1))
    t = statistics.mean(s[0] for s in steps)
    value = data.n_docs * cfg.k / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "s_per_iteration": t,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generator, seed 0)",
        "config": workload_config(cfg, data, "baseline"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores,
                         "kind": "reference" if kind == "ref" else "port",
                         "sample": f"per step: compute_centroids over all {data.n_docs} docs + full-scan assign "
                                   f"of {n_s} uniformly sampled docs vs k={cfg.k}, extrapolated x{data.n_docs / n_s:.0f}; "
                                   f"setup (reference seed assignment) {setup_s:.1f}s untimed",
                         "t_compute_centroids_s": statistics.mean(s[1] for s in steps),
                         "t_assign_sample_s": statistics.mean(s[2] for s in steps)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------- ours --
def algorithmic_assign_bytes(data, k):
    """B_assign = 4·Σ nnz_i·k_i + 8·nnz + 8·(N+1) + 24·N (full scan: k_i = k)."""
    n, nnz = data.n_docs, data.nnz
    return 4 * nnz * k + 8 * nnz + 8 * (n + 1) + 24 * n


def bound_screen_bytes(stats):
    """Algorithmic bytes the bound screen moves per assign, from
    the kernel's own counters: 8 B per high (cluster, value) pair, 16 B per
    document nonzero (idx, val and the two posting offsets of its term), 36 B per
    document visit (indptr pair, work-list id, running (arg, best) read and
    written), 4 B per centroid value gathered by a candidate's exact dot or by an
    own-cluster dot, and the 68 B the kernel writes per visited document for the
    drift bound (32 fp16 group bounds + the iteration stamp)."""
    m = lambda f: statistics.mean(getattr(s, f) for s in stats)
    pairs, dnnz, visits, cnnz = m("bound_pairs"), m("bound_doc_nnz"), m("bound_visits"), m("bound_cand_nnz")
    onnz = m("bound_own_nnz")
    ub = 68 * visits if any(s.skip_docs for s in stats) else 0  # the drift bound's outputs (full-scan passes)
    b = 8 * pairs + 16 * dnnz + 36 * visits + 4 * cnnz + 4 * onnz + ub
    return {"bytes": b, "own_dot_nnz": onnz, "high_pairs": pairs, "doc_nnz": dnnz, "visits": visits, "candidates": m("bound_candidates"),
            "own_dots": m("bound_own_dots"), "candidate_nnz": cnnz, "theta": m("bound_theta")}


def bound_roofline(stats, data):
    """roofline object of the dominant kernel (bound_screen_kernel) from the
    steps' own counters and CUDA-event times."""
    screen_ms = statistics.mean(s.screen_ms for s in stats)
    bb = bound_screen_bytes(stats)
    peak, peak_src = measured_peak_gbs()
    achieved = bb["bytes"] / (screen_ms / 1e3) / 1e9 if screen_ms > 0 else 0.0
    traffic, summ = ncu_traffic()
    kk = stats[0].n_changed if stats else 0
    bytes_dense = algorithmic_assign_bytes(data, max(kk, 1))
    out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": traffic, "kernel": "bound_screen_kernel",
           "bytes_per_assign": bb["bytes"], "bytes_breakdown": bb, "screen_ms_per_assign": screen_ms,
           "launches_per_assign": statistics.mean(s.screen_launches for s in stats), "peak_source": peak_src,
           "dense_equivalent": {"bytes": bytes_dense, "gbs": bytes_dense / (screen_ms / 1e3) / 1e9 if screen_ms else 0,
                                "note": "SURVEY 8d B_assign (4·Σ nnz_i·k): what a dense Ct scan would move"},
           "note": "algorithmic bytes of the bound screen = 8·high pairs + 16·doc nnz read + (36 + 68)·doc visits "
                   "+ 4·(candidate-dot + own-dot) nnz (DESIGN.md §3.1), over the kernel's CUDA-event time; "
                   "traffic = ncu dram__bytes_read+write per launch of the same bench command "
                   "(profiles/r02_ncu_bound_summary.json)"}
    if traffic and summ:
        out["traffic_over_algorithmic"] = traffic / summ.get("algorithmic_bytes_per_launch", bb["bytes"])
        out["traffic_capture"] = summ.get("capture", "")
    return out


def teacher_forced_step(eng, data, k, mode, n_sample=2000, n_cols=200, seed=1):
    """One more iteration, teacher-forced against the reference on a document
    sample (oracle/teacher.py), plus the reference's own timing per mode from the
    same state (cpu_baseline). Runs after the timed region."""
    from oracle import oracle as O
    from oracle.teacher import TeacherForcing

    kind = "ref" if O.ref_available() else "port"
    docs = np.sort(np.random.default_rng(seed).choice(data.n_docs, n_sample, replace=False))
    tf = TeacherForcing(data, k, mode, kind=kind, docs=docs)
    a_pre, s_pre, _ = eng.get_state()
    eng.update()
    it = eng.iteration
    cols = np.random.default_rng(100 + it).choice(k, min(k, n_cols), replace=False)
    t0 = time.perf_counter()
    up, (a_mid, s_mid, unch) = tf.check_update(eng, a_pre, s_pre, cols=cols)
    t_cc = time.perf_counter() - t0  # reference compute_centroids over all N (+ a column download)
    eng.assign()
    a_post, s_post, _ = eng.get_state()
    asg = tf.check_assign(eng, a_mid, s_mid, unch, it, a_post, s_post)
    parity = {"iteration": it, "kind": kind, "docs": asg["docs"], "mismatches": asg["mismatches"],
              "near_ties": asg["near_ties"], "sims_not_bitwise": asg["sims_not_bitwise"],
              "centroid_cols": up["cols"], "max_centroid_rel": up["max_centroid_rel"],
              "max_centroid_abs": up["max_centroid_abs"], "repairs_equal": up["repaired_equal"],
              "ok": bool(up["ok"] and asg["ok"]),
              "how": "GPU state before/after one more iteration fed to the reference: compute_centroids over "
                     "all documents (column sample compared), assign on a uniform document sample with the "
                     "GPU's fp32 centroids (oracle/teacher.py)"}
    # reference assign timing per mode, from the reference's own centroids and the GPU's state
    cs = sample_corpus(O, data, docs)
    ref_ct = tf.upd.get_centroids_csr()
    n_unch = int(unch.sum())
    modes = {}
    for md in ("baseline", "ncc", "ncc+index"):
        sa = O.Stepper(cs, k, md, kind=kind, sample=kind == "ref") if kind == "ref" else \
            O.Stepper(cs, min(k, n_sample), md, kind=kind)
        sa.set_centroids_csr(*ref_ct)
        sa.set_state(a_mid[docs], s_mid[docs], unch, it)
        t1 = time.perf_counter()
        r = sa.assign(n_unchanged=n_unch)
        t_as = time.perf_counter() - t1
        t_build = r.get("index_build_seconds", 0.0)
        t_iter = t_cc + t_build + (t_as - t_build) * data.n_docs / n_sample
        modes[md] = {"s_per_iteration": t_iter, "value": data.n_docs * k / t_iter,
                     "t_assign_sample_s": t_as, "index_build_s": t_build, "index_active": bool(r["index_active"]),
                     "sample_dot_products": int(r["dot_products"])}
    return parity, modes, t_cc, kind


def relaunch_under_torchrun(args):
    """--gpus N without torchrun: one process per GPU through torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the scaling run checks the communicator size in NCCL's log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_ours(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.distributed:
        from paper_2108_00895_b200 import distributed as D

        return D.bench_distributed(args, {"clock": ClockSampler, "roofline": bound_roofline})
    import corpora
    import paper_2108_00895_b200 as P
    from paper_2108_00895_b200 import synthetic

    rank = int(os.environ.get("RANK", "0"))
    t_ctx = time.perf_counter()
    probe = P.Engine(0)  # CUDA context creation, timed on its own
    probe.close()
    t_ctx = time.perf_counter() - t_ctx
    cfg = corpora.CONFIGS[args.config]
    data = synthetic.corpus(cfg)
    k = cfg.k
    seeds = corpora.init_seeds(data.n_docs, k, 0)
    K, W = args.steps, args.warmup
    e2e_line = e2e(P, data, k, seeds, K, args.mode, t_ctx) if not args.no_e2e else None

    eng = P.Engine(0)
    eng.upload(data)
    eng.configure(k, mode=args.mode, conv_sq_dist=1e-300, max_iters=10 ** 6)
    eng.init_from_seeds(seeds)
    # every step between two events (slot s = start of step s): iteration 1 and
    # the warm-up steps are reported too; the timed region is slots W .. W+K
    all_stats = []
    clk = ClockSampler(0).start()  # running before the warm-up: nothing is forked inside the timed region
    time.sleep(0.05)
    eng.synchronize()
    eng.timer_record(0)
    for s in range(W):
        all_stats.append(eng.step())
        eng.timer_record(s + 1)
    eng.synchronize()
    l0 = eng.launch_count()
    clk.begin()
    # the K timed steps in one native call (sskm_step_n): the step loop of the
    # C-ABI, as sskm_run / the C++ run() drive it, without a Python round trip
    # (ctypes call + stats conversion, ~60 us) between the steps
    all_stats += eng.step_n(K)
    eng.timer_record(W + 1)
    total_ms = eng.timer_elapsed(W, W + 1)
    clk.end()
    clk.stop()
    launches = eng.launch_count() - l0
    # warm-up steps: event-bracketed; timed steps: the engine's own per-phase events (update + assign)
    per_iter = [eng.timer_elapsed(s, s + 1) for s in range(W)] + [s.update_ms + s.assign_ms for s in all_stats[W:]]
    stats = all_stats[W:]
    value = data.n_docs * k * K / (total_ms / 1e3)
    performed = sum(s.gpu_dot_products for s in stats) / (total_ms / 1e3)
    peak, peak_src = measured_peak_gbs()
    roofline = bound_roofline(stats, data)
    roofline["full_postings_pairs_per_assign"] = eng.postings_work()
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": total_ms / K, "s_per_iteration": total_ms / K / 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generator, seed 0; fp32 storage, fp64 accumulation)",
        "config": workload_config(cfg, data, args.mode),
        "iterations_timed": [W + 1, W + K],
        "iteration_ms": {"iteration_1": per_iter[0], "warmup": per_iter[:W],
                         "timed_mean": total_ms / K, "last_5_mean": statistics.mean(per_iter[-5:]),
                         "timed": per_iter[W:]},
        "exact_dots_per_s": performed,
        "exact_dots_per_iter": statistics.mean(s.gpu_dot_products for s in stats),
        "phase_ms": {"update": statistics.mean(s.update_ms for s in stats),
                     "assign": statistics.mean(s.assign_ms for s in stats),
                     "assign_kernels": statistics.mean(s.assign_kernel_ms for s in stats),
                     "screen": roofline["screen_ms_per_assign"]},
        "drift_bound": {"docs_kept_per_iter": statistics.mean(s.skip_docs for s in stats),
                        "ms": statistics.mean(s.skip_ms for s in stats),
                        "last_5_docs_kept": statistics.mean(s.skip_docs for s in stats[-5:]),
                        "note": "documents the drift bound kept in their cluster without a screen "
                                "(drift bound pass, DESIGN.md §3.1b)"},
        "moved_per_iter": statistics.mean(s.n_moved for s in stats),
        "exact_scan_docs_per_iter": statistics.mean(s.n_exact for s in stats),
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if e2e_line:
        line["e2e"] = e2e_line
    if not args.no_cpu_baseline and rank == 0:
        parity, modes, t_cc, kind = teacher_forced_step(eng, data, k, args.mode, n_sample=args.ref_sample)
        line["parity"] = parity
        base = modes["baseline"]
        line["cpu_baseline"] = {
            "value": base["value"], "unit": UNIT, "cores": os.cpu_count(),
            "kind": "reference" if kind == "ref" else "port",
            "sample": f"compute_centroids over all {data.n_docs} docs ({t_cc:.2f}s) + assign of "
                      f"{args.ref_sample} uniformly sampled docs vs k={k}, extrapolated x{data.n_docs / args.ref_sample:.0f}, "
                      f"from the GPU's state after the timed steps (iteration {parity['iteration']}); "
                      f"ncc / ncc+index from the same state (unchanged flags as detect_unchanged sets them)",
            "s_per_iteration": base["s_per_iteration"], "modes": modes}
    print(json.dumps(line), flush=True)


def e2e(P, data, k, seeds, K, mode, t_ctx):
    """Same metric through the public API with host buffers, wall clock: the
    FIRST cluster() call of the process (engine construction and its device
    allocations, pinned staging, upload, seeding, K iterations, download of
    assignments and sims). A second call (engine cached) is reported beside it."""
    def one():
        t0 = time.perf_counter()
        r = P.cluster(data, k, mode=mode, init_seeds=seeds, max_iters=K, conv_sq_dist=1e-300)
        return time.perf_counter() - t0, r
    wall, r = one()
    wall2, _ = one()
    n_it = len(r.iterations)
    h2d = data.indptr.nbytes + data.indices.nbytes + data.values.nbytes + 4 * k
    d2h = r.assignments.nbytes + r.sims.nbytes
    return {"value": data.n_docs * k * n_it / wall, "unit": UNIT, "h2d_bytes_per_step": h2d / n_it,
            "d2h_bytes_per_step": d2h / n_it, "wall_s": wall, "iterations": n_it,
            "second_call": {"value": data.n_docs * k * n_it / wall2, "wall_s": wall2},
            "cuda_context_init_s": t_ctx,
            "note": "first cluster() call of the process (CUDA context already created, timed separately); "
                    "CSR uploaded once per call, bytes amortised per step"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c1")
    ap.add_argument("--mode", default="baseline", choices=["baseline", "ncc", "ncc+index"])
    ap.add_argument("--ref-sample", type=int, default=2000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--distributed", action="store_true", help="use the sharded driver even at N=1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
