"""Benchmark: effective doc·centroid comparisons/s of full Lloyd iterations on
BASELINE.json config 1 (N=1e6, d=262,144, k=1,000), B200-native vs the
reference's own CPU path.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c1]

A step is one Lloyd iteration (compute_centroids + detect_unchanged + assign +
objective) over the whole corpus in `--mode` (default baseline: every iteration
is a full k-scan, the reference's default mode). value = N·k·K / device time of
the K timed steps (max over ranks), inputs resident in HBM. e2e = the same metric
through the public API (paper_2108_00895_b200.cluster on host CSR arrays:
upload, seeding, K iterations, download of assignments and sims).

--impl reference times the reference C++ engine (oracle/_ref, built from the
unmodified sources; the C restatement if absent) on this box's host cores:
per step, compute_centroids over all N documents plus a full-scan assign of a
uniform document sample, extrapolated by N / |sample|.
"""
from __future__ import annotations

import argparse
import json
import os
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
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
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
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic():
    """Per-launch DRAM bytes of the bound screen from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_bound_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    return None, None


# ----------------------------------------------------------------- reference --
def reference_iteration(data, k, seeds, a=None, sims=None, n_sample=2000, threads=0, steps=1, warmup=0,
                        seed=1):
    """Reference C++ engine timing on a bounded sample (SURVEY §8d CPU plan)."""
    from oracle import oracle as O

    kind = "ref" if O.ref_available() else "port"
    c = O.Corpus(data.indptr, data.indices, data.values.astype(np.float64), data.dims)
    st = O.Stepper(c, k, "baseline", threads=threads, kind=kind)
    t0 = time.perf_counter()
    if a is None:
        st.init_seeds(seeds)  # the reference's own seed assignment (full scan vs seed docs)
        a, sims, _ = st.get_state()
    setup_s = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    sample = np.sort(rng.choice(data.n_docs, n_sample, replace=False))
    lens = np.diff(data.indptr)[sample]
    ptr = np.zeros(n_sample + 1, np.int64)
    ptr[1:] = np.cumsum(lens)
    idx = np.concatenate([data.indices[data.indptr[i]:data.indptr[i + 1]] for i in sample])
    val = np.concatenate([data.values[data.indptr[i]:data.indptr[i + 1]] for i in sample]).astype(np.float64)
    cs = O.Corpus(ptr, idx, val, data.dims)
    sa = O.Stepper(cs, min(k, n_sample), "baseline", threads=threads, kind=kind)
    per_step = []
    for s in range(warmup + steps):
        t1 = time.perf_counter()
        st.compute_centroids(a, sims)  # all N documents (engine.cpp:137-195)
        t_cc = time.perf_counter() - t1
        cptr, cidx, cval = st.get_centroids_csr()
        sa.set_centroids_csr(cptr, cidx, cval)
        sa.set_state(a[sample], sims[sample], np.zeros(k, np.uint8), 1)
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
    from paper_2108_00895_b200 import synthetic as S

    cfg = S.CONFIGS[args.config]
    data = S.corpus(cfg)
    seeds = S.init_seeds(data.n_docs, cfg.k, 0)
    kind, steps, cores, setup_s, n_s = reference_iteration(
        data, cfg.k, seeds, n_sample=args.ref_sample, steps=args.steps, warmup=min(args.warmup, 1))
    t = statistics.mean(s[0] for s in steps)
    value = data.n_docs * cfg.k / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "s_per_iteration": t,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generator, seed 0)",
        "config": workload_config(cfg, data, args.mode),
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


def workload_config(cfg, data, mode):
    return {"workload": f"{cfg.name}: N={data.n_docs}, d={cfg.dims}, k={cfg.k}, K_true={cfg.k_true}, "
                        f"mean len {cfg.mean_len:g} (sigma {cfg.sigma}), nnz={data.nnz}",
            "mode": mode, "init": "k distinct docs, numpy default_rng(0).choice",
            "l2": "inputs larger than L2 (CSR + Ct + sums >> 126 MB)", "parallelism": "doc-sharded"}


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
    written) and 4 B per centroid value gathered by a candidate's exact dot."""
    m = lambda f: statistics.mean(getattr(s, f) for s in stats)
    pairs, dnnz, visits, cnnz = m("bound_pairs"), m("bound_doc_nnz"), m("bound_visits"), m("bound_cand_nnz")
    b = 8 * pairs + 16 * dnnz + 36 * visits + 4 * cnnz
    return {"bytes": b, "high_pairs": pairs, "doc_nnz": dnnz, "visits": visits, "candidates": m("bound_candidates"),
            "candidate_nnz": cnnz, "theta": m("bound_theta")}


def bound_roofline(stats, data):
    """roofline object of the dominant kernel (bound_screen_kernel) from the
    steps' own counters and CUDA-event times."""
    screen_ms = statistics.mean(s.screen_ms for s in stats)
    bb = bound_screen_bytes(stats)
    peak, peak_src = measured_peak_gbs()
    achieved = bb["bytes"] / (screen_ms / 1e3) / 1e9 if screen_ms > 0 else 0.0
    traffic, _ = ncu_traffic()
    kk = stats[0].n_changed if stats else 0
    bytes_dense = algorithmic_assign_bytes(data, max(kk, 1))
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "bound_screen_kernel",
            "bytes_per_assign": bb["bytes"], "bytes_breakdown": bb, "screen_ms_per_assign": screen_ms,
            "launches_per_assign": statistics.mean(s.screen_launches for s in stats), "peak_source": peak_src,
            "dense_equivalent": {"bytes": bytes_dense, "gbs": bytes_dense / (screen_ms / 1e3) / 1e9 if screen_ms else 0,
                                 "note": "SURVEY 8d B_assign (4·Σ nnz_i·k): what a dense Ct scan would move"},
            "note": "algorithmic bytes of the bound screen = 8·high pairs + 16·doc nnz read + 36·doc visits "
                    "+ 4·candidate-dot nnz (DESIGN.md §3.1), over the kernel's CUDA-event time; "
                    "traffic = ncu dram bytes per launch (profiles/ncu_bound_summary.json)"}


def run_ours(args):
    import paper_2108_00895_b200 as P
    from paper_2108_00895_b200 import synthetic as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if world > 1 or args.distributed:
        from paper_2108_00895_b200 import distributed as D

        return D.bench_distributed(args, {"clock": ClockSampler, "roofline": bound_roofline})
    cfg = S.CONFIGS[args.config]
    data = S.corpus(cfg)
    k = cfg.k
    seeds = S.init_seeds(data.n_docs, k, 0)
    eng = P.Engine(0)
    eng.upload(data)
    eng.configure(k, mode=args.mode, conv_sq_dist=1e-300, max_iters=10 ** 6)
    eng.init_from_seeds(seeds)
    for _ in range(args.warmup):
        eng.step()
    eng.synchronize()
    l0 = eng.launch_count()
    stats = []
    with ClockSampler(0) as clk:
        eng.timer_record(0)
        for _ in range(args.steps):
            stats.append(eng.step())
        eng.timer_record(1)
        total_ms = eng.timer_elapsed(0, 1)
    launches = eng.launch_count() - l0
    a_post, s_post, _ = eng.get_state()
    K = args.steps
    value = data.n_docs * k * K / (total_ms / 1e3)
    performed = sum(s.gpu_dot_products for s in stats) / (total_ms / 1e3)
    kern_ms = [s.assign_kernel_ms for s in stats]
    peak, peak_src = measured_peak_gbs()
    roofline = bound_roofline(stats, data)
    roofline["full_postings_pairs_per_assign"] = eng.postings_work()
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "s_per_iteration": total_ms / K / 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generator, seed 0; fp32 storage, fp64 accumulation)",
        "config": workload_config(cfg, data, args.mode),
        "performed_comparisons_per_s": performed,
        "phase_ms": {"update": statistics.mean(s.update_ms for s in stats),
                     "assign": statistics.mean(s.assign_ms for s in stats),
                     "assign_kernels": statistics.mean(kern_ms),
                     "screen": roofline["screen_ms_per_assign"]},
        "exact_scan_docs_per_iter": statistics.mean(s.n_exact for s in stats),
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not args.no_e2e:
        line["e2e"] = e2e(P, data, k, seeds, K, args.mode)
    if not args.no_cpu_baseline and rank == 0:
        kind, steps, cores, setup_s, n_s = reference_iteration(data, k, seeds, a=a_post, sims=s_post,
                                                               n_sample=args.ref_sample, steps=1)
        t_iter = steps[0][0]
        line["cpu_baseline"] = {
            "value": data.n_docs * k / t_iter, "unit": UNIT, "cores": cores,
            "kind": "reference" if kind == "ref" else "port",
            "sample": f"compute_centroids over all {data.n_docs} docs + full-scan assign of {n_s} sampled docs "
                      f"vs k={k} (state after the timed GPU steps), extrapolated x{data.n_docs / n_s:.0f}",
            "s_per_iteration": t_iter}
    print(json.dumps(line), flush=True)


def e2e(P, data, k, seeds, K, mode):
    """Same metric through the public API with host buffers (upload + seed + K
    iterations + download), wall clock."""
    P.cluster(data, k, mode=mode, init_seeds=seeds, max_iters=1, conv_sq_dist=1e-300,
              return_centroids=False)  # context / module warm
    t0 = time.perf_counter()
    r = P.cluster(data, k, mode=mode, init_seeds=seeds, max_iters=K, conv_sq_dist=1e-300,
                  return_centroids=False)
    wall = time.perf_counter() - t0
    n_it = len(r.iterations)
    h2d = data.indptr.nbytes + data.indices.nbytes + data.values.nbytes + 4 * k
    d2h = r.assignments.nbytes + r.sims.nbytes
    return {"value": data.n_docs * k * n_it / wall, "unit": UNIT, "h2d_bytes_per_step": h2d / n_it,
            "d2h_bytes_per_step": d2h / n_it, "wall_s": wall, "iterations": n_it,
            "note": "one cluster() call; CSR uploaded once per run, amortised per step"}


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
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
