"""`sskm bench` on the GPU: the reference CLI's benchmark CSV (cmd_bench,
proj/tools/sskm_main.cpp:180-262) from GPU runs, plus the B200 columns.

  python -m paper_2108_00895_b200.bench_csv --config c1 --k-list 1000 \
      --modes baseline,ncc,ncc+index --repeats 3 --out bench.csv

Per (mode, k): `repeats` timed runs of the whole clustering (sskm::run: seeding
then the Lloyd loop — here through cluster(), host CSR in, assignments out),
median and inter-quartile range of the wall time exactly as the reference
computes them (sorted times; median of the middle pair for even counts; IQR =
t[3n/4] − t[n/4]), the reference-accounted dot products and iteration count of
the last run, and the median index build time. The reference's seven columns
come first, unchanged; the added ones are:

  comparisons_per_s   N·k·iterations / median_seconds (effective comparisons)
  exact_dots          dots the GPU evaluated in full (gpu_dot_products)
  screen_gbs          bound-screen algorithmic bytes / screen time
  roofline_frac       screen_gbs / measured HBM peak (MEASURED_PEAKS.json)

`--input` reads the reference's text matrix format (load_matrix); `--config`
builds a BASELINE corpus; `--init seeds` uses BASELINE's k-distinct-documents
init instead of k-means++.
"""
from __future__ import annotations

import argparse
import json
import os
import time

import numpy as np

from .api import cluster

HEADER = "mode,k,median_seconds,iqr_seconds,dot_products,iterations,index_build_seconds"
EXTRA = "comparisons_per_s,exact_dots,screen_gbs,roofline_frac"


def _peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    return 6650.0


def _median(v):
    v = sorted(v)
    n = len(v)
    return v[n // 2] if n % 2 == 1 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def bench_rows(data, ks, modes, repeats=1, init="kmeans++", seed=7, **cfg):
    """One row per (mode, k), the reference's loop order (modes outer, ks inner)."""
    if repeats < 1:
        raise ValueError("--repeats must be at least 1")
    peak = _peak_gbs()
    rows = []
    for mode in modes:
        for k in ks:
            times, builds = [], []
            last = None
            for _ in range(repeats):
                seeds = None
                if init == "seeds":
                    seeds = np.random.default_rng(0).choice(data.n_docs, k, replace=False).astype(np.uint32)
                t0 = time.perf_counter()
                r = cluster(data, k, mode=mode, seed=seed, init_seeds=seeds, **cfg)
                times.append(time.perf_counter() - t0)
                builds.append(r.total_index_build_seconds())
                last = r
            ts = sorted(times)
            n = len(ts)
            med = _median(ts)
            iqr = ts[(3 * n) // 4] - ts[n // 4]
            its = last.iterations
            screen_ms = sum(it.screen_ms for it in its)
            sbytes = sum(8 * it.bound_pairs + 16 * it.bound_doc_nnz + 36 * it.bound_visits + 4 * it.bound_cand_nnz
                         for it in its)
            gbs = sbytes / (screen_ms / 1e3) / 1e9 if screen_ms > 0 else 0.0
            rows.append({"mode": mode, "k": k, "median_seconds": med, "iqr_seconds": iqr,
                         "dot_products": last.total_dot_products(), "iterations": len(its),
                         "index_build_seconds": _median(builds),
                         "comparisons_per_s": data.n_docs * k * len(its) / med if med > 0 else 0.0,
                         "exact_dots": int(sum(it.gpu_dot_products for it in its)),
                         "screen_gbs": gbs, "roofline_frac": gbs / peak})
    return rows


def to_csv(rows) -> str:
    """The reference's formatting for its columns (fixed 6 digits for seconds,
    default formatting for counts), then the added columns."""
    out = [HEADER + "," + EXTRA]
    for r in rows:
        out.append(f"{r['mode']},{r['k']},{r['median_seconds']:.6f},{r['iqr_seconds']:.6f},{r['dot_products']},"
                   f"{r['iterations']},{r['index_build_seconds']:.6f},{r['comparisons_per_s']:.6g},"
                   f"{r['exact_dots']},{r['screen_gbs']:.6g},{r['roofline_frac']:.6g}")
    return "\n".join(out) + "\n"


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--input", help="matrix file in the reference's text format")
    src.add_argument("--config", help="BASELINE corpus c0..c4")
    ap.add_argument("--k-list", default="10")
    ap.add_argument("--modes", default="baseline,ncc,ncc+index")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--lambdas", default="0.1,0.25,0.4,0.6")
    ap.add_argument("--conv", type=float, default=0.0001)
    ap.add_argument("--ncc-eps", type=float, default=0.0)
    ap.add_argument("--index-activation", type=int, default=100)
    ap.add_argument("--max-iters", type=int, default=100)
    ap.add_argument("--init", choices=["kmeans++", "seeds"], default="kmeans++")
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    if a.input:
        from .io import load_matrix
        data = load_matrix(a.input)
    else:
        from . import synthetic
        data = synthetic.corpus(a.config)
    ks = [int(x) for x in a.k_list.split(",") if x]
    modes = [m for m in a.modes.split(",") if m]
    if not modes:
        raise SystemExit("--modes: empty list")
    rows = bench_rows(data, ks, modes, a.repeats, init=a.init, seed=a.seed,
                      lambdas=[float(x) for x in a.lambdas.split(",") if x], conv_sq_dist=a.conv,
                      ncc_epsilon=a.ncc_eps, index_activation_threshold=a.index_activation, max_iters=a.max_iters)
    with open(a.out, "w") as f:
        f.write(to_csv(rows))
    for r in rows:
        print(f"bench {r['mode']} k={r['k']}: median {r['median_seconds']:g} s, {r['dot_products']} dot products, "
              f"{r['iterations']} iterations")


if __name__ == "__main__":
    main()
