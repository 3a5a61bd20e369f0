"""GPU TF-IDF ingestion (sskm_vectorize) vs the reference's vectorize_corpus
(compiled oracle/_ref, one host thread: the reference is sequential) on seeded
synthetic texts; prints one JSON line per size. Results are checked bitwise."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2108_00895_b200 import vectorize_texts
from tests import textgen

for n in [int(x) for x in (sys.argv[1:] or ["20000", "200000"])]:
    texts = textgen.corpus(n, n_vocab=50000, seed=5)
    nbytes = sum(len(t.encode()) for t in texts)
    vectorize_texts(texts[:1000], stop_words=textgen.STOP)  # context + module warm
    t0 = time.perf_counter()
    g = vectorize_texts(texts, stop_words=textgen.STOP, max_df=0.5)
    wall = time.perf_counter() - t0
    r = O.ref_vectorize(texts, textgen.STOP, 0.5)
    same = (np.array_equal(g.matrix.indptr, r["indptr"]) and np.array_equal(g.matrix.indices, r["indices"])
            and np.array_equal(g.matrix.values64.view(np.uint64), r["values"].view(np.uint64))
            and g.vocab == r["vocab"] and np.array_equal(g.dropped_positions, r["dropped"]))
    print(json.dumps({"docs": n, "text_MB": nbytes / 1e6, "tokens": g.stats["tokens"], "vocab": len(g.vocab),
                      "nnz": int(g.matrix.nnz), "gpu_ms": g.stats["gpu_ms"], "call_s": wall,
                      "gpu_GBps_text": nbytes / (g.stats["gpu_ms"] * 1e-3) / 1e9, "launches": g.stats["launches"],
                      "ref_s": r["seconds"], "speedup_call": r["seconds"] / wall, "bitwise": bool(same)}), flush=True)
