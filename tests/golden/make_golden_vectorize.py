"""Generates tests/golden/vectorize_golden.npz by running the UNMODIFIED
reference's vectorize_corpus (corpus.cpp:101-134, compiled into
oracle/_ref/libsskm_ref.so) on a seeded synthetic text corpus (tests/textgen.py).
Run in the dev container (needs /root/reference):
    python tests/golden/make_golden_vectorize.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from tests import textgen  # noqa: E402

N, NV, SEED, MAX_DF = 2000, 3000, 11, 0.5
texts = textgen.corpus(N, n_vocab=NV, seed=SEED)
r = O.ref_vectorize(texts, textgen.STOP, MAX_DF)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "vectorize_golden.npz"), n_docs=N, n_vocab=NV, seed=SEED,
                    max_df=MAX_DF, indptr=r["indptr"], indices=r["indices"], values=r["values"], kept=r["kept"],
                    dropped=r["dropped"], doc_freq=r["doc_freq"], vocab=np.array("\n".join(r["vocab"])))
print(len(r["vocab"]), "terms", len(r["indices"]), "nonzeros", len(r["dropped"]), "dropped", r["seconds"], "s")
