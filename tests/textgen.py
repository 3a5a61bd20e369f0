"""Seeded synthetic text corpora for the vectorize parity tests (the
reference's own tests use hand-written strings, test_corpus.cpp:45-177): Zipf
word frequencies over a generated vocabulary with mixed case, digits, UTF-8
letters and ASCII punctuation separators, plus empty and stop-word-only
documents."""
import numpy as np

ALPHA = list("abcdefghijklmnopqrstuvwxyz")
EXTRA = ["é", "ü", "ß", "ñ", "日", "本", "ж"]
SEPS = [" ", " ", " ", " ", ", ", ". ", "-", "\n", "\t", "!", "'", "(", ")", "/", ":", ";", "  "]
STOP = ["the", "of", "and", "a", "to", "in", "is", "The"]  # "The" never matches a (lowercased) token


def vocab(n, rng):
    words = set()
    out = []
    while len(out) < n:
        L = int(rng.integers(1, 11))
        w = "".join(rng.choice(ALPHA, L))
        if rng.random() < 0.1:
            w += str(int(rng.integers(0, 100)))
        if rng.random() < 0.05:
            w = w[: L // 2] + str(rng.choice(EXTRA)) + w[L // 2:]
        if w not in words:
            words.add(w)
            out.append(w)
    return out


def corpus(n_docs, n_vocab=5000, mean_len=40, seed=0, s=1.1):
    rng = np.random.default_rng(seed)
    V = vocab(n_vocab, rng)
    Vu = [w.upper() for w in V]
    Vc = [w.capitalize() for w in V]
    cdf = np.cumsum(1.0 / np.arange(1, n_vocab + 1) ** s)
    cdf /= cdf[-1]
    texts = []
    for d in range(n_docs):
        r = rng.random()
        if r < 0.01:
            texts.append("")
            continue
        if r < 0.02:
            texts.append(" ".join(STOP[q] for q in rng.integers(0, 7, int(rng.integers(1, 5)))))
            continue
        if r < 0.025:
            texts.append(" ,.;! \t\n")
            continue
        L = max(1, int(rng.lognormal(np.log(mean_len), 0.6)))
        ids = np.minimum(np.searchsorted(cdf, rng.random(L)), n_vocab - 1)
        u = rng.random(L)
        st = rng.random(L) < 0.08
        sw = rng.integers(0, len(STOP), L)
        sp = rng.integers(0, len(SEPS), L)
        parts = []
        for q in range(L):
            w = STOP[sw[q]] if st[q] else (Vu if u[q] < 0.1 else Vc if u[q] < 0.2 else V)[ids[q]]
            parts.append(w)
            parts.append(SEPS[sp[q]])
        texts.append("".join(parts))
    return texts
