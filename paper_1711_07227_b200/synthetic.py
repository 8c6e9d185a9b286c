"""Deterministic synthetic workloads.

Embeddings are N(0,1) float32 (or clustered for precision stress tests).
Each histogram draws ``h_i`` word ids uniformly from [0, V) with ``h_i``
uniform in [h - h//2, h + h//2], sorts and de-duplicates them (so rows hold
about ``h`` unique words, ascending as corpus.py:93 requires) and gives them
weights ``(u + 0.1) / sum`` with ``u ~ U[0, 1)``, stored float32 -- the
L1-normalised term-frequency shape build_histograms produces
(corpus.py:398-399).
"""

from __future__ import annotations

import numpy as np

from .corpus import HistogramSet


def embeddings(vocab: int, dim: int, seed: int = 0, clustered: bool = False,
               centers: int = 500, spread: float = 0.05) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if not clustered:
        return rng.standard_normal((vocab, dim), dtype=np.float32)
    c = rng.standard_normal((centers, dim), dtype=np.float32)
    lab = rng.integers(0, centers, vocab)
    return (c[lab] + spread * rng.standard_normal((vocab, dim), dtype=np.float32)).astype(np.float32)


def histograms(n: int, vocab: int, h: int, seed: int = 1, chunk: int = 1 << 18) -> HistogramSet:
    """n rows of ~h unique words over a vocab of size ``vocab``."""
    rng = np.random.default_rng(seed)
    lo, hi = max(1, h - h // 2), h + h // 2
    hi = min(hi, vocab)
    lo = min(lo, hi)
    sizes_all = []
    ids_all = []
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        m = c1 - c0
        hs = rng.integers(lo, hi + 1, m)
        ids = rng.integers(0, vocab, (m, hi), dtype=np.int64)
        cols = np.arange(hi)[None, :]
        ids = np.where(cols < hs[:, None], ids, vocab)  # sentinel sorts last
        ids.sort(axis=1)
        keep = ids < vocab
        keep[:, 1:] &= ids[:, 1:] != ids[:, :-1]
        sizes_all.append(keep.sum(axis=1))
        ids_all.append(ids[keep].astype(np.int32))
    sizes = np.concatenate(sizes_all)
    col = np.concatenate(ids_all)
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(sizes, out=offs[1:])
    u = rng.random(len(col)) + 0.1
    rowsum = np.add.reduceat(u, offs[:-1]) if n else np.zeros(0)
    w = (u / np.repeat(rowsum, sizes)).astype(np.float32)
    return HistogramSet(offs, col, w, vocab)


def sample_rows(x: HistogramSet, n: int, seed: int = 2) -> HistogramSet:
    """Queries sampled from the resident set (the paper's protocol)."""
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(x.n_rows, size=n, replace=False))
    return x.take_rows(idx)
