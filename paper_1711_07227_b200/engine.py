"""Index lifecycle and the partitioned query driver (SPEC.md ``engine`` module).

The reference package specifies but does not ship this layer
(SURVEY §8f row 4); it is built here on the GPU kernels so a
user of the reference's functions gets the spec'd surface too:

* ``build_index`` -- ingest (tokenised docs or a corpus file), drop words
  without embeddings / stop-words, restrict the vocabulary to resident words
  (corpus.py:368-426) and keep the labels;
* ``save_index`` / ``open_index`` -- the LCRW v1 file (corpus.py:17-25) plus an
  optional labels side file (``device.load_index`` reads the same file
  straight into HBM);
* ``run_query`` -- the resident set split into P contiguous shards, the chosen
  method per shard, per-query ``topk_merge``.  Every pair
  distance is computed by shard-independent arithmetic, so the result is
  identical for every P; with ``self_exclusion`` a query's own
  resident id is dropped before the merge;
* ``benchmark`` -- JSON-lines timing records (method, n, h_mean, m, P,
  wall_ms, exact_solves).
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import corpus, device, emd
from .corpus import HistogramSet, Vocabulary
from .kernels import TopKResult, topk_merge

METHODS = ("wcd", "rwmd", "lc-rwmd", "wmd", "wmd-pruned")


@dataclass
class Index:
    """Resident set X1 over its restricted vocabulary, the matching embedding rows,
    the words, optional labels and the format version."""

    docs: HistogramSet
    embeddings: np.ndarray
    words: list[str]
    labels: list[str] | None = None
    version: int = corpus.INDEX_FORMAT_VERSION

    @property
    def vocabulary(self) -> Vocabulary:
        return Vocabulary.from_words(self.words)

    def histograms(self, docs: Sequence[Sequence[str]]) -> HistogramSet:
        """Transient documents over this index's vocabulary (out-of-index words dropped;
        documents left empty raise IngestError, as in corpus.build_histograms)."""
        hs, _ = corpus.build_histograms(docs, self.vocabulary)
        return hs


@dataclass
class QueryPlan:
    """method, k, batch size, partition count P, self-exclusion."""

    method: str = "lc-rwmd"
    k: int = 10
    batch_size: int = 32
    partitions: int = 1
    self_exclusion: bool = False

    def validate(self) -> None:
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}; expected one of {', '.join(METHODS)}")
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.partitions < 1:
            raise ValueError("partitions must be >= 1")


def build_index(docs: Sequence[Sequence[str]] | str | Path, vocab: Vocabulary, embeddings: np.ndarray,
                stopwords: frozenset[str] | None = None, labels: Sequence[str] | None = None) -> Index:
    """Ingest + restrict.  ``docs`` is a list of token lists or a corpus path."""
    if isinstance(docs, (str, Path)):
        _, docs = corpus.read_corpus(docs)
    hs, kept = corpus.build_histograms(docs, vocab, stopwords or frozenset())
    if labels is not None:
        labels = [labels[int(i)] for i in kept]
    restricted, e_r, remap = corpus.restrict_vocabulary(hs, np.asarray(embeddings, dtype=np.float32))
    used = np.flatnonzero(np.asarray(remap) >= 0)
    words = [vocab.words[int(i)] for i in used]
    return Index(restricted, np.ascontiguousarray(e_r, dtype=np.float32), words, list(labels) if labels else None)


def save_index(index: Index, path: str | Path) -> None:
    corpus.write_index_file(path, index.docs, index.embeddings, index.words)
    if index.labels is not None:
        Path(str(path) + ".labels").write_text("".join(f"{label}\n" for label in index.labels), encoding="utf-8")


def open_index(path: str | Path) -> Index:
    """Reload (bitwise round trip of every array)."""
    docs, emb, words = corpus.read_index_file(path)
    lp = Path(str(path) + ".labels")
    labels = corpus.read_labels(lp) if lp.exists() else None
    return Index(docs, emb, words, labels)


# ---------------------------------------------------------------------------
# per-shard methods: (n_q, <= kk) distances and global ids
# ---------------------------------------------------------------------------

def _shard_topk(method: str, x1: HistogramSet, base: int, x2: HistogramSet, E_t: torch.Tensor,
                prep: device.PreparedEmbeddings, kk: int) -> list[TopKResult]:
    n1, n2 = x1.n_rows, x2.n_rows
    kk = min(kk, n1)
    if method in ("lc-rwmd", "rwmd"):  # the quadratic relaxation equals LC-RWMD value for value
        d, i = device.symmetric(device.DeviceCSR.upload(x1, "x1"), device.DeviceCSR.upload(x2, "x2"), prep, kk,
                                id_offset=base)
        d, i = d.cpu().numpy(), i.cpu().numpy()
        return [TopKResult(d[j], i[j]) for j in range(n2)]
    if method == "wcd":
        c1 = device.centroids(device.DeviceCSR.upload(x1, "x1"), E_t)
        c2 = device.centroids(device.DeviceCSR.upload(x2, "x2"), E_t)
        D = device.pairwise(c2, c1)  # (n2, n1): each query's row
        od = torch.empty((n2, kk), dtype=torch.float32, device=D.device)
        oi = torch.empty((n2, kk), dtype=torch.int64, device=D.device)
        device.topk_matrix_rows(D, n2, n1, n1, base, kk, od, oi)
        od, oi = od.cpu().numpy(), oi.cpu().numpy()
        return [TopKResult(od[j], oi[j]) for j in range(n2)]
    if method == "wmd":  # exhaustive exact: every pair solved
        rows = [x1.row(i) for i in range(n1)]
        out = []
        for j in range(n2):
            q = x2.row(j)
            d = emd.solve_batch([r.weights for r in rows], [q.weights] * n1, embeddings=E_t,
                                ids1=[r.word_ids for r in rows], ids2=[q.word_ids] * n1)
            order = np.lexsort((np.arange(n1), d))[:kk]
            out.append(TopKResult(d[order], order.astype(np.int64) + base))
        return out
    if method == "wmd-pruned":
        res, _ = emd.prefiltered_topk_wmd_batch(x1, x2, E_t, kk)
        return [TopKResult(r.distances, r.ids + base) for r in res]
    raise ValueError(f"unknown method {method!r}")


def run_query(index: Index, queries: HistogramSet, plan: QueryPlan, query_ids: Sequence[int] | None = None
              ) -> list[TopKResult]:
    """Per-query top-k over the resident set, P contiguous shards merged with topk_merge
    (SPEC.md:357-365).  ``query_ids`` name each query's own resident row (X2 subset of X1)
    for ``self_exclusion``."""
    plan.validate()
    if queries.n_cols != index.docs.n_cols:
        raise ValueError(f"queries: histogram columns ({queries.n_cols}) do not match embedding rows "
                         f"({index.docs.n_cols})")
    if plan.self_exclusion and query_ids is None:
        raise ValueError("self_exclusion needs the queries' resident ids")
    n1, nq = index.docs.n_rows, queries.n_rows
    P = min(plan.partitions, n1)
    E_t = device.to_device(index.embeddings, torch.float32)
    prep = device.PreparedEmbeddings(E_t)
    kk = plan.k + (1 if plan.self_exclusion else 0)
    parts: list[list[TopKResult]] = [[] for _ in range(nq)]
    for r in range(P):
        lo, hi = n1 * r // P, n1 * (r + 1) // P
        if hi == lo:
            continue
        for j, t in enumerate(_shard_topk(plan.method, index.docs.slice_rows(lo, hi), lo, queries, E_t, prep, kk)):
            parts[j].append(t)
    out = []
    for j in range(nq):
        if plan.self_exclusion:
            own = int(query_ids[j])
            parts[j] = [TopKResult(t.distances[t.ids != own], t.ids[t.ids != own]) for t in parts[j]]
        m = topk_merge(parts[j], plan.k)
        out.append(TopKResult(np.asarray(m.distances), np.asarray(m.ids, dtype=np.int64)))
    return out


def benchmark(index: Index, queries: HistogramSet, methods: Sequence[str] = ("lc-rwmd",),
              partitions: Sequence[int] = (1,), k: int = 10, out=None) -> list[dict]:
    """JSON-lines timing records, one per (method, P)."""
    recs = []
    h_mean = float(np.mean(np.diff(index.docs.row_offsets))) if index.docs.n_rows else 0.0
    for method in methods:
        for P in partitions:
            plan = QueryPlan(method=method, k=k, partitions=P)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run_query(index, queries, plan)
            torch.cuda.synchronize()
            rec = {"method": method, "n": index.docs.n_rows, "h_mean": h_mean, "m": int(index.embeddings.shape[1]),
                   "P": P, "wall_ms": (time.perf_counter() - t0) * 1e3, "exact_solves": None}
            if method == "wmd-pruned":
                _, solves = emd.prefiltered_topk_wmd_batch(index.docs, queries, index.embeddings, k)
                rec["exact_solves"] = int(np.sum(solves))
            recs.append(rec)
            if out is not None:
                out.write(json.dumps(rec) + "\n")
    return recs
