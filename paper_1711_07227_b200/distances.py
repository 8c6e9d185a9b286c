"""LC-RWMD entry points -- drop-in for the hot path of ``movers.distances``.

Same names, signatures, return types and errors as
/root/reference/pkg/src/movers/distances.py:133-264, computed on the B200:

* Phase 1 (distances.py:147-178): tcgen05 f16 GEMM with the Gram expansion and
  segmented row-min fused in the epilogue (csrc/phase1.cu);
* Phase 2 (distances.py:203 / kernels.py:174-190): fp64-accumulating CSR SpMM
  (csrc/phase2.cu);
* symmetric combine (distances.py:264) fused into the reverse-direction SpMM.

Next to the path: ``wcd_block`` (distances.py:59-71, centroids by
the SpMM kernel + pairwise distances by the Phase-1 kernel) and
``rwmd_bounds`` / ``rwmd_quadratic`` (distances.py:78-130): the quadratic
relaxation equals the two-phase one value for value, so
both bounds come from the LC-RWMD kernels.

``lcrwmd_topk`` is the one extension: the symmetric bound reduced to each
query's k nearest resident documents without materialising the n1 x n2
matrix (the reference leaves top-k to callers, kernels.py:210-232).

Precision: operands are rounded once to f16 after an exact power-of-two
scaling (11-bit significand, the same as TF32-RN) with norms taken from the
rounded rows; the tensor cores accumulate in fp32 and identical vectors are
forced to exactly 0 as in the reference (kernels.py:91-92).  Distances match
the float64 reference within 1e-4 relative (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import numpy as np
import torch

from . import device
from .corpus import Histogram, HistogramSet
from .kernels import DEFAULT_COL_BLOCK, DEFAULT_ROW_BLOCK, DistanceBlock, TopKResult


def _check_space(x: HistogramSet, embeddings, name: str) -> None:
    """distances.py:47-52."""
    rows = embeddings.shape[0]
    if x.n_cols != rows:
        raise ValueError(f"{name}: histogram columns ({x.n_cols}) do not match embedding rows ({rows})")


def wcd_block(x1: HistogramSet, x2: HistogramSet, embeddings: np.ndarray, row_block: int = DEFAULT_ROW_BLOCK,
              col_block: int = DEFAULT_COL_BLOCK) -> DistanceBlock:
    """Word centroid distances for all pairs, (n1, n2) (distances.py:59-71)."""
    _check_space(x1, embeddings, "x1")
    _check_space(x2, embeddings, "x2")
    E = device.to_device(np.asarray(embeddings, dtype=np.float32), torch.float32)
    c1 = device.centroids(device.DeviceCSR.upload(x1, "x1"), E)
    c2 = device.centroids(device.DeviceCSR.upload(x2, "x2"), E)
    return DistanceBlock(device.pairwise(c1, c2).cpu().numpy())


def rwmd_bounds(x1: HistogramSet, x2: HistogramSet, embeddings: np.ndarray, row_block: int = DEFAULT_ROW_BLOCK,
                col_block: int = DEFAULT_COL_BLOCK) -> tuple[np.ndarray, np.ndarray]:
    """Both one-sided relaxation bounds for all pairs as (n1, n2) f32 arrays (distances.py:78-114):
    bound1 = x1 rows' mass to the nearest words of each x2 row, bound2 the swapped direction."""
    _check_space(x1, embeddings, "x1")
    _check_space(x2, embeddings, "x2")
    prep = device.PreparedEmbeddings(embeddings)
    dx1, dx2 = device.DeviceCSR.upload(x1, "x1"), device.DeviceCSR.upload(x2, "x2")
    b1 = device.one_sided_rows(dx1, dx2, prep).cpu().numpy()
    b2 = device.reverse_rows(dx1, dx2, prep).cpu().numpy()
    return b1, b2


def rwmd_quadratic(x1: HistogramSet, x2: HistogramSet, embeddings: np.ndarray, row_block: int = DEFAULT_ROW_BLOCK,
                   col_block: int = DEFAULT_COL_BLOCK) -> DistanceBlock:
    """Symmetric relaxed bound max(bound1, bound2) (distances.py:117-130)."""
    b1, b2 = rwmd_bounds(x1, x2, embeddings, row_block, col_block)
    return DistanceBlock(np.maximum(b1, b2))


def nearest_word_distances(embeddings: np.ndarray, query_vectors: np.ndarray,
                           row_block: int = DEFAULT_ROW_BLOCK, col_block: int = DEFAULT_COL_BLOCK) -> np.ndarray:
    """Phase 1 for one query: z[w] = distance from word w to its closest query word (distances.py:133-144)."""
    q = np.atleast_2d(np.asarray(query_vectors, dtype=np.float32))
    e = np.asarray(embeddings, dtype=np.float32)
    if q.shape[1] != e.shape[1]:
        raise ValueError(f"dimension mismatch: {e.shape[1]} vs {q.shape[1]}")
    if q.shape[0] == 0:
        raise ValueError("empty segment")
    return device.nearest_word_distances(e, q).cpu().numpy()


QUERY_BATCH = 4096  # queries per forward pass above which the one-sided bound runs in batches


def _one_sided_device(x1: HistogramSet, queries: HistogramSet, embeddings) -> np.ndarray:
    """(n1, n_q) forward bounds; query sets above QUERY_BATCH in batches (distances.py:198-203:
    batching never changes a value), so Z1 stays bounded for any query count."""
    if x1.n_rows == 0:
        return np.zeros((0, queries.n_rows), dtype=np.float32)
    prep = device.PreparedEmbeddings(embeddings)
    dx1 = device.DeviceCSR.upload(x1, "x1")
    dq = device.DeviceCSR.upload(queries, "queries")
    res = device.Restricted.build(dx1, prep)
    if queries.n_rows > QUERY_BATCH:
        D = torch.empty((x1.n_rows, queries.n_rows), dtype=torch.float32, device=res.A.device)
        device.forward_rows_into(res, prep, dq, D, QUERY_BATCH)
        return D.cpu().numpy()
    out = device.one_direction(res, prep, dq, layout="rows")
    return out[: x1.n_rows * queries.n_rows].view(x1.n_rows, queries.n_rows).cpu().numpy()


def lcrwmd_one_sided(x1: HistogramSet, query: Histogram, embeddings: np.ndarray,
                     row_block: int = DEFAULT_ROW_BLOCK, col_block: int = DEFAULT_COL_BLOCK) -> np.ndarray:
    """First-direction bound from one query to every x1 row, length n1 (distances.py:207-220)."""
    qset = HistogramSet.from_rows([(query.word_ids, query.weights)], x1.n_cols)
    _check_space(x1, embeddings, "resident")
    return _one_sided_device(x1, qset, embeddings)[:, 0]


def lcrwmd_batched(x1: HistogramSet, x2_batch: HistogramSet, embeddings: np.ndarray,
                   row_block: int = DEFAULT_ROW_BLOCK, col_block: int = DEFAULT_COL_BLOCK) -> np.ndarray:
    """One-sided bounds for a batch of queries, (n1, b) (distances.py:223-241).

    The reference skips vocabulary restriction here; restricting never changes
    a value (corpus.py:411-413), so the GPU path always restricts."""
    if x2_batch.n_rows < 1:
        raise ValueError("batch must hold at least one query")
    _check_space(x1, embeddings, "resident")
    return _one_sided_device(x1, x2_batch, embeddings)


def lcrwmd_full(x1: HistogramSet, x2: HistogramSet, embeddings: np.ndarray, batch_size: int = 32,
                row_block: int = DEFAULT_ROW_BLOCK, col_block: int = DEFAULT_COL_BLOCK) -> DistanceBlock:
    """Symmetric relaxed bound for all pairs, (n1, n2) (distances.py:244-264).

    ``batch_size`` is accepted for compatibility; query batching never changes
    results (distances.py:198-203) and the GPU processes all queries at once."""
    _check_space(x1, embeddings, "x1")
    _check_space(x2, embeddings, "x2")
    prep = device.PreparedEmbeddings(embeddings)
    d = device.symmetric(device.DeviceCSR.upload(x1, "x1"), device.DeviceCSR.upload(x2, "x2"), prep, None)
    return DistanceBlock(d.cpu().numpy())


def lcrwmd_topk(x1: HistogramSet, x2: HistogramSet, embeddings: np.ndarray, k: int) -> list[TopKResult]:
    """Symmetric LC-RWMD top-k: for each x2 row, its k nearest x1 rows under
    ascending (distance, id) -- ``topk_select`` over each column of
    ``lcrwmd_full(x1, x2, E)`` without materialising it."""
    if k < 1:
        raise ValueError("k must be >= 1")
    _check_space(x1, embeddings, "x1")
    _check_space(x2, embeddings, "x2")
    d, i = lcrwmd_topk_arrays(x1, x2, embeddings, k)
    return [TopKResult(d[j], i[j]) for j in range(x2.n_rows)]


def lcrwmd_all_pairs_topk(x: HistogramSet, embeddings: np.ndarray, k: int, batch_size: int = 4096
                          ) -> list[TopKResult]:
    """Each row's k nearest rows of the same set under the symmetric bound
    (= ``lcrwmd_topk(x, x, E, k)``; a row is its own nearest at distance 0).
    Extension for all-pairs clustering (BASELINE configs[4]): only the forward
    direction is computed, the reverse one being its transpose."""
    if k < 1:
        raise ValueError("k must be >= 1")
    _check_space(x, embeddings, "x")
    prep = device.PreparedEmbeddings(embeddings)
    D = device.all_pairs(device.DeviceCSR.upload(x, "x"), prep, batch_size)
    n = x.n_rows
    kk = min(k, n)
    od = torch.empty((max(n, 1), k), dtype=torch.float32, device=D.device)
    oi = torch.empty((max(n, 1), k), dtype=torch.int64, device=D.device)
    device.topk_matrix_rows(D, n, n, n, 0, k, od, oi)
    od, oi = od[:, :kk].cpu().numpy(), oi[:, :kk].cpu().numpy()
    return [TopKResult(od[j], oi[j]) for j in range(n)]


def lcrwmd_topk_arrays(x1, x2, embeddings, k: int, prep=None):
    """(n2, min(k, n1)) distances and int64 ids; accepts host sets or DeviceCSRs."""
    # E first (the query-side work needs only E and X2), then the resident set -- the big
    # copy -- over a side stream while E and the query side are prepared; device.symmetric
    # waits for X1 only where it is first read
    if prep is None and not isinstance(embeddings, torch.Tensor):
        embeddings = device.to_device(np.asarray(embeddings, dtype=np.float32), torch.float32)
    if not isinstance(x1, device.DeviceCSR):
        side = _copy_stream()
        side.wait_stream(torch.cuda.current_stream())  # after E's copy: it is needed first
        x1 = device.DeviceCSR.upload(x1, "x1", stream=side)
    dx1 = x1
    if prep is None:
        prep = device.PreparedEmbeddings(embeddings)
    dx2 = x2 if isinstance(x2, device.DeviceCSR) else device.DeviceCSR.upload(x2, "x2")
    d, i = device.symmetric(dx1, dx2, prep, k)
    return d.cpu().numpy(), i.cpu().numpy()


_COPY_STREAMS: dict = {}


def _copy_stream():
    dev = device.require_cuda()
    if dev.index not in _COPY_STREAMS:
        _COPY_STREAMS[dev.index] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[dev.index]
