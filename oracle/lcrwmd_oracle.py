"""CPU oracle for the LC-RWMD hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``movers``
(/root/reference/pkg/src/movers) for exactly the functions on the LC-RWMD
hot path.  It exists to CHECK the CUDA product, never to be it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
  ``cpu_baseline`` leg and ``--impl reference`` arm) may import it;
* nothing under ``paper_1711_07227_b200/`` imports it, and the product path
  raises when its CUDA library is missing instead of falling back here.

Parity status: PINNED.  ``tests/golden/make_golden.py`` imports the real
reference (in the build container, where /root/reference exists) and writes
its outputs on seeded inputs to ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this restatement against every one of
those vectors plus the SPEC.md known answers.

Arithmetic follows the reference: float64 Gram expansion
``sqrt(max(0, |a|^2 + |b|^2 - 2 a.b))`` rounded once to float32
(kernels.py:72-110), exact segmented minima (distances.py:177), float64
sparse products rounded once to float32 (kernels.py:174-190), and
(distance, id) lexicographic top-k (kernels.py:210-232).  The one
deliberate difference is HOW the float64 dots are formed: BLAS ``dgemm``
instead of the reference's broadcast-multiply + ``np.sum`` (kernels.py:105).
That only moves float64 round-off (~1e-16 relative), which the float32
rounding of every output absorbs; the golden tests hold it to 1e-6.

The dgemm-based blocks are distributed over all host cores with a thread
pool (each worker pinned to one BLAS thread), so the CPU baseline in
bench.py is the reference algorithm at full host parallelism.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

try:  # keep BLAS single-threaded inside pool workers
    from threadpoolctl import threadpool_limits
except Exception:  # pragma: no cover - threadpoolctl is in the image
    threadpool_limits = None


# ---------------------------------------------------------------------------
# Data model (corpus.py:100-176)
# ---------------------------------------------------------------------------

@dataclass
class CSR:
    """Histogram set in CSR form (corpus.py:100-107)."""

    row_offsets: np.ndarray  # int64 (n+1)
    column_ids: np.ndarray   # int32 (nnz)
    values: np.ndarray       # float32 (nnz)
    n_cols: int

    @property
    def n_rows(self) -> int:
        return len(self.row_offsets) - 1

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def slice_rows(self, start: int, stop: int) -> "CSR":
        """corpus.py:125-133."""
        lo, hi = int(self.row_offsets[start]), int(self.row_offsets[stop])
        return CSR(self.row_offsets[start:stop + 1] - lo, self.column_ids[lo:hi],
                   self.values[lo:hi], self.n_cols)


def as_csr(x) -> CSR:
    """Accept any object with the HistogramSet fields."""
    return CSR(np.asarray(x.row_offsets, dtype=np.int64),
               np.asarray(x.column_ids, dtype=np.int32),
               np.asarray(x.values, dtype=np.float32), int(x.n_cols))


def restrict_vocabulary(x: CSR, embeddings: np.ndarray):
    """corpus.py:405-426: drop unused words; new ids in ascending old order."""
    if x.n_rows == 0:
        raise ValueError("cannot restrict an empty histogram set")
    used = np.unique(x.column_ids)
    remap = np.full(x.n_cols, -1, dtype=np.int32)
    remap[used] = np.arange(len(used), dtype=np.int32)
    xr = CSR(x.row_offsets.copy(), remap[x.column_ids], x.values.copy(), len(used))
    return xr, np.ascontiguousarray(embeddings[used]), remap


# ---------------------------------------------------------------------------
# Phase 1 (kernels.py:66-110, distances.py:147-178)
# ---------------------------------------------------------------------------

def squared_norms(a: np.ndarray) -> np.ndarray:
    """kernels.py:66-69 (float64 row sums of squares)."""
    a64 = np.ascontiguousarray(a, dtype=np.float64)
    return np.sum(a64 * a64, axis=1)


def _row_groups(a: np.ndarray, b: np.ndarray):
    """Group ids such that two rows share a group iff they are bitwise identical."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    both = np.concatenate([a, b]).view(np.dtype((np.void, 4 * a.shape[1])))[:, 0]
    _, inv = np.unique(both, return_inverse=True)
    return inv[: len(a)], inv[len(a):]


def _euclid_block(e64, sq_e, t64, sq_t, ge=None, gt=None) -> np.ndarray:
    """kernels.py:105-109: fp64 Gram expansion, clamp, sqrt, store f32.

    The reference's identical-rows-give-exactly-zero property
    (kernels.py:91-92) comes from its norm and dot reductions coinciding
    bitwise; with BLAS dots it is restated explicitly via row groups."""
    dots = e64 @ t64.T
    sq = sq_e[:, None] + sq_t[None, :] - 2.0 * dots
    np.maximum(sq, 0.0, out=sq)
    if ge is not None:
        sq[ge[:, None] == gt[None, :]] = 0.0
    np.sqrt(sq, out=sq)
    return sq.astype(np.float32)


def _pool_map(fn, items, threads):
    if threads <= 1 or len(items) <= 1:
        return [fn(it) for it in items]

    def run(it):
        if threadpool_limits is not None:
            with threadpool_limits(1):
                return fn(it)
        return fn(it)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(run, items))


def phase1(embeddings: np.ndarray, stacked: np.ndarray, seg_offsets: np.ndarray,
           threads: int = 1, row_block: int = 512) -> np.ndarray:
    """distances.py:147-178: Z[w, j] = min_{t in seg j} |E[w] - T[t]| (v_e, b) f32.

    Segments must be non-empty (the reference's reduceat would silently
    return a wrong value for an empty one, distances.py:177)."""
    e64 = np.ascontiguousarray(embeddings, dtype=np.float64)
    t64 = np.ascontiguousarray(stacked, dtype=np.float64)
    if t64.ndim != 2 or t64.shape[1] != e64.shape[1]:
        raise ValueError(f"dimension mismatch: {e64.shape[1]} vs {t64.shape[-1]}")
    seg_offsets = np.asarray(seg_offsets, dtype=np.int64)
    if np.any(np.diff(seg_offsets) <= 0):
        raise ValueError("empty segment")
    sq_e = squared_norms(e64)
    sq_t = squared_norms(t64)
    ge, gt = _row_groups(embeddings, stacked)
    starts = seg_offsets[:-1]
    v_e = e64.shape[0]
    z = np.empty((v_e, len(starts)), dtype=np.float32)

    def block(r0):
        r1 = min(r0 + row_block, v_e)
        d = _euclid_block(e64[r0:r1], sq_e[r0:r1], t64, sq_t, ge[r0:r1], gt)
        z[r0:r1] = np.minimum.reduceat(d, starts, axis=1)

    _pool_map(block, list(range(0, v_e, row_block)), threads)
    return z


def nearest_word_distances(embeddings: np.ndarray, query_vectors: np.ndarray) -> np.ndarray:
    """distances.py:133-144."""
    q = np.atleast_2d(np.asarray(query_vectors))
    return phase1(embeddings, q, np.array([0, q.shape[0]], dtype=np.int64))[:, 0]


# ---------------------------------------------------------------------------
# Phase 2 (kernels.py:174-198)
# ---------------------------------------------------------------------------

def spmm(x: CSR, z: np.ndarray, threads: int = 1, row_block: int = 65536) -> np.ndarray:
    """kernels.py:174-190: fp64 products and per-row sums, rounded once to f32."""
    z = np.asarray(z)
    if z.ndim != 2:
        raise ValueError("spmm expects a 2-d right-hand side")
    if z.shape[0] != x.n_cols:
        raise ValueError(f"dimension mismatch: {x.n_cols} columns vs {z.shape[0]} rows")
    out = np.zeros((x.n_rows, z.shape[1]), dtype=np.float32)
    if x.n_rows == 0:
        return out
    z64 = z.astype(np.float64)
    vals = x.values.astype(np.float64)

    def block(r0):
        r1 = min(r0 + row_block, x.n_rows)
        lo, hi = int(x.row_offsets[r0]), int(x.row_offsets[r1])
        prod = vals[lo:hi, None] * z64[x.column_ids[lo:hi], :]
        acc = np.add.reduceat(prod, x.row_offsets[r0:r1] - lo, axis=0)
        out[r0:r1] = acc.astype(np.float32)

    _pool_map(block, list(range(0, x.n_rows, row_block)), threads)
    return out


# ---------------------------------------------------------------------------
# Directions and entry points (distances.py:181-264)
# ---------------------------------------------------------------------------

def one_direction(resident: CSR, resident_emb: np.ndarray, query_emb: np.ndarray,
                  queries: CSR, batch_words: int = 16384, threads: int = 1) -> np.ndarray:
    """distances.py:181-204: bounds moving resident mass to each query (n_res, n_q).

    Batches are formed by stacked-word count instead of a fixed query count;
    results are batch-invariant (distances.py docstring)."""
    out = np.empty((resident.n_rows, queries.n_rows), dtype=np.float32)
    b0 = 0
    offs = queries.row_offsets
    while b0 < queries.n_rows:
        b1 = int(np.searchsorted(offs, offs[b0] + batch_words, side="right")) - 1
        b1 = max(b1, b0 + 1)
        b1 = min(b1, queries.n_rows)
        batch = queries.slice_rows(b0, b1)
        t = query_emb[batch.column_ids]
        z = phase1(resident_emb, t, batch.row_offsets, threads=threads)
        out[:, b0:b1] = spmm(resident, z, threads=threads)
        b0 = b1
    return out


def lcrwmd_one_sided(x1, query_ids, query_weights, embeddings) -> np.ndarray:
    """distances.py:207-220."""
    x1 = as_csr(x1)
    q = CSR(np.array([0, len(query_ids)], dtype=np.int64),
            np.asarray(query_ids, dtype=np.int32), np.asarray(query_weights, dtype=np.float32),
            x1.n_cols)
    return one_direction(x1, embeddings, embeddings, q)[:, 0]


def lcrwmd_batched(x1, x2_batch, embeddings) -> np.ndarray:
    """distances.py:223-241 (no restriction, as in the reference)."""
    x1, x2 = as_csr(x1), as_csr(x2_batch)
    if x2.n_rows < 1:
        raise ValueError("batch must hold at least one query")
    return one_direction(x1, embeddings, embeddings, x2)


def lcrwmd_full(x1, x2, embeddings, threads: int = 1) -> np.ndarray:
    """distances.py:244-264: max(D1, D2^T) over per-direction restricted vocabularies."""
    x1, x2 = as_csr(x1), as_csr(x2)
    x1r, e1, _ = restrict_vocabulary(x1, embeddings)
    x2r, e2, _ = restrict_vocabulary(x2, embeddings)
    d1 = one_direction(x1r, e1, embeddings, x2, threads=threads)
    d2t = one_direction(x2r, e2, embeddings, x1, threads=threads)
    return np.maximum(d1, d2t.T)


def rwmd_quadratic(x1, x2, embeddings) -> np.ndarray:
    """distances.py:78-126 (quadratic comparator; small instances only)."""
    x1, x2 = as_csr(x1), as_csr(x2)
    e = np.asarray(embeddings)
    out = np.empty((x1.n_rows, x2.n_rows), dtype=np.float32)
    for j in range(x2.n_rows):
        lo2, hi2 = int(x2.row_offsets[j]), int(x2.row_offsets[j + 1])
        t2 = e[x2.column_ids[lo2:hi2]].astype(np.float64)
        w2 = x2.values[lo2:hi2].astype(np.float64)
        for i in range(x1.n_rows):
            lo1, hi1 = int(x1.row_offsets[i]), int(x1.row_offsets[i + 1])
            t1 = e[x1.column_ids[lo1:hi1]].astype(np.float64)
            w1 = x1.values[lo1:hi1].astype(np.float64)
            g1, g2 = _row_groups(t1.astype(np.float32), t2.astype(np.float32))
            d = _euclid_block(t1, squared_norms(t1), t2, squared_norms(t2), g1, g2)
            b1 = float(np.sum(w1 * d.min(axis=1).astype(np.float64)))
            b2 = float(np.sum(w2 * d.min(axis=0).astype(np.float64)))
            out[i, j] = max(np.float32(b1), np.float32(b2))
    return out


def rwmd_bounds(x1, x2, embeddings):
    """distances.py:78-114: (bound1, bound2) = the two one-sided bounds, (n1, n2) each.
    bound1 is the forward LC-RWMD direction, bound2 the reverse one transposed
    (the two-phase form equals the quadratic one value for value)."""
    x1, x2 = as_csr(x1), as_csr(x2)
    e = np.asarray(embeddings)
    x1r, e1, _ = restrict_vocabulary(x1, e)
    x2r, e2, _ = restrict_vocabulary(x2, e)
    return one_direction(x1r, e1, e, x2), one_direction(x2r, e2, e, x1).T


def pairwise_euclidean(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """kernels.py:113-130 (identical rows -> exactly 0, kernels.py:91-92)."""
    a = np.atleast_2d(np.asarray(a))
    b = np.atleast_2d(np.asarray(b))
    ga, gb = _row_groups(a.astype(np.float32), b.astype(np.float32))
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    return _euclid_block(a64, squared_norms(a64), b64, squared_norms(b64), ga, gb)


def centroids(x, embeddings) -> np.ndarray:
    """kernels.py:201-203 (= spmm of X by E)."""
    return spmm(as_csr(x), np.asarray(embeddings))


def wcd_block(x1, x2, embeddings) -> np.ndarray:
    """distances.py:59-71: centroid distances for all pairs."""
    return pairwise_euclidean(centroids(x1, embeddings), centroids(x2, embeddings))


# ---------------------------------------------------------------------------
# Exact mover's distance (emd.py) -- successive shortest paths, restated
# ---------------------------------------------------------------------------
EMD_FEAS_TOL = 1e-9      # emd.py:33
EMD_PRUNE_SLACK = 1e-6   # emd.py:39


def solve_emd_objective(supply, demand, cost) -> float:
    """The objective of ``solve_emd_plan``."""
    return solve_emd_plan(supply, demand, cost)[0]


def solve_emd_plan(supply, demand, cost):
    """emd.py:120-194: successive shortest augmenting paths with node potentials
    (multi-source Dijkstra over reduced costs clamped at 0, lowest-index ties);
    returns the objective.  Restated with the reference's order of operations
    and tolerances.  Where the reference raises "no augmenting path" because the
    float32-normalised totals differ by more than 1e-9 (emd.py:153-162), this
    stops once either side is exhausted -- the behaviour the CUDA solver has.
    Returns (objective, flow (h1, h2), potentials phi (h1 + h2)) -- the reference's
    plan is ``flow > 1e-9`` with dual_source = -phi[:h1], dual_sink = phi[h1:]
    (emd.py:186-194)."""
    s = np.asarray(supply, dtype=np.float64).copy()
    d = np.asarray(demand, dtype=np.float64).copy()
    c = np.ascontiguousarray(cost, dtype=np.float64)
    h1, h2 = c.shape
    n = h1 + h2
    flow = np.zeros((h1, h2))
    phi = np.zeros(n)
    while s.sum() > EMD_FEAS_TOL and d.sum() > EMD_FEAS_TOL:
        dist = np.full(n, np.inf)
        parent = np.full(n, -1, dtype=np.int64)
        dist[:h1][s > EMD_FEAS_TOL] = 0.0
        done = np.zeros(n, dtype=bool)
        for _ in range(n):
            u = int(np.argmin(np.where(done, np.inf, dist)))
            if done[u] or not np.isfinite(dist[u]):
                break
            done[u] = True
            if u < h1:
                rc = np.maximum(c[u] + phi[u] - phi[h1:], 0.0)
                cand = dist[u] + rc
                better = (cand < dist[h1:]) & ~done[h1:]
                dist[h1:][better] = cand[better]
                parent[h1:][better] = u
            else:
                q = u - h1
                rc = np.maximum(phi[u] - phi[:h1] - c[:, q], 0.0)
                cand = dist[u] + rc
                better = (flow[:, q] > EMD_FEAS_TOL) & (cand < dist[:h1]) & ~done[:h1]
                dist[:h1][better] = cand[better]
                parent[:h1][better] = u
        sink = np.where(d > EMD_FEAS_TOL, dist[h1:], np.inf)
        t = int(np.argmin(sink))
        if not np.isfinite(sink[t]):
            break
        phi += np.minimum(dist, sink[t])
        node, bott = h1 + t, d[t]
        while parent[node] != -1:
            prev = int(parent[node])
            if node < h1:
                bott = min(bott, flow[node, prev - h1])
            node = prev
        root = node
        bott = min(bott, s[root])
        node = h1 + t
        while parent[node] != -1:
            prev = int(parent[node])
            if node >= h1:
                flow[prev, node - h1] += bott
            else:
                flow[node, prev - h1] -= bott
            node = prev
        s[root] -= bott
        d[t] -= bott
    return float(np.sum(flow * c)), flow, phi


def wmd(x1_ids, x1_w, x2_ids, x2_w, embeddings) -> float:
    """emd.py:199-211: exact WMD over the pairwise word distances of the two documents."""
    e = np.asarray(embeddings)
    cost = pairwise_euclidean(e[x1_ids], e[x2_ids]).astype(np.float64)
    return solve_emd_objective(np.asarray(x1_w, np.float64), np.asarray(x2_w, np.float64), cost)


def prefiltered_topk_wmd(x1, q_ids, q_w, embeddings, k):
    """emd.py:214-261: exact top-k WMD, candidates in ascending (LC-RWMD bound, id) order,
    the k best seed a cutoff, stop at the first bound above cutoff*(1+1e-6)+1e-12."""
    x1 = as_csr(x1)
    e = np.asarray(embeddings)
    n1 = x1.n_rows
    q = CSR(np.array([0, len(q_ids)], np.int64), np.asarray(q_ids, np.int32), np.asarray(q_w, np.float32),
            x1.n_cols)
    bounds = lcrwmd_full(x1, q, e)[:, 0].astype(np.float64)
    order = np.lexsort((np.arange(n1), bounds))

    def row(i):
        lo, hi = int(x1.row_offsets[i]), int(x1.row_offsets[i + 1])
        return x1.column_ids[lo:hi], x1.values[lo:hi]

    top = []
    for idx in order[:k]:
        top.append((wmd(*row(int(idx)), q_ids, q_w, e), int(idx)))
    solves = k
    top.sort()
    cutoff = top[-1][0]
    for pos in range(k, n1):
        idx = int(order[pos])
        if bounds[idx] > cutoff * (1.0 + EMD_PRUNE_SLACK) + 1e-12:
            break
        dist = wmd(*row(idx), q_ids, q_w, e)
        solves += 1
        if (dist, idx) < top[-1]:
            top[-1] = (dist, idx)
            top.sort()
            cutoff = top[-1][0]
    return np.array([t[0] for t in top]), np.array([t[1] for t in top], np.int64), solves


# ---------------------------------------------------------------------------
# Top-k (kernels.py:210-232)
# ---------------------------------------------------------------------------

# ---------------------------------------------------------------------------
# The remaining movers.kernels primitives, restated in the form csrc/prims.cu
# computes them (pinned bitwise to tests/golden/prims.npz)
# ---------------------------------------------------------------------------
def pairwise_sum(v) -> float:
    """numpy's pairwise summation of a contiguous float64 run (what np.sum(..., axis=-1)
    does, kernels.py:69,105): < 8 terms sequential from 0.0; <= 128 terms eight
    strided partial sums ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; above,
    split at n2 = n/2 - (n/2) % 8 and add the halves."""
    v = [float(x) for x in v]
    n = len(v)
    if n < 8:
        r = 0.0
        for x in v:
            r += x
        return r
    if n <= 128:
        r = v[:8]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += v[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += v[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(v[:n2]) + pairwise_sum(v[n2:])


def squared_norms_pairwise(a) -> np.ndarray:
    """kernels.py:66-69 as pairwise sums of float64 squares."""
    a64 = np.asarray(a, dtype=np.float64)
    return np.array([pairwise_sum(r * r) for r in a64], dtype=np.float64)


def euclidean_pairwise(a64, sq_a, b64, sq_b) -> np.ndarray:
    """kernels.py:105-109 per entry: sqrt(max(0, (sq_a + sq_b) - 2 * pairwise_sum(a*b))), f64."""
    a64, b64 = np.asarray(a64, np.float64), np.asarray(b64, np.float64)
    out = np.empty((len(a64), len(b64)), dtype=np.float64)
    for i in range(len(a64)):
        for j in range(len(b64)):
            sq = (sq_a[i] + sq_b[j]) - 2.0 * pairwise_sum(a64[i] * b64[j])
            out[i, j] = np.sqrt(max(sq, 0.0)) if sq == sq else sq
    return out


def _np_min_seq(vals):
    acc = vals[0]
    for x in vals[1:]:
        acc = acc if (acc < x or acc != acc) else x
    return acc


def segmented_min_seq(values, seg_offsets, axis: int = 0) -> np.ndarray:
    """kernels.py:153-167 (np.minimum.reduceat) restated as left-to-right np.minimum
    per segment: acc = acc if (acc < x or acc is NaN) else x."""
    v = np.moveaxis(np.asarray(values), axis, 0)
    out = np.empty((len(seg_offsets) - 1,) + v.shape[1:], dtype=v.dtype)
    for s in range(len(seg_offsets) - 1):
        seg = v[seg_offsets[s]:seg_offsets[s + 1]]
        flat = seg.reshape(len(seg), -1)
        out[s] = np.array([_np_min_seq(list(flat[:, c])) for c in range(flat.shape[1])],
                          dtype=v.dtype).reshape(v.shape[1:])
    return np.moveaxis(out, 0, axis)


def topk_select(distances: np.ndarray, ids: np.ndarray, k: int):
    """kernels.py:210-223: k smallest under ascending (distance, id)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    distances = np.asarray(distances)
    ids = np.asarray(ids, dtype=np.int64)
    if distances.shape != ids.shape:
        raise ValueError("distances and ids must align")
    order = np.lexsort((ids, distances))[: min(k, len(ids))]
    return distances[order].copy(), ids[order].copy()


def topk_merge(parts, k: int):
    """kernels.py:226-232."""
    if not parts:
        return np.zeros(0, dtype=np.float32), np.zeros(0, dtype=np.int64)
    d = np.concatenate([p[0] for p in parts])
    i = np.concatenate([p[1] for p in parts])
    return topk_select(d, i, k)


def topk_per_query(dmat: np.ndarray, k: int):
    """Top-k docs for every query column of an (n1, n2) matrix: (n2,k) dists, ids."""
    n1, n2 = dmat.shape
    kk = min(k, n1)
    dist = np.empty((n2, kk), dtype=dmat.dtype)
    ids = np.empty((n2, kk), dtype=np.int64)
    ar = np.arange(n1, dtype=np.int64)
    for j in range(n2):
        d, i = topk_select(dmat[:, j], ar, kk)
        dist[j], ids[j] = d, i
    return dist, ids


def lcrwmd_topk(x1, x2, embeddings, k: int, threads: int = 1):
    """Symmetric LC-RWMD + per-query top-k (the bench workload's CPU restatement)."""
    d = lcrwmd_full(x1, x2, embeddings, threads=threads)
    return topk_per_query(d, k)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)
