"""Compute primitives -- drop-in for the hot-path part of ``movers.kernels``.

Same names, signatures, result types and error messages as
/root/reference/pkg/src/movers/kernels.py; the arithmetic runs in sm_100a
kernels through the C ABI (include/lcrwmd.h):

* ``spmm`` / ``spmv``            -> lcrw_spmm (kernels.py:174-198): fp64 products and
                                    row sums in ascending nonzero order, rounded once
                                    to f32 -- bitwise equal to the reference for equal z.
* ``topk_select`` / ``topk_merge`` -> lcrw_topk_segments / lcrw_topk_sort
                                    (kernels.py:210-232): ascending (distance, id).
* ``pairwise_euclidean``           -> lcrw_phase1 with one segment per b row
                                    (kernels.py:113-130), f16 operands as on the hot path.
* ``centroids``                    -> lcrw_spmm of X by E (kernels.py:201-203), bitwise.

``row_block`` / ``col_block`` are accepted for compatibility; tiling never
changes results (kernels.py:6-10) and the GPU tiles are compile-time.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .corpus import HistogramSet

DEFAULT_ROW_BLOCK = 256
DEFAULT_COL_BLOCK = 256


@dataclass
class DistanceBlock:
    """Dense block of pairwise distances with its global index ranges (kernels.py:30-44)."""

    values: np.ndarray
    row_start: int = 0
    col_start: int = 0

    @property
    def row_ids(self) -> range:
        return range(self.row_start, self.row_start + self.values.shape[0])

    @property
    def col_ids(self) -> range:
        return range(self.col_start, self.col_start + self.values.shape[1])


@dataclass
class TopKResult:
    """Per-query nearest documents, ascending by (distance, id) (kernels.py:47-55)."""

    distances: np.ndarray
    ids: np.ndarray

    def __len__(self) -> int:
        return len(self.ids)


def _z_panels(z: np.ndarray) -> tuple[np.ndarray, int]:
    """Row-major (v, b) -> the 8-column panel layout the kernels read."""
    v, b = z.shape
    nb = (b + 7) // 8
    zp = np.zeros((nb * 8, v), dtype=np.float32)
    zp[:b] = z.T
    return np.ascontiguousarray(zp.reshape(nb, 8, v).transpose(0, 2, 1)).reshape(-1), 8 * v


def spmm(x: HistogramSet, z: np.ndarray) -> np.ndarray:
    """CSR x dense: out[i] = sum_p x[i][p] * z[p], float32 (n, b) (kernels.py:174-190)."""
    z = np.asarray(z)
    if z.ndim != 2:
        raise ValueError("spmm expects a 2-d right-hand side")
    if z.shape[0] != x.n_cols:
        raise ValueError(f"dimension mismatch: {x.n_cols} columns vs {z.shape[0]} rows")
    if x.n_rows == 0:
        return np.zeros((0, z.shape[1]), dtype=np.float32)
    b = z.shape[1]
    if b == 0:
        return np.zeros((x.n_rows, 0), dtype=np.float32)
    dx = device.DeviceCSR.upload(x, "x")
    zp, z_panel = _z_panels(np.asarray(z, dtype=np.float32))
    zd = device.to_device(zp, torch.float32)
    out = torch.empty(x.n_rows * b, dtype=torch.float32, device=zd.device)
    device.spmm(dx.offsets, dx.cols, dx.vals, x.n_rows, zd, z_panel, b, out, b, 8)
    return out.view(x.n_rows, b).cpu().numpy()


def spmv(x: HistogramSet, z: np.ndarray) -> np.ndarray:
    """CSR x vector; identical to the matching spmm column bitwise (kernels.py:193-198)."""
    z = np.asarray(z)
    if z.ndim != 1:
        raise ValueError("spmv expects a 1-d right-hand side")
    return spmm(x, z[:, None])[:, 0]


def pairwise_euclidean(a: np.ndarray, b: np.ndarray, row_block: int = DEFAULT_ROW_BLOCK,
                       col_block: int = DEFAULT_COL_BLOCK, row_start: int = 0, col_start: int = 0) -> DistanceBlock:
    """All-pairs Euclidean distances between the rows of a and b (kernels.py:113-130)."""
    a = np.atleast_2d(np.asarray(a))
    b = np.atleast_2d(np.asarray(b))
    if a.shape[1] != b.shape[1]:
        raise ValueError(f"dimension mismatch: {a.shape[1]} vs {b.shape[1]}")
    ad = device.to_device(np.asarray(a, dtype=np.float32), torch.float32)
    bd = device.to_device(np.asarray(b, dtype=np.float32), torch.float32)
    return DistanceBlock(device.pairwise(ad, bd).cpu().numpy(), row_start=row_start, col_start=col_start)


def centroids(x: HistogramSet, embeddings: np.ndarray) -> np.ndarray:
    """Weighted average of each row's embedding vectors, float32 (n, m) (kernels.py:201-203)."""
    e = np.asarray(embeddings)
    if e.shape[0] != x.n_cols:
        raise ValueError(f"dimension mismatch: {x.n_cols} columns vs {e.shape[0]} rows")
    if x.n_rows == 0:
        return np.zeros((0, e.shape[1]), dtype=np.float32)
    return device.centroids(device.DeviceCSR.upload(x, "x"), device.to_device(e, torch.float32)).cpu().numpy()


def topk_select(distances: np.ndarray, ids: np.ndarray, k: int) -> TopKResult:
    """The k smallest candidates under ascending (distance, id) (kernels.py:210-223)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    distances = np.asarray(distances)
    ids = np.asarray(ids, dtype=np.int64)
    if distances.shape != ids.shape:
        raise ValueError("distances and ids must align")
    n = distances.size
    if n == 0:
        return TopKResult(distances.astype(distances.dtype).copy(), ids.copy())
    dd = device.to_device(np.asarray(distances, dtype=np.float32).reshape(-1), torch.float32)
    di = device.to_device(ids.reshape(-1), torch.int64)
    if k <= 1024:
        od, oi = device.topk_rows(dd, di, 1, n, k)
        od, oi = od[0], oi[0]
    else:
        od, oi = device.topk_sort(dd, di, k)
    return TopKResult(od.cpu().numpy().astype(distances.dtype, copy=False), oi.cpu().numpy())


def topk_merge(parts: list[TopKResult], k: int) -> TopKResult:
    """Merge per-shard results; equals topk_select on the concatenation (kernels.py:226-232)."""
    if not parts:
        return TopKResult(np.zeros(0, dtype=np.float32), np.zeros(0, dtype=np.int64))
    d = np.concatenate([p.distances for p in parts])
    i = np.concatenate([p.ids for p in parts])
    return topk_select(d, i, k)
