"""Compute primitives -- drop-in for the hot-path part of ``movers.kernels``.

Same names, signatures, result types and error messages as
/root/reference/pkg/src/movers/kernels.py; the arithmetic runs in sm_100a
kernels through the C ABI (include/lcrwmd.h):

* ``spmm`` / ``spmv``            -> lcrw_spmm (kernels.py:174-198): fp64 products and
                                    row sums in ascending nonzero order, rounded once
                                    to f32 -- bitwise equal to the reference for equal z.
* ``topk_select`` / ``topk_merge`` -> lcrw_topk_segments / lcrw_topk_sort (f32) and
                                    lcrw_topk_sort_any (any other numeric dtype, kept as
                                    is) (kernels.py:210-232): ascending (distance, id).
* ``squared_norms`` / ``euclidean_into`` -> lcrw_squared_norms / lcrw_euclidean_f64
                                    (kernels.py:66-110): the reference's float64
                                    arithmetic bit for bit (numpy pairwise sums).
* ``row_min`` / ``col_min`` / ``segmented_min`` -> lcrw_segmented_min (kernels.py:137-167).
* ``pairwise_euclidean``           -> lcrw_phase1 with one segment per b row
                                    (kernels.py:113-130), f16 operands as on the hot path.
* ``centroids``                    -> lcrw_spmm of X by E (kernels.py:201-203), bitwise.

``row_block`` / ``col_block`` are accepted for compatibility; tiling never
changes results (kernels.py:6-10) and the GPU tiles are compile-time.
"""

from __future__ import annotations

import ctypes as C
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


# numpy dtype -> lcrw_dtype code of include/lcrwmd.h (bool travels as uint8)
_DTYPE_CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.float16): 2,
                np.dtype(np.int8): 3, np.dtype(np.int16): 4, np.dtype(np.int32): 5, np.dtype(np.int64): 6,
                np.dtype(np.uint8): 7, np.dtype(np.uint16): 8, np.dtype(np.uint32): 9, np.dtype(np.uint64): 10,
                np.dtype(np.bool_): 7}


def _dtype_code(dt: np.dtype) -> int:
    code = _DTYPE_CODES.get(np.dtype(dt))
    if code is None:
        raise TypeError(f"unsupported dtype {np.dtype(dt)} (numeric dtypes only)")
    return code


def _raw_device(a: np.ndarray) -> torch.Tensor:
    """The bytes of a C-contiguous host array on the device (any dtype)."""
    a = np.ascontiguousarray(a)
    return device.to_device(a.reshape(-1).view(np.uint8), torch.uint8)


def _raw_host(t: torch.Tensor, dtype, shape) -> np.ndarray:
    return t.cpu().numpy().view(np.dtype(dtype)).reshape(shape)


def squared_norms(a: np.ndarray) -> np.ndarray:
    """Float64 squared row norms (kernels.py:66-69), bitwise equal to the reference:
    float64 products reduced with numpy's pairwise summation (lcrw_squared_norms)."""
    a = np.asarray(a)
    if a.ndim != 2:
        raise ValueError("squared_norms expects a 2-d (rows, m) array")
    rows, m = a.shape
    if rows == 0:
        return np.zeros(0, dtype=np.float64)
    if a.dtype != np.float32:
        a = np.ascontiguousarray(a, dtype=np.float64)
    ad = device.to_device(a, torch.float32 if a.dtype == np.float32 else torch.float64)
    out = torch.empty(rows, dtype=torch.float64, device=ad.device)
    device._lib.call("lcrw_squared_norms", device._p(ad), 0 if a.dtype == np.float32 else 1, rows, m,
                     device._p(out), device._stream())
    return out.cpu().numpy()


def euclidean_into(a64: np.ndarray, sq_a: np.ndarray, b64: np.ndarray, sq_b: np.ndarray, out: np.ndarray,
                   row_block: int = DEFAULT_ROW_BLOCK, col_block: int = DEFAULT_COL_BLOCK) -> np.ndarray:
    """Fill ``out`` (r x c) with sqrt(max(0, |a|^2 + |b|^2 - 2 a.b)) from the given squared
    norms (kernels.py:72-110), bitwise equal to the reference (float64 dots with numpy's
    pairwise summation, lcrw_euclidean_f64); tiles never change results."""
    r, m = a64.shape
    c = b64.shape[0]
    if b64.shape[1] != m:
        raise ValueError(f"dimension mismatch: {m} vs {b64.shape[1]}")
    if out.dtype not in (np.float32, np.float64):
        raise TypeError("euclidean_into: out must be float32 or float64")
    if r == 0 or c == 0:
        return out
    f64 = torch.float64
    ad = device.to_device(np.ascontiguousarray(a64, dtype=np.float64), f64)
    bd = device.to_device(np.ascontiguousarray(b64, dtype=np.float64), f64)
    sa = device.to_device(np.ascontiguousarray(sq_a, dtype=np.float64).reshape(-1), f64)
    sb = device.to_device(np.ascontiguousarray(sq_b, dtype=np.float64).reshape(-1), f64)
    od = torch.empty((r, c), dtype=torch.float32 if out.dtype == np.float32 else f64, device=ad.device)
    device._lib.call("lcrw_euclidean_f64", device._p(ad), device._p(sa), r, device._p(bd), device._p(sb), c, m,
                     device._p(od), 0 if out.dtype == np.float32 else 1, c, device._stream())
    out[...] = od.cpu().numpy()
    return out


def _block_values(block) -> np.ndarray:
    return block.values if isinstance(block, DistanceBlock) else np.asarray(block)


def _axis_min(values: np.ndarray, axis: int, seg_offsets: np.ndarray | None) -> np.ndarray:
    """np.minimum over ``axis`` (whole axis, or reduceat segments) on the device."""
    code = _dtype_code(values.dtype)
    shape = values.shape
    outer = int(np.prod(shape[:axis], dtype=np.int64))
    n = int(shape[axis])
    inner = int(np.prod(shape[axis + 1:], dtype=np.int64))
    n_seg = 1 if seg_offsets is None else len(seg_offsets) - 1
    out_shape = shape[:axis] + ((n_seg,) if seg_offsets is not None else ()) + shape[axis + 1:]
    vd = _raw_device(values)
    od = torch.empty(max(1, outer * n_seg * inner) * values.dtype.itemsize, dtype=torch.uint8, device=vd.device)
    sd = None if seg_offsets is None else device.to_device(np.asarray(seg_offsets, np.int64), torch.int64)
    device._lib.call("lcrw_segmented_min", device._p(vd), code, outer, n, inner, device._p(sd), n_seg,
                     device._p(od), device._stream())
    return _raw_host(od[: outer * n_seg * inner * values.dtype.itemsize], values.dtype, out_shape)


def row_min(block) -> np.ndarray:
    """Exact minimum of each row (kernels.py:137-142)."""
    values = _block_values(block)
    if values.size == 0:
        raise ValueError("row_min of an empty block")
    if values.ndim < 2:
        raise np.exceptions.AxisError(1, values.ndim)
    return _axis_min(values, 1, None)


def col_min(block) -> np.ndarray:
    """Exact minimum of each column (kernels.py:145-150)."""
    values = _block_values(block)
    if values.size == 0:
        raise ValueError("col_min of an empty block")
    return _axis_min(values, 0, None)


def segmented_min(values: np.ndarray, seg_offsets: np.ndarray, axis: int = 0) -> np.ndarray:
    """Per-segment minima along ``axis`` for contiguous CSR-style segments (kernels.py:153-167)."""
    values = np.asarray(values)
    seg_offsets = np.asarray(seg_offsets, dtype=np.int64)
    if len(seg_offsets) < 2:
        raise ValueError("need at least one segment")
    if np.any(np.diff(seg_offsets) <= 0):
        raise ValueError("empty segment")
    ax = axis + values.ndim if axis < 0 else axis
    if not 0 <= ax < values.ndim:
        raise np.exceptions.AxisError(axis, values.ndim)
    if seg_offsets[-1] != values.shape[ax]:
        raise ValueError("segment offsets do not cover the reduced axis")
    if seg_offsets[0] < 0:
        raise IndexError(f"index {int(seg_offsets[0])} out-of-bounds in minimum.reduceat")
    # reduceat semantics: segment s = [start_s, start_{s+1}), the last one to the end of the axis
    return _axis_min(values, ax, seg_offsets)


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
        return TopKResult(distances.reshape(-1).copy(), ids.reshape(-1).copy())
    di = device.to_device(ids.reshape(-1), torch.int64)
    if distances.dtype == np.float32:
        dd = device.to_device(distances.reshape(-1), torch.float32)
        if k <= 1024:
            od, oi = device.topk_rows(dd, di, 1, n, k)
            od, oi = od[0], oi[0]
        else:
            od, oi = device.topk_sort(dd, di, k)
        return TopKResult(od.cpu().numpy(), oi.cpu().numpy())
    # any other dtype keeps its values and order (np.lexsort on the caller's dtype)
    code = _dtype_code(distances.dtype)
    dd = _raw_device(distances)
    kk = min(k, n)
    ws_bytes = C.c_size_t(0)
    device._lib.call("lcrw_topk_sort_any_workspace", n, C.byref(ws_bytes))
    ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=dd.device)
    od = torch.empty(kk * distances.dtype.itemsize, dtype=torch.uint8, device=dd.device)
    oi = torch.empty(kk, dtype=torch.int64, device=dd.device)
    device._lib.call("lcrw_topk_sort_any", device._p(dd), code, device._p(di), n, k, device._p(od), device._p(oi),
                     device._p(ws), ws_bytes.value, device._stream())
    return TopKResult(_raw_host(od, distances.dtype, (kk,)), oi.cpu().numpy())


def topk_merge(parts: list[TopKResult], k: int) -> TopKResult:
    """Merge per-shard results; equals topk_select on the concatenation (kernels.py:226-232)."""
    if not parts:
        return TopKResult(np.zeros(0, dtype=np.float32), np.zeros(0, dtype=np.int64))
    d = np.concatenate([p.distances for p in parts])
    i = np.concatenate([p.ids for p in parts])
    return topk_select(d, i, k)
