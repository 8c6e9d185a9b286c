"""HBM-resident data and the LC-RWMD pipeline over the C ABI.

PyTorch is used only as plumbing here: it owns device memory (caching
allocator), the current stream and host<->device copies.  Every arithmetic
step of the path is one of our sm_100a kernels, invoked through ``_lib``.

Pipeline for ``lcrwmd_topk`` / ``lcrwmd_full`` (distances.py:244-264):

  prepare E   f16 operand rows (power-of-two scaled), fp32 norms, identity classes
  restrict    x1 -> (remap1, used1);  x2 -> (remap2, used2)       corpus.py:405-426
  forward     Z1 = phase1(E[used1], E[x2 words]) ; D1 = spmm(x1r, Z1)   distances.py:262
  reverse     per doc batch: Z2 = phase1(E[used2], E[batch words]);
              D = max(D1, spmm(x2r, Z2)) -> per-(query, chunk) top-k  distances.py:263-264
  merge       per-query top-k over the chunk candidates            kernels.py:210-232
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .corpus import CorpusError, HistogramSet

# ---------------------------------------------------------------------------
# plumbing
# ---------------------------------------------------------------------------


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1711_07227_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def _p(t) -> C.c_void_p | None:
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def sm_count() -> int:
    out = C.c_int(0)
    _lib.call("lcrw_sm_count", C.byref(out))
    return out.value


def padded_dim(m: int) -> int:
    return int(_lib.value("lcrw_padded_dim", m))


def to_device(a, dtype, non_blocking: bool = True) -> torch.Tensor:
    """Host array -> device tensor (async when the host buffer is pinned)."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype, non_blocking=non_blocking).contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    if non_blocking and not t.is_pinned() and t.numel():
        # stage through torch's caching pinned allocator: a pageable copy would wait for
        # every kernel already queued on the stream and leave the GPU idle meanwhile
        t = t.pin_memory()
    return t.to(dev, non_blocking=non_blocking and t.is_pinned())




# ---------------------------------------------------------------------------
# resident data
# ---------------------------------------------------------------------------


@dataclass
class DeviceCSR:
    """A HistogramSet in HBM (int64 offsets, int32 ids, f32 weights) plus host offsets for planning.

    The host copies of ids and weights (query-side planning of the reverse pass) are the
    caller's own arrays when uploaded from a HistogramSet (no copy), else read back from
    the device on first use (``host_ids``)."""

    offsets: torch.Tensor
    cols: torch.Tensor
    vals: torch.Tensor
    n_cols: int
    host_offsets: np.ndarray
    host_cols: np.ndarray | None = None
    host_vals: np.ndarray | None = None
    ready: "torch.cuda.Event | None" = None  # set when uploaded on a side stream

    def wait(self) -> None:
        """Make the current stream wait for a side-stream upload (no host sync)."""
        if self.ready is not None:
            cur = torch.cuda.current_stream()
            cur.wait_event(self.ready)
            for t in (self.offsets, self.cols, self.vals):
                t.record_stream(cur)
            self.ready = None

    @property
    def n_rows(self) -> int:
        return len(self.host_offsets) - 1

    @property
    def nnz(self) -> int:
        return int(self.host_offsets[-1])

    def host_ids(self) -> tuple[np.ndarray, np.ndarray]:
        """(ids int32, weights f32) on the host (one device->host read if not kept)."""
        if self.host_cols is None or self.host_vals is None:
            self.host_cols = self.cols.cpu().numpy()
            self.host_vals = self.vals.cpu().numpy()
        return self.host_cols, self.host_vals

    def slice_rows(self, r0: int, r1: int) -> "DeviceCSR":
        """Rows [r0, r1) as a DeviceCSR sharing the id / weight storage (offsets rebased)."""
        lo, hi = int(self.host_offsets[r0]), int(self.host_offsets[r1])
        ho = self.host_offsets[r0:r1 + 1] - lo
        return DeviceCSR(self.offsets[r0:r1 + 1] - lo, self.cols[lo:hi], self.vals[lo:hi], self.n_cols, ho,
                         None if self.host_cols is None else self.host_cols[lo:hi],
                         None if self.host_vals is None else self.host_vals[lo:hi])

    @classmethod
    def upload(cls, x: HistogramSet, name: str = "x", stream: "torch.cuda.Stream | None" = None) -> "DeviceCSR":
        """Copy to HBM (async from pinned arrays).  With ``stream`` the copies run there and
        the set's first device use (``wait``) orders the consuming stream after them."""
        offs = np.asarray(x.row_offsets, dtype=np.int64)
        if x.n_rows and np.any(np.diff(offs) <= 0):
            raise CorpusError(f"{name}: every row must hold at least one word")
        if int(offs[0]) != 0 or len(x.column_ids) != int(offs[-1]) or len(x.values) != int(offs[-1]):
            raise CorpusError(f"{name}: offset/array length mismatch")
        cols = np.asarray(x.column_ids, dtype=np.int32)
        vals = np.asarray(x.values, dtype=np.float32)
        if stream is None:
            return cls(to_device(offs, torch.int64), to_device(cols, torch.int32), to_device(vals, torch.float32),
                       int(x.n_cols), offs, cols, vals)
        require_cuda()
        with torch.cuda.stream(stream):
            d = (to_device(offs, torch.int64), to_device(cols, torch.int32), to_device(vals, torch.float32))
            ev = torch.cuda.Event()
            ev.record(stream)
        return cls(*d, int(x.n_cols), offs, cols, vals, ready=ev)


class PreparedEmbeddings:
    """E in HBM: f32 original, f16 operand rows, norms, scale and identity classes.

    For m <= SPLIT_MAX_DIM the operand rows use the "3 x f16" split layout
    (K = 3m: A rows [hi, hi, lo], B rows [hi, lo, hi]) -- ~22-bit operands at
    no extra cost, because K is padded to 64 anyway; above it, one f16 pass
    (11-bit significand, like TF32-RN) whose distance error shrinks like
    1/sqrt(m).

    ``extra`` arrays (e.g. free query vectors for nearest_word_distances)
    take part in the power-of-two scale choice so they share E's scaling."""

    SPLIT_MAX_DIM = 64

    def __init__(self, embeddings, extra=(), split: bool | None = None):
        dev = require_cuda()
        st = _stream()
        self.E32 = to_device(np.asarray(embeddings, dtype=np.float32) if not isinstance(embeddings, torch.Tensor)
                             else embeddings, torch.float32)
        if self.E32.dim() != 2:
            raise ValueError("embeddings must be a 2-d (v, m) matrix")
        self.V, self.m = int(self.E32.shape[0]), int(self.E32.shape[1])
        self.split = (self.m <= self.SPLIT_MAX_DIM) if split is None else bool(split)
        self.k_eff = int(_lib.value("lcrw_operand_k", self.m, int(self.split)))
        self.kp = padded_dim(self.k_eff)
        mx = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("lcrw_max_sqnorm", _p(self.E32), self.V, self.m, _p(mx), st)
        for x in extra:
            _lib.call("lcrw_max_sqnorm", _p(x), int(x.shape[0]), self.m, _p(mx), st)
        self.scale = torch.empty(2, dtype=torch.float32, device=dev)
        _lib.call("lcrw_scale_from_max_sqnorm", _p(mx), _p(self.scale), st)
        # A side (vocabulary rows): [x, 1, 1, 1]; B side (query words): [-2x, |x|^2 pieces]
        self.EhA, self.norms = self._rows(self.E32, int(self.split))
        self.EhB = self._rows(self.E32, 2 + int(self.split), norms=False)[0]
        # exact-identity classes (kernels.py:91-92 semantics)
        ws_bytes = C.c_size_t(0)
        _lib.call("lcrw_row_classes_workspace", self.V, C.byref(ws_bytes))
        ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=dev)
        self.canon = torch.empty(self.V, dtype=torch.int32, device=dev)
        self.next = torch.empty(self.V, dtype=torch.int32, device=dev)
        self.sorted_hash = torch.empty(self.V, dtype=torch.int64, device=dev)
        self.sorted_ids = torch.empty(self.V, dtype=torch.int32, device=dev)
        n_dup = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.call("lcrw_row_classes", _p(self.E32), self.V, self.m, _p(self.canon), _p(self.next), _p(n_dup),
                  _p(self.sorted_hash), _p(self.sorted_ids), _p(ws), ws_bytes.value, st)
        self.n_dup = int(n_dup.item())

    def _rows(self, X: torch.Tensor, layout: int, norms: bool = True):
        n = int(X.shape[0])
        Xh = torch.empty((max(n, 1), self.kp), dtype=torch.float16, device=X.device)
        xn = torch.empty(max(n, 1), dtype=torch.float32, device=X.device) if norms else None
        _lib.call("lcrw_prepare_rows", _p(X), n, self.m, self.kp, layout, _p(self.scale), _p(Xh), _p(xn),
                  _stream())
        return Xh, xn

    def prepare_free_rows(self, Q: torch.Tensor) -> torch.Tensor:
        """B-side f16 operand rows for vectors that are not rows of E (same scale)."""
        return self._rows(Q, 2 + int(self.split), norms=False)[0]

    def representatives(self, word_ids: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor | None]:
        """(rep, next) arguments of lcrw_zero_identical for rows given by E ids."""
        if self.n_dup == 0:
            return word_ids, None
        rep = torch.empty_like(word_ids)
        _lib.call("lcrw_remap_ids", _p(word_ids), word_ids.numel(), _p(self.canon), _p(rep), _stream())
        return rep, self.next


# ---------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------


def restrict(cols: torch.Tensor, n_cols: int) -> tuple[torch.Tensor, torch.Tensor, int]:
    """(remap, used[:n_used], n_used) of corpus.py:405-426 (reads back one scalar)."""
    dev = cols.device
    ws_bytes = C.c_size_t(0)
    _lib.call("lcrw_restrict_workspace", n_cols, C.byref(ws_bytes))
    ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=dev)
    remap = torch.empty(n_cols, dtype=torch.int32, device=dev)
    used = torch.empty(n_cols, dtype=torch.int32, device=dev)
    n_used = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.call("lcrw_restrict", _p(cols), cols.numel(), n_cols, _p(remap), _p(used), _p(n_used), _p(ws),
              ws_bytes.value, _stream())
    n = int(n_used.item())
    return remap, used[:n], n


def remap_ids(cols: torch.Tensor, remap: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(cols)
    _lib.call("lcrw_remap_ids", _p(cols), cols.numel(), _p(remap), _p(out), _stream())
    return out


def gather_rows(prep: PreparedEmbeddings, ids: torch.Tensor, side: str):
    """Operand rows E[ids] for the A (vocabulary, with norms) or B (query word) side."""
    n = ids.numel()
    src = prep.EhA if side == "A" else prep.EhB
    T = torch.empty((max(n, 1), prep.kp), dtype=torch.float16, device=ids.device)
    tn = torch.empty(max(n, 1), dtype=torch.float32, device=ids.device) if side == "A" else None
    _lib.call("lcrw_gather_rows", _p(src), _p(prep.norms), prep.kp, _p(ids), n, _p(T), _p(tn), _stream())
    return T, tn


def _range_cols(b_rows: int, a_rows: int) -> int:
    n_mtiles = max(1, (a_rows + 127) // 128)
    want = (n_mtiles * b_rows) // (8 * sm_count())
    return int(min(16384, max(1024, (want + 255) // 256 * 256)))  # a work unit takes two ranges


def spmm_z_shift(n_seg: int) -> int:
    """Panel width (log2) of a Z read by lcrw_spmm: 128-segment panels make each
    nonzero's Z row one contiguous 512-byte run; small segment counts keep 8."""
    return 7 if n_seg > 64 else 3


def segment_plan(seg_offsets: torch.Tensor, n_seg: int, b_rows: int, a_rows: int, range_cols: int | None = None):
    """(endmask, range_seg, n_ranges) of lcrw_segment_plan for segments over b_rows B rows."""
    dev = seg_offsets.device
    rc = range_cols or _range_cols(b_rows, a_rows)
    n_ranges = int(_lib.value("lcrw_plan_ranges", b_rows, rc))
    endmask = torch.empty(int(_lib.value("lcrw_endmask_words", b_rows)), dtype=torch.int32, device=dev)
    range_seg = torch.empty(n_ranges + 1, dtype=torch.int32, device=dev)
    _lib.call("lcrw_segment_plan", _p(seg_offsets), 0, n_seg, b_rows, rc, _p(endmask), _p(range_seg), n_ranges,
              _stream())
    return endmask, range_seg, n_ranges


def phase1(A: torch.Tensor, a_norms: torch.Tensor, a_rows: int, B: torch.Tensor,
           b_rows: int, seg_offsets: torch.Tensor, n_seg: int, prep: PreparedEmbeddings,
           range_cols: int | None = None, z_shift: int = 3) -> tuple[torch.Tensor, int]:
    """Z ((1 << z_shift)-segment panels, z_panel = a_rows << z_shift) of distances.py:147-178,
    without the exact-zero pass."""
    dev = A.device
    st = _stream()
    endmask, range_seg, n_ranges = segment_plan(seg_offsets, n_seg, b_rows, a_rows, range_cols)
    w = 1 << z_shift
    z_panel = w * max(a_rows, 1)
    Z = torch.empty(((n_seg + w - 1) // w) * z_panel, dtype=torch.float32, device=dev)
    if n_seg % w:  # slots past the last segment: defined values (lcrw_spmm reads 4 segments at a time)
        Z[(n_seg // w) * z_panel:].zero_()
    _lib.call("lcrw_phase1", _p(A), _p(a_norms), a_rows, _p(B), b_rows, prep.k_eff, prep.kp,
              _p(seg_offsets), 0, n_seg, _p(endmask), _p(range_seg), n_ranges, _p(prep.scale), _p(Z), z_panel,
              z_shift, st)
    return Z, z_panel


def zero_identical(seg_offsets, n_seg, rep, nxt, remap, Z, z_panel, z_shift: int = 3) -> None:
    _lib.call("lcrw_zero_identical", _p(seg_offsets), n_seg, _p(rep), _p(nxt), _p(remap), _p(Z), z_panel, z_shift,
              _stream())


def refine_near(Z, z_panel, z_shift, a_rows, n_seg, seg_offsets, seg_ids, a_ids, a_norms, prep: "PreparedEmbeddings",
                B32: torch.Tensor | None = None, mode: int = 0, count: torch.Tensor | None = None) -> None:
    """Exact re-evaluation of the near entries of a Phase-1 Z (lcrw_refine_near, scan
    mode): entries with 0 < d < tau |a| become the exact segment minimum from the f32
    rows (A rows E32[a_ids], segment rows B32[seg_ids], B32 = E32 by default).
    mode 1 marks them instead (count += their number), mode 2 finalizes marked entries
    (after lcrw_near_scatter); ``count`` is an int64 device scalar."""
    B = prep.E32 if B32 is None else B32
    _lib.call("lcrw_refine_near", _p(Z), z_panel, z_shift, a_rows, n_seg, _p(seg_offsets), 0, _p(seg_ids),
              _p(prep.E32), _p(a_ids), _p(B), prep.m, _p(a_norms), _p(prep.scale), None, _p(count), 0, mode,
              _stream())


NEAR_CAP = 1 << 24  # near-pair candidates per query set (LCRW_NEAR_CAP overrides; LCRW_NEAR=0: no near pairs)
NEAR_SLICE_BYTES = 4 << 30  # GEMM form: the candidates come from distance tables of query-vocabulary row slices


class NearPairs:
    """Near word pairs of a query set (near.cu, include/lcrwmd.h), lowering the marked near
    entries of both directions to their exact minima (scatter) before refine_near
    finalizes them.  With the query set's distance table they are built on the stream when
    the forward direction marked near entries (device-side gate); in the GEMM form (no
    table: large vocabularies) from tables of row slices, after a host read of the forward
    direction's mark count (built only when it is non-zero).  An optimisation only:
    without it (LCRW_NEAR=0, or a candidate overflow) the marked entries are recomputed in
    full, bitwise the same."""

    def __init__(self, table: torch.Tensor | None, res2: "Restricted", prep: PreparedEmbeddings):
        self.cap = int(os.environ.get("LCRW_NEAR_CAP", NEAR_CAP))
        self.a_rows, self.v_rows = res2.v_e, prep.V
        dev = res2.A.device
        self.gate = torch.zeros(1, dtype=torch.int64, device=dev)  # entries the forward direction marked
        self.table, self.res2, self.prep = table, res2, prep
        self.built = table is not None  # (GEMM form: decided after the forward direction's marks)
        self.ws = None
        if table is not None:  # an empty header until built (a rank with no forward rows never builds)
            self.ws = self._workspace()
            _lib.call("lcrw_near_pairs_reset", self.a_rows, self.v_rows, self.cap, _p(self.ws), _stream())

    def _workspace(self) -> torch.Tensor:
        ws_bytes = C.c_size_t(0)
        _lib.call("lcrw_near_pairs_workspace", self.a_rows, self.v_rows, self.cap, C.byref(ws_bytes))
        return torch.empty(ws_bytes.value, dtype=torch.uint8, device=self.gate.device)

    @staticmethod
    def enabled() -> bool:
        return os.environ.get("LCRW_NEAR", "1") != "0"

    def _build(self) -> None:
        p, r2 = self.prep, self.res2
        if self.table is not None:
            _lib.call("lcrw_near_pairs_build", _p(self.table), self.a_rows, self.v_rows, _p(r2.used),
                      _p(r2.a_norms), _p(p.norms), _p(p.E32), p.m, _p(p.scale), _p(self.gate), self.cap,
                      _p(self.ws), _stream())
            return
        self.built = int(self.gate.item()) > 0
        if not self.built:
            return
        self.ws = self._workspace()
        _lib.call("lcrw_near_pairs_reset", self.a_rows, self.v_rows, self.cap, _p(self.ws), _stream())
        chunk = int(_lib.value("lcrw_table_chunk"))
        rows = max(1, NEAR_SLICE_BYTES // (p.V * TABLE_ROW_BYTES)) * chunk
        dev = r2.A.device
        seg = torch.arange(p.V + 1, dtype=torch.int64, device=dev)
        plan = segment_plan(seg, p.V, p.V, min(rows, self.a_rows))
        no_rows = torch.full((p.V,), -1, dtype=torch.int32, device=dev)  # (exact zeros: not needed)
        for r0 in range(0, self.a_rows, rows):
            n = min(rows, self.a_rows - r0)
            T = torch.empty(int(_lib.value("lcrw_table_bytes", n, p.V)), dtype=torch.uint8, device=dev)
            Ap, anp = _table_operand(r2.used[r0:r0 + n], p)
            _lib.call("lcrw_distance_table", _p(Ap), _p(anp), n, _p(p.EhB), p.V, p.k_eff, p.kp, _p(seg), _p(plan[0]),
                      _p(plan[1]), plan[2], _p(p.scale), _p(p.canon), _p(p.next), _p(no_rows), _p(T), _stream())
            _lib.call("lcrw_near_pairs_candidates", _p(T), r0, n, self.a_rows, p.V, _p(r2.a_norms), _p(p.norms), p.m,
                      None, self.cap, _p(self.ws), _stream())
            del T
        _lib.call("lcrw_near_pairs_finish", self.a_rows, self.v_rows, _p(r2.used), _p(r2.a_norms), _p(p.norms),
                  _p(p.E32), p.m, _p(p.scale), self.cap, _p(self.ws), _stream())

    def forward(self, Z, zp, zs, a_rows: int, a_ids, a_norms, row_map, queries_offsets, query_cols, n_q) -> None:
        """Forward Z1 over this query set (rows: E ids a_ids with scaled squared norms
        a_norms, row_map = E id -> Z1 row or -1; segments: the queries): mark, build the
        pairs (skipped when nothing was marked), scatter, finalize."""
        refine_near(Z, zp, zs, a_rows, n_q, queries_offsets, query_cols, a_ids, a_norms, self.prep,
                    mode=1, count=self.gate)
        self._build()
        if self.built:
            _lib.call("lcrw_near_scatter", _p(self.ws), self.a_rows, self.v_rows, self.cap, 1, _p(Z), zp, zs, n_q,
                      _p(queries_offsets), 0, _p(query_cols), _p(self.res2.remap), _p(row_map), _p(self.gate),
                      _stream())
        refine_near(Z, zp, zs, a_rows, n_q, queries_offsets, query_cols, a_ids, a_norms, self.prep,
                    mode=2, count=self.gate)

    def n_candidates(self) -> int:
        """Candidate pairs of the last build (reads the device header; tests)."""
        return int(self.ws[:8].view(torch.int64).item()) if self.built else 0


def _table_operand(ids: torch.Tensor, prep: PreparedEmbeddings):
    """The distance-table build's A operand: the query-vocabulary rows E[ids] and their norms."""
    return gather_rows(prep, ids, "A")


def spmm(x_offsets, x_cols, x_vals, n_rows, Z, z_panel, n_seg, out, ld_row, ld_panel,
         z_block_rows: int = 0, z_block_stride: int = 0, z_shift: int = 3, dist: bool = False) -> None:
    """lcrw_spmm, or lcrw_spmm_dist (bitwise the same) when Z holds Phase-1 distances."""
    _lib.call("lcrw_spmm_dist" if dist else "lcrw_spmm", _p(x_offsets), _p(x_cols), _p(x_vals), n_rows, _p(Z), z_panel, z_shift, z_block_rows,
              z_block_stride, n_seg, _p(out), ld_row, ld_panel, _stream())


def topk_rows(d: torch.Tensor, ids: torch.Tensor, n_seg: int, seg_len: int, k: int):
    """Per-segment k smallest (distance, id); k <= 1024."""
    kk = min(k, seg_len)
    out_d = torch.empty((n_seg, k), dtype=torch.float32, device=d.device)
    out_i = torch.empty((n_seg, k), dtype=torch.int64, device=d.device)
    _lib.call("lcrw_topk_segments", _p(d), _p(ids), n_seg, seg_len, k, _p(out_d), _p(out_i), _stream())
    return out_d[:, :kk], out_i[:, :kk]


def topk_matrix_rows(D: torch.Tensor, n_rows: int, row_len: int, ld: int, id_base: int, k: int,
                     out_d: torch.Tensor, out_i: torch.Tensor) -> None:
    """Per-row k smallest (distance, id_base + column) of a row-major matrix (lcrw_topk_rows)."""
    ws_bytes = C.c_size_t(0)
    _lib.call("lcrw_topk_rows_workspace", n_rows, row_len, k, C.byref(ws_bytes))
    ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=D.device)
    _lib.call("lcrw_topk_rows", _p(D), ld, n_rows, row_len, id_base, k, _p(out_d), _p(out_i), _p(ws),
              ws_bytes.value, _stream())


def topk_sort(d: torch.Tensor, ids: torch.Tensor, k: int):
    n = d.numel()
    ws_bytes = C.c_size_t(0)
    _lib.call("lcrw_topk_sort_workspace", n, C.byref(ws_bytes))
    ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=d.device)
    kk = min(k, n)
    out_d = torch.empty(max(kk, 1), dtype=torch.float32, device=d.device)
    out_i = torch.empty(max(kk, 1), dtype=torch.int64, device=d.device)
    _lib.call("lcrw_topk_sort", _p(d), _p(ids), n, k, _p(out_d), _p(out_i), _p(ws), ws_bytes.value, _stream())
    return out_d[:kk], out_i[:kk]


# ---------------------------------------------------------------------------
# one direction and the symmetric pipeline
# ---------------------------------------------------------------------------


@dataclass
class Restricted:
    """A resident set restricted to its own words (corpus.py:405-426), on device."""

    csr: DeviceCSR
    remap: torch.Tensor
    used: torch.Tensor
    v_e: int
    cols_r: torch.Tensor
    A: torch.Tensor
    a_norms: torch.Tensor
    host_rank: np.ndarray | None = None  # host copy of remap (host_plan only)

    @classmethod
    def build(cls, x: DeviceCSR, prep: PreparedEmbeddings, host_plan: bool = False) -> "Restricted":
        """Restriction of ``x`` to its own words (ascending word id, as
        corpus.py:417).  With ``host_plan`` the restriction is computed from the
        host copy of x's ids (a small query set) so that the remap is also
        available on the host for planning lcrw_reverse_panels.  Ascending ids
        scatter each query's words over the Z2 tiles, which balances the
        per-(tile, warp) entry lists of that kernel."""
        if host_plan:
            seen = np.zeros(x.n_cols, dtype=bool)  # (a mask, not np.unique's sort: ~0.2 vs ~4 ms at C2,
            seen[x.host_ids()[0]] = True            #  spent while the GPU waits for work)
            order = np.flatnonzero(seen).astype(np.int32)
            rank = np.full(x.n_cols, -1, dtype=np.int32)
            rank[order] = np.arange(len(order), dtype=np.int32)
            used = to_device(order, torch.int32)
            remap = to_device(rank, torch.int32)
            v_e = len(order)
        else:
            rank = None
            remap, used, v_e = restrict(x.cols, x.n_cols)
        A, an = gather_rows(prep, used, "A")
        return cls(x, remap, used, v_e, remap_ids(x.cols, remap), A, an, rank)


def nearest_distances(res: Restricted, prep: PreparedEmbeddings, seg_offsets: torch.Tensor, word_ids: torch.Tensor,
                      n_seg: int, z_shift: int = 3, near: NearPairs | None = None) -> tuple[torch.Tensor, int]:
    """Z over res's vocabulary for segments of E rows ``word_ids`` (with exact zeros);
    ``near``: the segments are the query set of those near pairs (faster refinement)."""
    B, _ = gather_rows(prep, word_ids, "B")
    Z, zp = phase1(res.A, res.a_norms, res.v_e, B, word_ids.numel(), seg_offsets, n_seg, prep, z_shift=z_shift)
    rep, nxt = prep.representatives(word_ids)
    zero_identical(seg_offsets, n_seg, rep, nxt, res.remap, Z, zp, z_shift)
    if near is None:
        refine_near(Z, zp, z_shift, res.v_e, n_seg, seg_offsets, word_ids, res.used, res.a_norms, prep)
    else:
        near.forward(Z, zp, z_shift, res.v_e, res.used, res.a_norms, res.remap, seg_offsets, word_ids, n_seg)
    return Z, zp


def one_direction(res: Restricted, prep: PreparedEmbeddings, queries: DeviceCSR, layout: str = "rows",
                  near: NearPairs | None = None) -> torch.Tensor:
    """distances.py:181-204 for all queries at once: (n_res, n_q) bounds.

    layout "rows" -> row-major (n_res, n_q); "panels" -> out[(q>>3)*8*n_res + i*8 + (q&7)]."""
    n_res, n_q = res.csr.n_rows, queries.n_rows
    zs = spmm_z_shift(n_q)
    Z, zp = nearest_distances(res, prep, queries.offsets, queries.cols, n_q, zs, near)
    if layout == "rows":
        out = torch.empty(n_res * max(n_q, 1), dtype=torch.float32, device=Z.device)
        ld_row, ld_panel = n_q, 8
    else:
        out = torch.empty(((n_q + 7) // 8) * 8 * n_res, dtype=torch.float32, device=Z.device)
        ld_row, ld_panel = 8, 8 * n_res
        if n_q % 8:  # the last panel's padding queries: defined values (lcrw_reverse_panels reads 8 at a time)
            out[(n_q // 8) * 8 * n_res:].zero_()
    spmm(res.csr.offsets, res.cols_r, res.csr.vals, n_res, Z, zp, n_q, out, ld_row, ld_panel, z_shift=zs, dist=True)
    return out


REVERSE_Z2_BYTES = 4 << 30   # Z2 batch budget (docs per batch = budget / (4 * v_e2), multiple of 32)


def query_entries(x: DeviceCSR, rank: np.ndarray, a_rows: int):
    """The reverse pass's plan for x (host ids of a DeviceCSR) built natively on the host
    (lcrw_plan_reverse, identical to plan_query_entries) and copied to the device:
    (e_blk, e_tile)."""
    hc, hv = x.host_ids()
    blk, tile = plan_query_entries_native(x.host_offsets, hc, hv, rank, a_rows, *reverse_panels_geometry())
    return to_device(blk.view(np.int32), torch.int32), to_device(tile, torch.int64)


def plan_query_entries_native(offsets, cols, vals, rank, a_rows: int, T: int, G: int, W: int, I: int):
    """lcrw_plan_reverse (csrc/plan.cu, host code): same output as plan_query_entries."""
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    rank = np.ascontiguousarray(rank, dtype=np.int32)
    n_q = len(offsets) - 1
    cap = int(_lib.value("lcrw_plan_reverse_words_bound", n_q, int(offsets[-1]) if n_q else 0, a_rows, T, G, W, I))
    words = np.empty(max(cap, 1), dtype=np.uint32)
    n_tiles = (a_rows + T - 1) // T
    n_groups = (n_q + G - 1) // G
    tile_off = np.empty(n_groups * n_tiles + 1, dtype=np.int64)
    n_words = C.c_int64(0)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.call("lcrw_plan_reverse", ptr(offsets), n_q, ptr(cols), ptr(vals), ptr(rank), a_rows, T, G, W, I,
              ptr(words), cap, ptr(tile_off), C.byref(n_words))
    return words[: n_words.value], tile_off


def reverse_panels_geometry() -> tuple[int, int, int, int]:
    """(tile rows T, query group G, warps W, group size I) of lcrw_reverse_panels."""
    return tuple(int(_lib.value(f"lcrw_reverse_panels_{n}")) for n in ("tile_rows", "group", "warps", "ilp"))


def plan_query_entries(offsets: np.ndarray, cols: np.ndarray, vals: np.ndarray, rank: np.ndarray, a_rows: int,
                       T: int, G: int, W: int, I: int):
    """Word-major plan of the query CSR for lcrw_reverse_panels (include/lcrwmd.h).

    One block of uint32 words per (query group, T-row tile): W cumulative list
    ends, then the entries (two words: (row - t*T) << 16 | (q - g*G), bits of
    x) of the W per-warp lists (warp = local query % W).  Each list is laid out
    in groups of I entries naming distinct queries, by LEVEL: the j-th entry
    (ascending row) of every query of the list is on level j, and level j's
    entries (ascending query) fill ceil(n_j / I) groups, levels in order.  So
    each query's terms are accumulated in ascending row (= word id) order
    whatever the other queries of the set are -- the fp32 sums, and D, do not
    depend on how the queries are batched (distances.py:198-203); empty slots
    are padding (scratch query G + warp, weight 0).  Returns (blocks uint32, block
    word offsets int64 [n_groups*n_tiles+1]).
    Built on the host from the (small) query set -- index planning, no
    arithmetic."""
    if T > 128 or G > 1024:
        raise ValueError("plan encoding holds rows < 128 and queries <= 1024")
    n_q = len(offsets) - 1
    n_tiles = (a_rows + T - 1) // T
    n_groups = (n_q + G - 1) // G
    n_lists = n_groups * n_tiles * W
    q = np.repeat(np.arange(n_q, dtype=np.int64), np.diff(offsets))
    r = rank[cols].astype(np.int64)
    g, ql = q // G, q % G
    t, rl, w = r // T, r % T, ql % W
    key = (g * n_tiles + t) * W + w
    order = np.lexsort((rl, ql, key))
    key, ql, rl = key[order], ql[order], rl[order]
    xv = np.asarray(vals)[order].astype(np.float32)
    # level of an entry = its position inside its (list, query) run (ascending row)
    new_run = np.ones(key.size, dtype=bool)
    new_run[1:] = (key[1:] != key[:-1]) | (ql[1:] != ql[:-1])
    run_id = np.cumsum(new_run) - 1
    run_start = np.flatnonzero(new_run)
    level = np.arange(key.size, dtype=np.int64) - run_start[run_id]
    L = int(level.max()) + 1 if key.size else 1
    # (list, level) cells, ascending query inside each: position p -> group p // I, slot p % I
    order2 = np.lexsort((ql, level, key))
    key, ql, rl, xv, level = key[order2], ql[order2], rl[order2], xv[order2], level[order2]
    cell = key * L + level
    n_cell = np.bincount(cell, minlength=n_lists * L)
    cell_start = np.zeros(n_lists * L + 1, dtype=np.int64)
    np.cumsum(n_cell, out=cell_start[1:])
    cpos = np.arange(key.size, dtype=np.int64) - cell_start[cell]     # position inside its cell
    g_cell = ((n_cell + I - 1) // I).reshape(n_lists, L)              # groups per (list, level)
    g_off = np.zeros((n_lists, L), dtype=np.int64)                    # first group of each level in its list
    np.cumsum(g_cell[:, :-1], axis=1, out=g_off[:, 1:])
    groups = g_cell.sum(axis=1)
    lens = (groups * I).reshape(n_groups * n_tiles, W)               # padded list lengths (entries)
    ends = np.cumsum(lens, axis=1)                                   # per-block cumulative list ends
    blk_words = W + 2 * ends[:, -1]
    blk_words = (blk_words + 3) // 4 * 4                             # 16-byte aligned blocks
    tile_off = np.zeros(n_groups * n_tiles + 1, dtype=np.int64)
    np.cumsum(blk_words, out=tile_off[1:])
    words = np.zeros(tile_off[-1], dtype=np.uint32)
    hdr = tile_off[:-1, None] + np.arange(W)
    words[hdr.ravel()] = ends.ravel().astype(np.uint32)
    list_start = np.zeros(n_lists, dtype=np.int64)                   # first entry of each list inside its block
    list_start.reshape(-1, W)[:, 1:] = ends[:, :-1]
    ent_base = tile_off[:-1].repeat(W) + W + 2 * list_start          # word offset of each list's first entry
    # every slot starts as padding (weight 0, the list's own scratch query G + warp: no two
    # warps touch the same accumulator row), then the real entries
    flat = lens.ravel()
    pos = np.arange(flat.sum(), dtype=np.int64) - np.repeat(np.cumsum(flat) - flat, flat)
    scratch = ((G + np.arange(n_lists, dtype=np.int64) % W) * 128).astype(np.uint32)
    words[np.repeat(ent_base, flat) + 2 * pos] = np.repeat(scratch, flat)
    slot = ent_base[key] + 2 * ((g_off[key, level] + cpos // I) * I + cpos % I)
    words[slot] = (((rl * 128) << 18) | (ql * 128)).astype(np.uint32)
    words[slot + 1] = xv.view(np.uint32)
    return words, tile_off


REVERSE_TABLE_Z2_FRACTION = 3  # table mode: Z2 batches up to 1/3 of HBM -- each batch re-streams the table
                               # once and larger batches keep one chunk L2-resident for longer (C2 on
                               # B200: 16 GB 502 ms, 32 GB 490 ms, 64 GB 485 ms per step)
TABLE_CHUNK_L2_BYTES = 80 << 20   # a table chunk (v_rows x 512 B) must stay L2-resident
TABLE_ROW_BYTES = 512             # per vocabulary word per 256-word chunk: 256 16-bit keys


def reverse_mode(v_rows: int, a_rows: int, nnz_docs: int, total_memory: int | None = None,
                 split: bool = False) -> str:
    """"table" when the reverse Phase 1 is cheaper as a distance table + per-doc gathers
    (table.cu): the vocabulary is small next to nnz(X1) (each (w, u) distance is then
    needed ~nnz/V times), a 256-word chunk of it fits in L2, and the table fits in HBM;
    else "gemm".  LCRW_REVERSE=gemm|table overrides (tests, A/B runs)."""
    env = os.environ.get("LCRW_REVERSE", "")
    if env in ("gemm", "table"):
        return env
    if split or v_rows * TABLE_ROW_BYTES > TABLE_CHUNK_L2_BYTES or 2 * v_rows > nnz_docs:
        return "gemm"  # (split operands, m <= 64: the GEMM form keeps Z2 in f32 instead of 16-bit keys)
    table_bytes = int(_lib.value("lcrw_table_bytes", a_rows, v_rows))
    if total_memory is None:  # (mem_get_info would stall the stream)
        total_memory = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
    return "table" if table_bytes < total_memory // 4 else "gemm"


def distance_table(res2: "Restricted", prep: PreparedEmbeddings, via_transpose: bool = False) -> torch.Tensor:
    """The reverse Phase-1 distance table (include/lcrwmd.h, table.cu) of the query
    vocabulary res2 against every E row: lcrw_phase1 with singleton segments (the GEMM
    form's operands and roles, so each entry is the value it would compute) storing
    128-row panels directly, plus the exact zeros (lcrw_distance_table).
    ``via_transpose``: the two-pass build (segment panels + lcrw_zero_identical +
    lcrw_table_transpose), kept as a cross-check."""
    V = prep.V
    dev = res2.A.device
    seg = torch.arange(V + 1, dtype=torch.int64, device=dev)
    T = torch.empty(max(16, int(_lib.value("lcrw_table_bytes", res2.v_e, V))), dtype=torch.uint8, device=dev)
    if via_transpose:
        zs = 7  # lcrw_table_transpose reads 128-segment panels
        Tp, zp = phase1(res2.A, res2.a_norms, res2.v_e, prep.EhB, V, seg, V, prep, z_shift=zs)
        zero_identical(seg, V, prep.canon, prep.next, res2.remap, Tp, zp, zs)
        _lib.call("lcrw_table_transpose", _p(Tp), _p(res2.a_norms), res2.v_e, V, _p(prep.scale), _p(T), _stream())
        return T
    endmask, range_seg, n_ranges = segment_plan(seg, V, V, res2.v_e)
    Ap, anp = _table_operand(res2.used, prep)
    _lib.call("lcrw_distance_table", _p(Ap), _p(anp), res2.v_e, _p(prep.EhB), V, prep.k_eff, prep.kp,
              _p(seg), _p(endmask), _p(range_seg), n_ranges, _p(prep.scale), _p(prep.canon), _p(prep.next),
              _p(res2.remap), _p(T), _stream())
    return T


def reverse_batch_docs(n_docs: int, v_e2: int, budget_bytes: int = REVERSE_Z2_BYTES) -> int:
    nb = max(32, budget_bytes // (4 * max(v_e2, 1)))
    nb = min(nb, max(32, n_docs))
    return int((nb + 31) // 32 * 32)


FUSED_TOPK_MAX = 32  # k up to which the max -> top-k is fused into lcrw_reverse_panels (no D)
QUERY_SLICE = 16384  # queries per pass of the symmetric pipeline (bounds D, D1, plan and table per pass)


def symmetric(x1: DeviceCSR, x2: DeviceCSR, prep: PreparedEmbeddings, k: int | None,
              z2_budget_bytes: int = REVERSE_Z2_BYTES, d1: torch.Tensor | None = None, id_offset: int = 0,
              query_slice: int = QUERY_SLICE, prepared: "QuerySide | None" = None):
    """lcrwmd_full (k=None -> (n1, n2) matrix) or its per-query top-k ((n2, min(k, n1))
    dists, ids).  Query sets of any size: queries are processed in slices of
    ``query_slice`` (a multiple of 8), each slice a full pass (restriction, table, both
    directions) -- query batching never changes a result (distances.py:198-203).

    ``d1`` (8-query panels) may be supplied by a caller that computed the
    forward direction itself (parallel.py), with the query side it prepared for it
    (``prepared``, a single-pass query set only); ``id_offset`` shifts returned doc ids."""
    n1, n2 = x1.n_rows, x2.n_rows
    dev = x1.cols.device
    if n1 == 0 or n2 == 0:
        if k is None:
            return torch.empty((n1, n2), dtype=torch.float32, device=dev)
        return (torch.empty((n2, 0), dtype=torch.float32, device=dev),
                torch.empty((n2, 0), dtype=torch.int64, device=dev))
    qs = max(8, query_slice // 8 * 8)
    if n2 <= qs:
        return _symmetric_pass(x1, x2, prep, k, z2_budget_bytes, d1, id_offset, prepared)
    if k is None:
        D = torch.empty((n1, n2), dtype=torch.float32, device=dev)
    else:
        kk = min(k, n1)
        out_d = torch.empty((n2, kk), dtype=torch.float32, device=dev)
        out_i = torch.empty((n2, kk), dtype=torch.int64, device=dev)
    for q0 in range(0, n2, qs):
        q1 = min(n2, q0 + qs)
        d1s = None if d1 is None else d1[(q0 // 8) * 8 * n1:((q1 + 7) // 8) * 8 * n1]
        r = _symmetric_pass(x1, x2.slice_rows(q0, q1), prep, k, z2_budget_bytes, d1s, id_offset)
        if k is None:
            D[:, q0:q1] = r
        else:
            out_d[q0:q1], out_i[q0:q1] = r
        del r
    return D if k is None else (out_d, out_i)


@dataclass
class QuerySide:
    """A query set's device-side preparation for one pass: its restriction, the reverse
    distance table (None: GEMM form) and the near word pairs (None: disabled)."""

    res2: "Restricted"
    table: torch.Tensor | None
    near: NearPairs | None

    @classmethod
    def build(cls, x2: DeviceCSR, prep: PreparedEmbeddings, nnz_docs: int) -> "QuerySide":
        res2 = Restricted.build(x2, prep, host_plan=True)
        mode = reverse_mode(prep.V, res2.v_e, nnz_docs, split=prep.split)
        table = distance_table(res2, prep) if mode == "table" else None
        return cls(res2, table, NearPairs(table, res2, prep) if NearPairs.enabled() else None)


def _symmetric_pass(x1: DeviceCSR, x2: DeviceCSR, prep: PreparedEmbeddings, k: int | None,
                    z2_budget_bytes: int = REVERSE_Z2_BYTES, d1: torch.Tensor | None = None, id_offset: int = 0,
                    prepared: QuerySide | None = None):
    """One pass of ``symmetric`` over all of x2's queries."""
    n1, n2 = x1.n_rows, x2.n_rows
    dev = x1.cols.device
    st = _stream()
    d1_ready = None  # (a side-stream forward pass measured slower: persistent kernels contend for SMs)
    # the query side's device work first (restriction, distance table: only X2 and E), so an
    # X1 still being copied in on another stream (DeviceCSR.upload(..., stream=)) overlaps it;
    # then the forward pass; the host-side plan of the reverse pass is built while the
    # forward kernels run
    # near word pairs (near.cu): built only when the forward direction marks near entries;
    # they replace the per-entry exact recomputation (a caller that supplies D1 passes the
    # query side its forward direction used, or goes without them)
    if prepared is None:
        prepared = QuerySide.build(x2, prep, x1.nnz)
        if d1 is not None:
            prepared.near = None
    res2, table, near = prepared.res2, prepared.table, prepared.near
    x1.wait()
    if d1 is None:
        res1 = Restricted.build(x1, prep)
        d1 = one_direction(res1, prep, x2, layout="panels", near=near)  # D1[(q>>3)*8*n1 + j*8 + (q&7)]
        del res1
    e_blk, e_tile = query_entries(x2, res2.host_rank, res2.v_e)
    if table is not None and z2_budget_bytes == REVERSE_Z2_BYTES:
        total = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
        live = torch.cuda.memory_allocated()  # host-side counter (mem_get_info would stall the stream)
        z2_budget_bytes = max(REVERSE_Z2_BYTES, min(total // REVERSE_TABLE_Z2_FRACTION, (total - live) // 2))
    batch = reverse_batch_docs(n1, res2.v_e, z2_budget_bytes)
    ho = x1.host_offsets
    max_words = 0 if table is not None else max(int(ho[min(n1, j0 + batch)] - ho[j0]) for j0 in range(0, n1, batch))
    ws_bytes = C.c_size_t(0)
    _lib.call("lcrw_reverse_workspace", res2.v_e, prep.kp, batch, max_words, C.byref(ws_bytes))
    ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device=dev)
    fused = k is not None and k <= FUSED_TOPK_MAX and not os.environ.get("LCRW_TOPK_VIA_D")
    top_d = top_i = None
    if k is None:
        D = torch.empty(n1 * n2, dtype=torch.float32, device=dev)  # reference orientation (n1, n2)
        ld_q, ld_doc = 1, n2
    elif fused:
        # max -> top-k fused into lcrw_reverse_panels: per-(query, CTA) lists, D never exists
        slots = int(_lib.value("lcrw_reverse_panels_top_slots"))
        top_d = torch.full((n2, slots, k), float("inf"), dtype=torch.float32, device=dev)
        top_i = torch.full((n2, slots, k), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        D, ld_q, ld_doc = None, 0, 0
    else:
        D = torch.empty(n2 * n1, dtype=torch.float32, device=dev)  # query-major for the per-query top-k
        ld_q, ld_doc = n1, 1
    rep, nxt = prep.representatives(x1.cols) if table is None else (None, None)
    host_offs = np.ascontiguousarray(ho, dtype=np.int64)
    _lib.call("lcrw_reverse_pipeline", _p(res2.A), _p(res2.a_norms), res2.v_e, _p(prep.EhB), prep.V, prep.k_eff,
              prep.kp,
              _p(prep.scale), _p(x1.offsets), host_offs.ctypes.data_as(C.c_void_p), n1, _p(x1.cols), _p(rep),
              _p(nxt), _p(res2.remap), _p(e_blk), _p(e_tile), n2, _p(d1), 8 * n1, _p(D), ld_q, ld_doc,
              _p(top_d), _p(top_i), k if fused else 0, id_offset, batch, 0, _p(table),
              _p(near.ws) if near is not None and near.built else None, near.cap if near is not None else 0,
              0 if prep.split else 1, _p(prep.E32), prep.m,
              _p(res2.used),
              C.c_void_p(d1_ready.cuda_event) if d1_ready is not None else None, _p(ws), ws_bytes.value, st)
    del ws, table, near
    if k is None:
        return D.view(n1, n2)
    kk = min(k, n1)
    if fused:
        d, i = topk_rows(top_d.view(n2, -1), top_i.view(n2, -1), n2, top_d.shape[1] * k, k)
        return d[:, :kk].contiguous(), i[:, :kk].contiguous()
    if k > 1024:  # beyond the selection kernels: one (distance, id) sort per query row
        out_d = torch.empty((n2, kk), dtype=torch.float32, device=dev)
        out_i = torch.empty((n2, kk), dtype=torch.int64, device=dev)
        ids = torch.arange(id_offset, id_offset + n1, dtype=torch.int64, device=dev)
        for q in range(n2):
            od, oi = topk_sort(D[q * n1:(q + 1) * n1], ids, kk)
            out_d[q], out_i[q] = od, oi
        return out_d, out_i
    out_d = torch.empty((n2, k), dtype=torch.float32, device=dev)
    out_i = torch.empty((n2, k), dtype=torch.int64, device=dev)
    topk_matrix_rows(D, n2, n1, n1, id_offset, k, out_d, out_i)
    return out_d[:, :kk], out_i[:, :kk]


def nearest_word_distances(E, Q) -> torch.Tensor:
    """distances.py:133-144 on device: z over every row of E for one free query."""
    dev = require_cuda()
    Qd = to_device(np.atleast_2d(np.asarray(Q, dtype=np.float32)) if not isinstance(Q, torch.Tensor) else Q,
                   torch.float32)
    prep = PreparedEmbeddings(E, extra=(Qd,))
    if Qd.shape[1] != prep.m:
        raise ValueError(f"dimension mismatch: {prep.m} vs {Qd.shape[1]}")
    nq = int(Qd.shape[0])
    Qh = prep.prepare_free_rows(Qd)
    seg = torch.tensor([0, nq], dtype=torch.int64, device=dev)
    Z, zp = phase1(prep.EhA, prep.norms, prep.V, Qh, nq, seg, 1, prep)
    rep = torch.empty(nq, dtype=torch.int32, device=dev)
    _lib.call("lcrw_match_rows", _p(Qd), nq, _p(prep.E32), prep.m, _p(prep.sorted_hash), _p(prep.sorted_ids),
              prep.V, _p(prep.canon), _p(rep), _stream())
    zero_identical(seg, 1, rep, prep.next, None, Z, zp)
    refine_near(Z, zp, 3, prep.V, 1, seg, torch.arange(nq, dtype=torch.int32, device=dev),
                torch.arange(prep.V, dtype=torch.int32, device=dev), prep.norms, prep, B32=Qd.contiguous())
    return Z[: zp].view(prep.V, 8)[:, 0]


# ---------------------------------------------------------------------------
# rows next to the hot path: pairwise distances, centroids, WCD, both bounds
# ---------------------------------------------------------------------------


def pairwise(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """kernels.py:113-130 on the tensor cores: (na, nb) Euclidean distances between rows.

    The Phase-1 kernel with every b row its own segment: A = a's operand rows,
    B = b's, one shared power-of-two scale and exact-identity classes over
    a U b, so identical rows give exactly 0 as in the reference (kernels.py:91-92)."""
    na, nb = int(a.shape[0]), int(b.shape[0])
    dev = a.device
    out = torch.zeros((na, nb), dtype=torch.float32, device=dev)
    if na == 0 or nb == 0:
        return out
    prep = PreparedEmbeddings(torch.cat([a, b], dim=0))
    ids = torch.arange(na, na + nb, dtype=torch.int32, device=dev)
    seg = torch.arange(nb + 1, dtype=torch.int64, device=dev)
    Z, zp = phase1(prep.EhA[:na], prep.norms[:na], na, prep.EhB[na:na + nb], nb, seg, nb, prep, z_shift=3)
    remap = torch.full((na + nb,), -1, dtype=torch.int32, device=dev)
    remap[:na] = torch.arange(na, dtype=torch.int32, device=dev)
    rep, nxt = prep.representatives(ids)
    zero_identical(seg, nb, rep, nxt, remap, Z, zp, 3)
    refine_near(Z, zp, 3, na, nb, seg, ids, torch.arange(na, dtype=torch.int32, device=dev), prep.norms[:na], prep)
    panels = (nb + 7) // 8
    return Z[: panels * zp].view(panels, na, 8).permute(1, 0, 2).reshape(na, panels * 8)[:, :nb].contiguous()


def centroids(x: DeviceCSR, E: torch.Tensor) -> torch.Tensor:
    """kernels.py:201-203: X . E with fp64 products and sums in ascending nonzero order,
    rounded once (lcrw_spmm; bitwise equal to the reference)."""
    V, m = int(E.shape[0]), int(E.shape[1])
    zs = spmm_z_shift(m)
    w = 1 << zs
    mp = (m + w - 1) // w * w
    Ep = torch.zeros((V, mp), dtype=torch.float32, device=E.device)
    Ep[:, :m] = E
    Zp = Ep.view(V, mp // w, w).permute(1, 0, 2).contiguous()  # (1 << zs)-dimension panels
    out = torch.empty((max(x.n_rows, 1), m), dtype=torch.float32, device=E.device)
    spmm(x.offsets, x.cols, x.vals, x.n_rows, Zp, w * V, m, out, m, 8, z_shift=zs)
    return out[: x.n_rows]


def one_sided_rows(x1: DeviceCSR, x2: DeviceCSR, prep: PreparedEmbeddings) -> torch.Tensor:
    """bound1 of distances.py:78-114 (= lcrwmd_batched): (n1, n2) row-major."""
    res = Restricted.build(x1, prep)
    out = one_direction(res, prep, x2, layout="rows")
    return out[: x1.n_rows * x2.n_rows].view(x1.n_rows, x2.n_rows)


def reverse_rows(x1: DeviceCSR, x2: DeviceCSR, prep: PreparedEmbeddings) -> torch.Tensor:
    """bound2 of distances.py:78-114: the reverse direction alone, (n1, n2), through the
    symmetric pipeline with D1 = -inf (its max-combine then passes D2 through)."""
    n1, n2 = x1.n_rows, x2.n_rows
    d1 = torch.full((((n2 + 7) // 8) * 8 * max(n1, 1),), float("-inf"), dtype=torch.float32, device=x1.cols.device)
    return symmetric(x1, x2, prep, None, d1=d1)


def forward_rows_into(res: "Restricted", prep: PreparedEmbeddings, q: DeviceCSR, D: torch.Tensor,
                      batch: int = 4096) -> None:
    """D[i, c] = forward bound of resident row i (res) to query c of q (distances.py:181-204),
    written in place into the row-major (n_res, n_q) matrix D, queries in batches."""
    n = res.csr.n_rows
    ho = q.host_offsets
    ld = int(D.stride(0))
    for q0 in range(0, q.n_rows, batch):
        q1 = min(q.n_rows, q0 + batch)
        nq = q1 - q0
        lo, hi = int(ho[q0]), int(ho[q1])
        seg = q.offsets[q0:q1 + 1] - lo
        zs = spmm_z_shift(nq)
        Z, zp = nearest_distances(res, prep, seg, q.cols[lo:hi], nq, zs)
        out = D.view(-1)[q0:]  # D[i, q0 + c] = out[i * ld + c]
        spmm(res.csr.offsets, res.cols_r, res.csr.vals, n, Z, zp, nq, out, ld, 8, z_shift=zs, dist=True)
        del Z


def max_transposed(D: torch.Tensor, R: torch.Tensor) -> None:
    """D = max(D, R^T) in place (lcrw_max_transposed); D (rows, cols), R (cols, rows)."""
    rows, cols = int(D.shape[0]), int(D.shape[1])
    _lib.call("lcrw_max_transposed", _p(D), int(D.stride(0)), _p(R), int(R.stride(0)), rows, cols, _stream())


def max_transposed_into(out: torch.Tensor, A: torch.Tensor, R: torch.Tensor) -> None:
    """out = max(A, R^T) (lcrw_max_transposed_into); out, A (rows, cols), R (cols, rows),
    each row-major with its own row stride."""
    rows, cols = int(A.shape[0]), int(A.shape[1])
    assert tuple(out.shape) == (rows, cols) and tuple(R.shape) == (cols, rows)
    _lib.call("lcrw_max_transposed_into", _p(out), int(out.stride(0)), _p(A), int(A.stride(0)), _p(R),
              int(R.stride(0)), rows, cols, _stream())


def all_pairs(x: DeviceCSR, prep: PreparedEmbeddings, batch: int = 4096) -> torch.Tensor:
    """Symmetric LC-RWMD of a set against itself, (n, n) on the device (BASELINE configs[4]).

    With X1 == X2 the reverse bound of (j, q) is the forward bound of (q, j)
    (distances.py:262-264), so only the forward direction is computed: for each
    batch of ``batch`` query docs, Phase 1 over x's own vocabulary and the fp64
    SpMM write D1[:, batch] in place, then D = max(D1, D1^T) (lcrw_symmetrize_max).
    The result is exactly symmetric with a zero diagonal; ~1/3 of the FLOPs of
    running the reverse direction per batch."""
    n = x.n_rows
    dev = x.cols.device
    D = torch.empty((max(n, 1), max(n, 1)), dtype=torch.float32, device=dev)
    if n == 0:
        return D[:0, :0]
    forward_rows_into(Restricted.build(x, prep), prep, x, D, batch)
    _lib.call("lcrw_symmetrize_max", _p(D), n, n, _stream())
    return D


def load_index(path) -> tuple[DeviceCSR, torch.Tensor, list[str]]:
    """LCRW v1 index (corpus.py:17-25, 460-489) straight into HBM: the file is read once
    into a pinned host buffer and each section is copied asynchronously from it
    (no intermediate numpy arrays for the big sections).  Returns (DeviceCSR of the
    stored set, f32 embeddings (v_e, m) on the device, words)."""
    from pathlib import Path as _Path
    from .corpus import _index_words, index_layout
    dev = require_cuda()
    nbytes = _Path(path).stat().st_size
    buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    with open(path, "rb") as fh:
        got = fh.readinto(memoryview(buf.numpy()))
    if got != nbytes:
        raise CorpusError(f"{path}: short read")
    host = buf.numpy()
    v_e, n, m, sec = index_layout(host, path)

    def section(name, dtype):
        off, nb = sec[name]
        return buf[off:off + nb].view(dtype)

    offs_h = section("offsets", torch.int64).numpy().copy()
    if n and np.any(np.diff(offs_h) <= 0):
        raise CorpusError(f"{path}: every row must hold at least one word")
    cols = section("ids", torch.int32).to(dev, non_blocking=True)
    vals = section("values", torch.float32).to(dev, non_blocking=True)
    E = section("embeddings", torch.float32).view(v_e, m).to(dev, non_blocking=True)
    offs = torch.from_numpy(offs_h).to(dev)
    words = _index_words(host, sec["words"][0], v_e, path)
    torch.cuda.current_stream().synchronize()  # the pinned buffer is released on return
    # host ids / weights are read back from the device only if a caller plans with them
    return DeviceCSR(offs, cols, vals, v_e, offs_h), E, words


def restrict_vocabulary_host(x: HistogramSet, embeddings):
    """corpus.restrict_vocabulary on the GPU; returns host (set, E rows, remap)."""
    dx = DeviceCSR.upload(x, "hist_set")
    remap, used, n = restrict(dx.cols, dx.n_cols)
    cols_r = remap_ids(dx.cols, remap)
    used_h = used.cpu().numpy()
    out = HistogramSet(np.asarray(x.row_offsets, dtype=np.int64).copy(), cols_r.cpu().numpy(),
                       np.asarray(x.values, dtype=np.float32).copy(), n)
    return out, np.ascontiguousarray(np.asarray(embeddings)[used_h]), remap.cpu().numpy()
