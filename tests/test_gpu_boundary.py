"""GPU: the rest of the drop-in surface and the size cliffs removed in round 2.

* movers.kernels primitives (squared_norms, euclidean_into, row_min, col_min,
  segmented_min) and top-k on the caller's dtype: bitwise against the reference's
  own outputs (tests/golden/prims.npz, made by tests/golden/make_golden.py prims);
* query sets of any size (sliced passes == one pass, bitwise; a 5M-nonzero query
  set), any k, empty sides, large transport problems (test_gpu_parity.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, rel_close
from oracle import lcrwmd_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1711_07227_b200 import _lib
    _lib.load()


@pytest.fixture(scope="module")
def prims():
    return np.load(GOLDEN / "prims.npz")


def test_squared_norms_and_euclidean_into_bitwise(prims):
    from paper_1711_07227_b200 import kernels as K
    z = prims
    assert np.array_equal(K.squared_norms(z["sn_a32"]), z["sn_r32"])
    assert np.array_equal(K.squared_norms(z["sn_a64"]), z["sn_r64"])
    for i in range(4):
        a, b = z[f"eu{i}_a"], z[f"eu{i}_b"]
        sa, sb = K.squared_norms(a), K.squared_norms(b)
        o32 = np.full(z[f"eu{i}_o32"].shape, -1, np.float32)
        assert K.euclidean_into(a, sa, b, sb, o32, 7, 5) is o32
        assert np.array_equal(o32, z[f"eu{i}_o32"]), i
        o64 = np.empty(z[f"eu{i}_o64"].shape, np.float64)
        K.euclidean_into(a, sa, b, sb, o64)
        assert np.array_equal(o64, z[f"eu{i}_o64"]), i
        assert np.all(o32[: min(3, b.shape[0]), : min(3, b.shape[0])].diagonal() == 0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        K.euclidean_into(np.zeros((2, 3)), np.zeros(2), np.zeros((2, 4)), np.zeros(2), np.zeros((2, 2), np.float32))


def test_minima_bitwise(prims):
    from paper_1711_07227_b200 import kernels as K
    z = prims
    for nm in ("f", "i", "d"):
        v = z[f"mn_{nm}"]
        r, c = K.row_min(v), K.col_min(K.DistanceBlock(v))
        assert r.dtype == v.dtype and c.dtype == v.dtype
        np.testing.assert_array_equal(r, z[f"rmin_{nm}"])
        np.testing.assert_array_equal(c, z[f"cmin_{nm}"])
    np.testing.assert_array_equal(K.segmented_min(z["mn_f"], z["seg0"], axis=0), z["smin_f0"])
    np.testing.assert_array_equal(K.segmented_min(z["mn_f"], z["seg1"], axis=1), z["smin_f1"])
    np.testing.assert_array_equal(K.segmented_min(z["mn_d"], np.array([0, 10, 11, 40]), axis=-1), z["smin_d1"])
    np.testing.assert_array_equal(K.segmented_min(z["smin_v"], z["smin_v_seg"]), z["smin_v_out"])
    with pytest.raises(ValueError, match="row_min of an empty block"):
        K.row_min(np.zeros((0, 3), np.float32))
    with pytest.raises(ValueError, match="col_min of an empty block"):
        K.col_min(np.zeros((0, 3), np.float32))
    with pytest.raises(ValueError, match="empty segment"):
        K.segmented_min(np.ones(4), [0, 2, 2, 4])
    with pytest.raises(ValueError, match="need at least one segment"):
        K.segmented_min(np.ones(4), [0])
    with pytest.raises(ValueError, match="do not cover"):
        K.segmented_min(np.ones(4), [0, 3])


def test_topk_keeps_dtype_bitwise(prims):
    """topk_select / topk_merge on f64 (near-ties 1e-12 apart), integers and f16 equal the
    reference's np.lexsort on the caller's dtype; f32 is not involved."""
    from paper_1711_07227_b200 import kernels as K
    z = prims
    for k in (1, 10, 700, 5000):
        for nm in ("d64", "dint", "d16"):
            r = K.topk_select(z[f"tk_{nm}"], z["tk_ids"], k)
            assert r.distances.dtype == z[f"tk_{nm}"].dtype
            assert np.array_equal(r.distances, z[f"tk_{nm}_{k}_d"]), (nm, k)
            assert np.array_equal(r.ids, z[f"tk_{nm}_{k}_i"]), (nm, k)
    r = K.topk_select(np.array([1.0, 1.0 + 1e-12]), np.array([7, 3]), 1)
    assert r.ids.tolist() == [7] and r.distances.tolist() == [1.0]
    parts = [K.topk_select(z["tk_d64"][a:a + 700], z["tk_ids"][a:a + 700], 50) for a in range(0, 3000, 700)]
    m = K.topk_merge(parts, 50)
    assert np.array_equal(m.distances, z["tk_merge_d"]) and np.array_equal(m.ids, z["tk_merge_i"])


def test_topk_nan_and_signed_zero_f32_and_f64():
    """numpy's order: NaN after +inf (NaNs tie -> by id), -0 == +0 (-> by id)."""
    from paper_1711_07227_b200 import kernels as K
    d = np.array([np.nan, 1.0, -0.0, 0.0, np.inf, np.nan, -np.inf, 2.0])
    ids = np.array([5, 9, 4, 2, 8, 1, 7, 3], dtype=np.int64)
    for dt in (np.float64, np.float32):
        r = K.topk_select(d.astype(dt), ids, 8)
        want = O.topk_select(d.astype(dt), ids, 8)
        assert r.ids.tolist() == want[1].tolist(), dt
        assert np.array_equal(r.distances, want[0], equal_nan=True), dt


@pytest.mark.parametrize("reverse", ["table", "gemm"])
def test_query_slices_equal_one_pass(monkeypatch, reverse):
    """Query sets are processed in slices of QUERY_SLICE queries; slicing never changes a
    value (distances.py:198-203): sliced == unsliced, bitwise, for D and for top-k."""
    import torch
    from paper_1711_07227_b200 import device, synthetic as S
    monkeypatch.setenv("LCRW_REVERSE", reverse)
    V = 3000
    E = S.embeddings(V, 64, seed=3)
    x1 = S.histograms(700, V, 30, seed=4)
    x2 = S.histograms(61, V, 30, seed=5)
    prep = device.PreparedEmbeddings(E)
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
    full = device.symmetric(d1, d2, prep, None)
    td, ti = device.symmetric(d1, d2, prep, 7)
    sl = device.symmetric(d1, d2, prep, None, query_slice=16)
    sd, si = device.symmetric(d1, d2, prep, 7, query_slice=16)
    assert torch.equal(full, sl)
    assert torch.equal(td, sd) and torch.equal(ti, si)


def test_query_set_with_5m_nonzeros():
    """A query set above the round-1 limit (4.19M nonzeros): 100k queries x 50 words
    against 2k docs, through lcrwmd_full; sampled entries vs the oracle (subset invariance)."""
    from paper_1711_07227_b200 import distances as D, synthetic as S
    V = 20_000
    E = S.embeddings(V, 64, seed=6)
    x1 = S.histograms(2000, V, 50, seed=7)
    x2 = S.histograms(100_000, V, 50, seed=8)
    assert x2.nnz > 4_500_000
    full = D.lcrwmd_full(x1, x2, E).values
    assert full.shape == (2000, 100_000)
    rng = np.random.default_rng(9)
    di = np.sort(rng.choice(2000, 40, replace=False))
    qj = np.sort(rng.choice(100_000, 40, replace=False))
    ref = O.lcrwmd_full(x1.take_rows(di), x2.take_rows(qj), E)
    got = full[np.ix_(di, qj)]
    atol = 1e-5 * float(np.sqrt((E.astype(np.float64) ** 2).sum(1).max()))
    ok, err = rel_close(got, ref, 1e-4, atol)
    assert ok, err
    top = D.lcrwmd_topk(x1, x2.take_rows(qj), E, 5)
    for j, t in enumerate(top):
        want = O.topk_select(full[:, qj[j]], np.arange(2000), 5)
        assert np.array_equal(t.ids, want[1]) and np.array_equal(t.distances, want[0])


def test_k_above_1024_and_empty_sides():
    import torch
    from paper_1711_07227_b200 import device, distances as D, synthetic as S
    V = 2000
    E = S.embeddings(V, 48, seed=10)
    x1 = S.histograms(3000, V, 20, seed=11)
    x2 = S.histograms(5, V, 20, seed=12)
    full = D.lcrwmd_full(x1, x2, E).values
    res = D.lcrwmd_topk(x1, x2, E, 1500)
    for j, t in enumerate(res):
        want_d, want_i = O.topk_select(full[:, j], np.arange(3000), 1500)
        assert np.array_equal(t.ids, want_i) and np.array_equal(t.distances, want_d), j
    prep = device.PreparedEmbeddings(E)
    empty = device.DeviceCSR.upload(x1.slice_rows(0, 0))
    dq = device.DeviceCSR.upload(x2)
    assert tuple(device.symmetric(empty, dq, prep, None).shape) == (0, 5)
    d, i = device.symmetric(empty, dq, prep, 3)
    assert tuple(d.shape) == (5, 0) and tuple(i.shape) == (5, 0)
    assert tuple(device.symmetric(dq, empty, prep, None).shape) == (5, 0)
    assert D.lcrwmd_batched(x1.slice_rows(0, 0), x2, E).shape == (0, 5)
    del torch


def test_engine_wmd_keeps_f64():
    """The engine merges exact WMD distances with topk_merge: f64 values survive bitwise
    (round 1 cast them to f32)."""
    from paper_1711_07227_b200 import emd, engine
    from paper_1711_07227_b200.corpus import HistogramSet
    rng = np.random.default_rng(13)
    V, m = 300, 16
    E = rng.standard_normal((V, m)).astype(np.float32)
    rows = []
    for _ in range(40):
        h = int(rng.integers(2, 9))
        ids = np.sort(rng.choice(V, h, replace=False)).astype(np.int32)
        c = rng.integers(1, 5, h).astype(np.int64)
        tot = int(c.sum())
        sc = 1 << int(np.ceil(np.log2(tot)))
        c[0] += sc - tot
        rows.append((ids, (c / sc).astype(np.float32)))
    x = HistogramSet.from_rows(rows, V)
    q = x.take_rows(np.arange(3))
    idx = engine.Index(x, E, [f"w{i}" for i in range(V)])
    for method in ("wmd", "wmd-pruned"):
        res = engine.run_query(idx, q, engine.QueryPlan(method=method, k=4, partitions=3))
        for j, r in enumerate(res):
            want, _ = emd.prefiltered_topk_wmd(x, q.row(j), E, 4)
            assert r.distances.dtype == np.float64
            assert np.array_equal(r.ids, want.ids) and np.array_equal(r.distances, want.distances), (method, j)


@pytest.mark.parametrize("k", [1, 10, 32, 33])
@pytest.mark.parametrize("reverse", ["table", "gemm"])
def test_fused_topk_equals_topk_of_materialised_d(monkeypatch, k, reverse):
    """The max -> top-k fused into lcrw_reverse_panels (per-(query, CTA) lists, k <= 32,
    no D) returns exactly the (distance, id) top-k of the materialised query-major D
    (LCRW_TOPK_VIA_D), ties included: duplicated docs give equal distances that must be
    ordered by id (kernels.py:218-223).  k = 33 takes the D path both times."""
    import torch
    from paper_1711_07227_b200 import device, synthetic as S
    monkeypatch.setenv("LCRW_REVERSE", reverse)
    V = 4000
    E = S.embeddings(V, 300, seed=11)
    base = S.histograms(1500, V, 40, seed=12)
    x1 = base.take_rows(np.concatenate([np.arange(1500), np.arange(0, 1500, 7), np.arange(3, 1500, 11)]))
    x2 = S.histograms(40, V, 40, seed=13)
    prep = device.PreparedEmbeddings(E)
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
    fd, fi = device.symmetric(d1, d2, prep, k, id_offset=5)
    monkeypatch.setenv("LCRW_TOPK_VIA_D", "1")
    rd, ri = device.symmetric(d1, d2, prep, k, id_offset=5)
    assert torch.equal(fd, rd) and torch.equal(fi, ri)
    full = device.symmetric(d1, d2, prep, None).cpu().numpy()  # (n1, n2)
    for j in range(x2.n_rows):
        order = np.lexsort((np.arange(x1.n_rows), full[:, j]))[:k]
        assert np.array_equal(fi[j].cpu().numpy(), order + 5)
        assert np.array_equal(fd[j].cpu().numpy(), full[order, j])


@pytest.mark.parametrize("zs,nq", [(3, 37), (7, 200)])
def test_spmm_dist_bitwise_equals_spmm(zs, nq):
    """lcrw_spmm_dist (f32 -> f64 widening by exponent shift, weight pre-scaled by 2^896,
    8-row batches of loads + a serial tail) equals lcrw_spmm bit for bit on distance
    matrices: zeros, tiny and large normal values, weights that take the fallback
    (|x| >= 2^126), empty rows and rows of 1..99 nonzeros (1-4 staged blocks), lanes
    past the last query (8- and 128-query panels)."""
    import torch
    from paper_1711_07227_b200 import device
    rng = np.random.default_rng(21 + zs)
    V, n = 700, 300
    rows = []
    for i in range(n):
        ids = np.sort(rng.choice(V, int(rng.integers(0, 100)) if i % 7 else 32 * (i % 4) + i % 9,
                                 replace=False)).astype(np.int32)
        x = (rng.random(len(ids)) + 0.05).astype(np.float32)
        if i % 50 == 0 and len(x):
            x[0] = np.float32(2.0 ** 126 * 1.5)  # fallback path
        rows.append((ids, x))
    offs = np.zeros(n + 1, np.int64)
    offs[1:] = np.cumsum([len(r[0]) for r in rows])
    cols = np.concatenate([r[0] for r in rows])
    vals = np.concatenate([r[1] for r in rows])
    z = (rng.random((V, nq)) * 30).astype(np.float32)
    z[rng.random((V, nq)) < 0.05] = 0.0
    z[rng.random((V, nq)) < 0.01] = np.float32(1e-20)
    z[rng.random((V, nq)) < 0.01] = np.float32(3e30)
    dev = torch.device("cuda")
    w = 1 << zs
    panels = (nq + w - 1) // w
    Zp = np.zeros((panels, V, w), np.float32)
    for p in range(panels):
        c = z[:, p * w:(p + 1) * w]
        Zp[p, :, :c.shape[1]] = c
    Zd = torch.as_tensor(Zp.ravel(), device=dev)
    o, c_, v_ = (torch.as_tensor(a, device=dev) for a in (offs, cols, vals))
    out = {}
    for dist in (False, True):
        t = torch.empty(n * nq, dtype=torch.float32, device=dev)
        device.spmm(o, c_, v_, n, Zd, w * V, nq, t, nq, 8, z_shift=zs, dist=dist)
        out[dist] = t.cpu().numpy()
    assert np.array_equal(out[False].view(np.uint32), out[True].view(np.uint32))
    ref = np.array([(vals[offs[i]:offs[i + 1]].astype(np.float64)[:, None] * z[cols[offs[i]:offs[i + 1]]]
                     .astype(np.float64)).sum(0) for i in range(n)], dtype=np.float64)
    with np.errstate(over="ignore"):  # the 2^126 weights times 3e30 overflow f32, as in the kernel
        ref = ref.astype(np.float32).ravel()
    assert np.allclose(out[True], ref, rtol=1e-6)


def test_refine_list_overflow_falls_back_to_scan():
    """lcrw_refine_near with a producer list whose count exceeds its capacity scans the
    whole Z instead (device-side decision), giving the same Z as the scan mode; a list
    within capacity refines exactly its entries."""
    import ctypes as C
    import torch
    from paper_1711_07227_b200 import _lib, device
    rng = np.random.default_rng(31)
    V, m = 2000, 64
    c = rng.standard_normal((40, m)).astype(np.float32)
    E = (c[rng.integers(0, 40, V)] + 0.05 * rng.standard_normal((V, m))).astype(np.float32)
    from paper_1711_07227_b200 import synthetic as S
    x2 = S.histograms(50, V, 30, seed=32)
    prep = device.PreparedEmbeddings(E)
    d2 = device.DeviceCSR.upload(x2)
    res = device.Restricted.build(device.DeviceCSR.upload(S.histograms(300, V, 30, seed=33)), prep)
    B, _ = device.gather_rows(prep, d2.cols, "B")
    Z0, zp = device.phase1(res.A, res.a_norms, res.v_e, B, d2.nnz, d2.offsets, d2.n_rows, prep, z_shift=3)
    rep, nxt = prep.representatives(d2.cols)
    device.zero_identical(d2.offsets, d2.n_rows, rep, nxt, res.remap, Z0, zp, 3)
    scan = Z0.clone()
    device.refine_near(scan, zp, 3, res.v_e, d2.n_rows, d2.offsets, d2.cols, res.used, res.a_norms, prep)
    assert not torch.equal(scan, Z0)  # clustered rows: some entries were near
    lst = torch.zeros(16, dtype=torch.int64, device=Z0.device)
    cnt = torch.tensor([1 << 20], dtype=torch.int64, device=Z0.device)  # > capacity 8
    over = Z0.clone()
    _lib.call("lcrw_refine_near", device._p(over), zp, 3, res.v_e, d2.n_rows, device._p(d2.offsets), 0,
              device._p(d2.cols), device._p(prep.E32), device._p(res.used), device._p(prep.E32), prep.m,
              device._p(res.a_norms), device._p(prep.scale), device._p(lst), device._p(cnt), 8, 0, device._stream())
    assert torch.equal(over, scan)
    empty = Z0.clone()
    cnt.zero_()
    _lib.call("lcrw_refine_near", device._p(empty), zp, 3, res.v_e, d2.n_rows, device._p(d2.offsets), 0,
              device._p(d2.cols), device._p(prep.E32), device._p(res.used), device._p(prep.E32), prep.m,
              device._p(res.a_norms), device._p(prep.scale), device._p(lst), device._p(cnt), 8, 0, device._stream())
    assert torch.equal(empty, Z0)  # an empty list changes nothing
    # mark (flagged -> all bits, counted) then finalize without any near pairs: every marked
    # entry is recomputed -- the fix scan's Z, bitwise
    marked = Z0.clone()
    cnt.zero_()
    device.refine_near(marked, zp, 3, res.v_e, d2.n_rows, d2.offsets, d2.cols, res.used, res.a_norms, prep,
                       mode=1, count=cnt)
    n_marked = int(cnt.item())
    assert n_marked > 0 and n_marked == int((marked.view(torch.int32) == -1).sum())
    assert torch.equal(marked.view(torch.int32) == -1, marked != Z0)  # only the marks changed
    device.refine_near(marked, zp, 3, res.v_e, d2.n_rows, d2.offsets, d2.cols, res.used, res.a_norms, prep,
                       mode=2, count=cnt)
    assert torch.equal(marked, scan)
