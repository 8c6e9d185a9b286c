"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the pinned CPU oracle.

Tolerances (written here, justified in DESIGN.md §Precision):
  * distances: |d - d_ref| <= 1e-4 * |d_ref| + 1e-6
    The relative term covers operand rounding (f16 = 11-bit significand, like
    TF32-RN; split 3 x f16 below m = 64), the fp32 tensor-core accumulation
    of the Gram expansion and the reverse direction's 16-bit keys (2^-15).
    The Gram expansion's error scales with the norms, not the distance, so
    entries with d < 0.5 |a| (near-duplicate words, clustered data) are
    recomputed exactly from the f32 rows (lcrw_refine_near); the 1e-6 only
    absorbs values within rounding of zero.
  * exact zeros where the reference has them (identical vectors)
  * spmm / topk_select / restrict_vocabulary: bitwise
  * top-k ids: identical except where the reference's k-th and (k+1)-th
    distances are within the distance tolerance (ties)
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, load_case, rel_close
from oracle import lcrwmd_oracle as O

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1711_07227_b200 import _lib
    _lib.load()


def _pkg():
    from paper_1711_07227_b200 import corpus, distances, kernels
    return corpus, distances, kernels


def _check_topk(d, i, dref_full, k, ATOL=ATOL):
    """Tie-aware top-k check against a full reference matrix (n1, n2)."""
    n1, n2 = dref_full.shape
    for j in range(n2):
        col = dref_full[:, j].astype(np.float64)
        rd, ri = O.topk_select(dref_full[:, j], np.arange(n1), k)
        kk = len(ri)
        assert len(i[j]) == kk
        # our distances agree with the reference distances of the ids we returned
        ok, err = rel_close(d[j], col[i[j]], RTOL, ATOL)
        assert ok, (j, err)
        # and with the reference's k best values position by position
        ok, err = rel_close(d[j], rd, RTOL, ATOL)
        assert ok, (j, err)
        # ids identical except inside tie bands
        tol = RTOL * np.abs(rd) + ATOL
        for r in range(kk):
            if i[j][r] != ri[r]:
                assert abs(col[i[j][r]] - rd[r]) <= 2 * tol[r] + 1e-6, (j, r)


def _atol(E):
    """The absolute term of the tolerance: a constant 1e-6 (no norm-scaled slack)."""
    return ATOL


def test_golden_full_batched_onesided(golden_case):
    name, z, x1, x2 = golden_case
    _, D, _ = _pkg()
    E = z["E"]
    ATOL = _atol(E)
    full = D.lcrwmd_full(x1, x2, E).values
    ok, err = rel_close(full, z["full"], RTOL, ATOL)
    assert ok, (name, "full", err)
    assert np.array_equal(full == 0, z["full"] == 0), name
    bat = D.lcrwmd_batched(x1, x2, E)
    ok, err = rel_close(bat, z["batched"], RTOL, ATOL)
    assert ok, (name, "batched", err)
    assert np.array_equal(bat == 0, z["batched"] == 0), name
    one = D.lcrwmd_one_sided(x1, x2.row(0), E)
    ok, err = rel_close(one, z["one_sided0"], RTOL, ATOL)
    assert ok, (name, "one_sided", err)
    q0 = x2.row(0)
    nwd = D.nearest_word_distances(E, E[q0.word_ids])
    ok, err = rel_close(nwd, z["nwd0"], RTOL, 1e-4)
    assert ok, (name, "nwd", err)
    assert np.array_equal(nwd == 0, z["nwd0"] == 0), name


def test_golden_topk(golden_case):
    name, z, x1, x2 = golden_case
    _, D, _ = _pkg()
    k = int(z["topk_k"])
    res = D.lcrwmd_topk(x1, x2, z["E"], k)
    d = [r.distances for r in res]
    i = [r.ids for r in res]
    _check_topk(d, i, z["full"], k, _atol(z["E"]))


def test_golden_restrict_spmm(golden_case):
    name, z, x1, x2 = golden_case
    C, _, K = _pkg()
    xr, er, remap = C.restrict_vocabulary(x1, z["E"])
    assert np.array_equal(xr.column_ids, z["r1_ids"])
    assert np.array_equal(er, z["r1_E"])
    assert np.array_equal(remap, z["r1_remap"])
    assert np.array_equal(K.spmm(x1, z["spmm_z"]), z["spmm"])  # bitwise (fp64 accumulation)
    assert np.array_equal(K.spmv(x1, z["spmm_z"][:, 2]), z["spmm"][:, 2])


def test_golden_topk_select_merge():
    _, _, K = _pkg()
    z = np.load(GOLDEN / "topk.npz")
    for k in (1, 10, 128, 20_000):
        r = K.topk_select(z["d"], z["ids"], k)
        assert np.array_equal(r.distances, z[f"d{k}"]), k
        assert np.array_equal(r.ids, z[f"i{k}"]), k
    parts = [K.topk_select(z["d"][a:a + 2500], z["ids"][a:a + 2500], 64) for a in range(0, 10_000, 2500)]
    m = K.topk_merge(parts, 64)
    assert np.array_equal(m.distances, z["merge_d"]) and np.array_equal(m.ids, z["merge_i"])


def test_spec_known_answers():
    C, D, K = _pkg()
    E = np.array([[0, 0], [1, 0], [0, 2]], dtype=np.float32)
    x1 = C.HistogramSet(np.array([0, 2]), np.array([0, 1], np.int32), np.array([.5, .5], np.float32), 3)
    x2 = C.HistogramSet(np.array([0, 2]), np.array([1, 2], np.int32), np.array([.5, .5], np.float32), 3)
    assert D.lcrwmd_full(x1, x2, E).values[0, 0] == pytest.approx(1.0, rel=1e-6)
    z = D.nearest_word_distances(np.array([[0, 0]], np.float32), np.array([[3, 4]], np.float32))
    assert z[0] == pytest.approx(5.0, rel=1e-6)
    xs = C.HistogramSet(np.array([0, 1]), np.array([2], np.int32), np.array([1.0], np.float32), 4)
    assert K.spmm(xs, np.array([[5], [6], [7], [8]], np.float32))[0, 0] == 7.0
    r = K.topk_select(np.array([3, 1, 2], np.float32), np.array([0, 1, 2]), 2)
    assert list(r.ids) == [1, 2] and list(r.distances) == [1, 2]
    r = K.topk_select(np.array([1.0, 1.0], np.float32), np.array([7, 3]), 1)
    assert list(r.ids) == [3]
    # X1 == X2 -> zero diagonal
    z0, a, _ = load_case("small_m16")
    d = D.lcrwmd_full(a, a, z0["E"]).values
    assert np.all(np.diag(d) == 0)
    # symmetry when X1 == X2, to the reverse direction's 16-bit key rounding (2^-15 relative)
    ok, err = rel_close(d, d.T, 4e-5, 1e-6)
    assert ok, err


def test_errors_match_reference():
    C, D, K = _pkg()
    z, x1, x2 = load_case("small_m16")
    with pytest.raises(ValueError, match="do not match embedding rows"):
        D.lcrwmd_full(x1, x2, z["E"][:-1])
    with pytest.raises(ValueError, match="k must be >= 1"):
        K.topk_select(np.zeros(3, np.float32), np.arange(3), 0)
    with pytest.raises(ValueError, match="spmm expects a 2-d right-hand side"):
        K.spmm(x1, np.zeros(x1.n_cols, np.float32))
    with pytest.raises(ValueError, match="batch must hold at least one query"):
        D.lcrwmd_batched(x1, x1.slice_rows(0, 0), z["E"])
    bad = C.HistogramSet(np.array([0, 1, 1]), np.array([3], np.int32), np.array([1.0], np.float32), x1.n_cols)
    with pytest.raises(C.CorpusError, match="at least one word"):
        D.lcrwmd_full(bad, x2, z["E"])


@pytest.mark.parametrize("clustered", [False, True])
def test_c1_shaped_vs_oracle(clustered):
    """Config-1 shape (m=300, h~40) at reduced n: symmetric + one-sided + top-k vs the oracle."""
    from paper_1711_07227_b200 import synthetic as S
    _, D, _ = _pkg()
    V = 5000
    E = S.embeddings(V, 300, seed=3, clustered=clustered, centers=200)
    x1 = S.histograms(600, V, 40, seed=4)
    x2 = S.histograms(40, V, 40, seed=5)
    ref = O.lcrwmd_full(x1, x2, E, threads=8)
    got = D.lcrwmd_full(x1, x2, E).values
    ok, err = rel_close(got, ref, RTOL, ATOL)  # 1e-4 relative (+ 1e-6)
    assert ok, err
    res = D.lcrwmd_topk(x1, x2, E, 10)
    _check_topk([r.distances for r in res], [r.ids for r in res], ref, 10)
    one = D.lcrwmd_batched(x1, x2, E)
    ref1 = O.lcrwmd_batched(x1, x2, E)
    ok, err = rel_close(one, ref1, RTOL, ATOL)
    assert ok, err


def test_queries_from_docs_exact_self_match():
    """Paper protocol: queries sampled from the resident set -> self at distance exactly 0."""
    from paper_1711_07227_b200 import synthetic as S
    _, D, _ = _pkg()
    V = 3000
    E = S.embeddings(V, 300, seed=8)
    x1 = S.histograms(900, V, 30, seed=9)
    idx = np.arange(5, 900, 37)
    x2 = x1.take_rows(idx)
    res = D.lcrwmd_topk(x1, x2, E, 3)
    for j, r in enumerate(res):
        assert r.distances[0] == 0.0 and r.ids[0] == idx[j]


def test_large_sampled_parity_and_batching():
    """Many docs (multiple reverse batches, many Phase-1 ranges): sampled parity by subset invariance."""
    import torch
    from paper_1711_07227_b200 import device, synthetic as S
    V = 20000
    E = S.embeddings(V, 300, seed=21)
    x1 = S.histograms(30000, V, 50, seed=22)
    x2 = S.histograms(64, V, 50, seed=23)
    prep = device.PreparedEmbeddings(E)
    d1 = device.DeviceCSR.upload(x1)
    d2 = device.DeviceCSR.upload(x2)
    full = device.symmetric(d1, d2, prep, None, z2_budget_bytes=4 * 200 * 8192).cpu().numpy()
    rng = np.random.default_rng(0)
    di = np.sort(rng.choice(30000, 300, replace=False))
    qj = np.sort(rng.choice(64, 12, replace=False))
    ref = O.lcrwmd_full(x1.take_rows(di), x2.take_rows(qj), E, threads=8)
    ok, err = rel_close(full[np.ix_(di, qj)], ref, RTOL, ATOL)
    assert ok, err
    # fused top-k over several doc batches == top-k of the full matrix
    td, ti = device.symmetric(d1, d2, prep, 10, z2_budget_bytes=4 * 200 * 8192)
    td, ti = td.cpu().numpy(), ti.cpu().numpy()
    for j in range(64):
        rd, ri = O.topk_select(full[:, j], np.arange(30000), 10)
        assert np.array_equal(td[j], rd) and np.array_equal(ti[j], ri)
    torch.cuda.synchronize()


def test_sharded_pipeline_emulated_ranks():
    """The multi-GPU decomposition run rank by rank on one GPU: vocabulary-slice
    Z1 blocks (blocked SpMM addressing), per-shard reverse + top-k with global ids,
    merge -- identical to the single-GPU result for several world sizes."""
    import torch
    from paper_1711_07227_b200 import device, parallel, synthetic as S
    V, k = 6000, 10
    E = S.embeddings(V, 300, seed=31)
    x1 = S.histograms(5000, V, 40, seed=32)
    x2 = S.histograms(37, V, 40, seed=33)
    prep = device.PreparedEmbeddings(E)
    dx2 = device.DeviceCSR.upload(x2)
    want_d, want_i = device.symmetric(device.DeviceCSR.upload(x1), dx2, prep, k)
    for W in (2, 3, 8):
        slices = [parallel.z1_slice(dx2, prep, r, W) for r in range(W)]
        R = slices[0][1]
        zall = torch.stack([z for z, _ in slices])
        parts_d, parts_i = [], []
        for r in range(W):
            lo, hi = parallel.shard_range(x1.n_rows, r, W)
            dx1 = device.DeviceCSR.upload(x1.slice_rows(lo, hi))
            d1 = parallel.d1_from_slices(dx1, zall, R, x2.n_rows)
            ld, li = device.symmetric(dx1, dx2, prep, k, d1=d1, id_offset=lo)
            parts_d.append(ld)
            parts_i.append(li)
        cd = torch.cat(parts_d, 1).contiguous()
        ci = torch.cat(parts_i, 1).contiguous()
        gd, gi = device.topk_rows(cd, ci, x2.n_rows, cd.shape[1], k)
        assert torch.equal(gd, want_d) and torch.equal(gi, want_i), W


@pytest.mark.parametrize("mode", ["table", "gemm"])
def test_sharded_pipeline_emulated_ranks_near_pairs(monkeypatch, mode):
    """The same decomposition on clustered embeddings with each rank's query side
    (device.QuerySide: restriction, table, near word pairs) shared by its forward slice and
    its reverse pass, as parallel.sharded_topk does: the near pairs are built per rank from
    its own slice's marks, and the merged top-k equals the single-GPU result bitwise."""
    import torch
    from paper_1711_07227_b200 import device, parallel, synthetic as S
    monkeypatch.setenv("LCRW_REVERSE", mode)
    V, k, W = 4000, 10, 3
    E = S.embeddings(V, 300, seed=41, clustered=True, centers=40, spread=0.1)
    x1 = S.histograms(3000, V, 40, seed=42)
    x2 = S.histograms(29, V, 40, seed=43)
    prep = device.PreparedEmbeddings(E)
    dx2 = device.DeviceCSR.upload(x2)
    want_d, want_i = device.symmetric(device.DeviceCSR.upload(x1), dx2, prep, k)
    shards = [parallel.shard_range(x1.n_rows, r, W) for r in range(W)]
    dx1s = [device.DeviceCSR.upload(x1.slice_rows(lo, hi)) for lo, hi in shards]
    qsides = [device.QuerySide.build(dx2, prep, dx1s[r].nnz) for r in range(W)]
    slices = [parallel.z1_slice(dx2, prep, r, W, qsides[r].near) for r in range(W)]
    assert all(q.near is not None and q.near.n_candidates() > 0 for q in qsides)
    R = slices[0][1]
    zall = torch.stack([z for z, _ in slices])
    parts_d, parts_i = [], []
    for r, (lo, hi) in enumerate(shards):
        d1 = parallel.d1_from_slices(dx1s[r], zall, R, x2.n_rows)
        ld, li = device.symmetric(dx1s[r], dx2, prep, k, d1=d1, id_offset=lo, prepared=qsides[r])
        parts_d.append(ld)
        parts_i.append(li)
    cd = torch.cat(parts_d, 1).contiguous()
    ci = torch.cat(parts_i, 1).contiguous()
    gd, gi = device.topk_rows(cd, ci, x2.n_rows, cd.shape[1], k)
    assert torch.equal(gd, want_d) and torch.equal(gi, want_i)


@pytest.mark.slow
def test_c2_full_size_sampled_parity():
    """BASELINE configs[1] at full size (1M docs x 1k queries, V=100k, m=300):
    sampled entries of the symmetric matrix vs the oracle on the sampled subsets
    (subset invariance), and fused top-k == top-k of the full matrix."""
    import torch
    from paper_1711_07227_b200 import device, synthetic as S
    V = 100_000
    E = S.embeddings(V, 300, seed=0)
    x1 = S.histograms(1_000_000, V, 50, seed=1)
    x2 = S.histograms(1000, V, 50, seed=2)
    prep = device.PreparedEmbeddings(E)
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
    full = device.symmetric(d1, d2, prep, None)  # (1M, 1k) on device, 4 GB
    rng = np.random.default_rng(5)
    di = np.sort(rng.choice(1_000_000, 256, replace=False))
    qj = np.sort(rng.choice(1000, 16, replace=False))
    got = full[torch.as_tensor(di, device=full.device)][:, torch.as_tensor(qj, device=full.device)].cpu().numpy()
    ref = O.lcrwmd_full(x1.take_rows(di), x2.take_rows(qj), E, threads=O.default_threads())
    ok, err = rel_close(got, ref, RTOL, ATOL)
    assert ok, err
    print(f"C2 sampled parity: max rel err {float(np.max(np.abs(got - ref) / np.abs(ref))):.2e}")
    td, ti = device.symmetric(d1, d2, prep, 10)
    fd, fi = device.topk_rows(full.t().contiguous(),
                              torch.arange(1_000_000, device=full.device).repeat(1000, 1).contiguous(),
                              1000, 1_000_000, 10)
    assert torch.equal(td, fd) and torch.equal(ti, fi)


# --- edge cases ----------------------------------------------------------------

def _rand_set(rng, n, V, lo, hi):
    from paper_1711_07227_b200.corpus import HistogramSet
    rows = []
    for _ in range(n):
        h = int(rng.integers(lo, hi + 1))
        ids = np.sort(rng.choice(V, size=min(h, V), replace=False)).astype(np.int32)
        u = rng.random(len(ids)) + 0.1
        rows.append((ids, (u / u.sum()).astype(np.float32)))
    return HistogramSet.from_rows(rows, V)


def test_k_larger_than_docs_and_single_rows():
    _, D, _ = _pkg()
    rng = np.random.default_rng(41)
    E = rng.standard_normal((60, 300)).astype(np.float32)
    x1 = _rand_set(rng, 5, 60, 1, 9)
    x2 = _rand_set(rng, 3, 60, 1, 9)
    ref = O.lcrwmd_full(x1, x2, E)
    res = D.lcrwmd_topk(x1, x2, E, 10)
    assert all(len(r.ids) == 5 for r in res)
    _check_topk([r.distances for r in res], [r.ids for r in res], ref, 10)
    one = D.lcrwmd_full(x1.slice_rows(0, 1), x2.slice_rows(0, 1), E).values
    ok, err = rel_close(one, ref[:1, :1], RTOL, ATOL)
    assert ok, err


def test_very_long_segments_cross_tiles_and_ranges():
    """Docs of up to 3000 words: Phase-1 segments span many 256-column tiles and
    exceed the column-range size, exercising the carried running minimum."""
    _, D, _ = _pkg()
    rng = np.random.default_rng(42)
    V = 6000
    E = rng.standard_normal((V, 300)).astype(np.float32)
    x1 = _rand_set(rng, 40, V, 1, 3000)
    x2 = _rand_set(rng, 6, V, 500, 2500)
    ref = O.lcrwmd_full(x1, x2, E, threads=8)
    got = D.lcrwmd_full(x1, x2, E).values
    ok, err = rel_close(got, ref, RTOL, ATOL)
    assert ok, err
    qv = E[rng.choice(V, 1500, replace=False)]
    ok, err = rel_close(D.nearest_word_distances(E, qv), O.nearest_word_distances(E, qv), RTOL, 1e-4)
    assert ok, err


def test_many_queries_multiple_groups():
    """More than 1024 queries: the reverse pass splits queries into groups."""
    _, D, _ = _pkg()
    rng = np.random.default_rng(43)
    V = 2000
    E = rng.standard_normal((V, 64)).astype(np.float32)
    x1 = _rand_set(rng, 300, V, 5, 40)
    x2 = _rand_set(rng, 1500, V, 5, 40)
    ref = O.lcrwmd_full(x1, x2, E, threads=8)
    got = D.lcrwmd_full(x1, x2, E).values
    ok, err = rel_close(got, ref, RTOL, 1e-5 * float(np.sqrt((E.astype(np.float64) ** 2).sum(1).max())))
    assert ok, err
    res = D.lcrwmd_topk(x1, x2, E, 7)
    _check_topk([r.distances for r in res], [r.ids for r in res], ref, 7,
                1e-5 * float(np.sqrt((E.astype(np.float64) ** 2).sum(1).max())))


@pytest.mark.parametrize("m", [1, 448, 509, 510, 768, 1024])
def test_dimension_extremes(m):
    """m > 509 (operand K > 512): the Phase-1 kernel streams A's K blocks through the ring."""
    _, D, _ = _pkg()
    rng = np.random.default_rng(44 + m)
    V = 400
    E = rng.standard_normal((V, m)).astype(np.float32)
    x1 = _rand_set(rng, 30, V, 1, 20)
    x2 = _rand_set(rng, 5, V, 1, 20)
    ref = O.lcrwmd_full(x1, x2, E)
    got = D.lcrwmd_full(x1, x2, E).values
    ok, err = rel_close(got, ref, RTOL, _atol(E))
    assert ok, (m, err)


def test_dimension_too_large_is_reported():
    _, D, _ = _pkg()
    rng = np.random.default_rng(45)
    E = rng.standard_normal((50, 4094)).astype(np.float32)
    x1 = _rand_set(rng, 4, 50, 1, 5)
    with pytest.raises(NotImplementedError, match="unsupported"):
        D.lcrwmd_full(x1, x1, E)


@pytest.mark.gpu
@pytest.mark.parametrize("k,row_len", [(1, 100_003), (10, 100_003), (32, 98_304), (33, 100_003), (10, 98_304)])
def test_topk_matrix_rows_long_rows_with_ties(k, row_len):
    """lcrw_topk_rows (kernels.py:210-223 per row): chunked warp lists + merge for long rows;
    quantised values make ties common, so the (distance, id) tie-break is exercised."""
    import torch
    from paper_1711_07227_b200 import device
    rng = np.random.default_rng(k)
    n_rows, id_base = 7, 5_000   # row_len % 4 == 0 takes the float4 path
    D = np.round(rng.random((n_rows, row_len)) * 300).astype(np.float32)   # values 0..300: many ties
    D[3, :] = 1.0                                                          # an all-tie row
    Dd = torch.from_numpy(D).cuda()
    od = torch.empty((n_rows, k), dtype=torch.float32, device="cuda")
    oi = torch.empty((n_rows, k), dtype=torch.int64, device="cuda")
    device.topk_matrix_rows(Dd, n_rows, row_len, row_len, id_base, k, od, oi)
    od, oi = od.cpu().numpy(), oi.cpu().numpy()
    for r in range(n_rows):
        cols = np.arange(row_len)
        order = np.lexsort((cols, D[r]))[:k]
        assert np.array_equal(oi[r], order + id_base), r
        assert np.array_equal(od[r], D[r, order]), r


@pytest.mark.gpu
def test_load_index_to_device(tmp_path):
    """device.load_index: the reference-written LCRW file lands in HBM bitwise, and the
    symmetric bound computed from it equals the one from the host arrays."""
    import torch
    from paper_1711_07227_b200 import corpus as Cc, device, distances
    g = np.load(GOLDEN / "widen_m300.npz")
    f = tmp_path / "x.lcrw"
    f.write_bytes(g["index_bytes"].tobytes())
    hs, E, words = Cc.read_index_file(f)
    dx, Ed, w2 = device.load_index(f)
    assert w2 == words and dx.n_cols == hs.n_cols and dx.n_rows == hs.n_rows
    assert np.array_equal(dx.offsets.cpu().numpy(), hs.row_offsets)
    assert np.array_equal(dx.cols.cpu().numpy(), hs.column_ids)
    assert np.array_equal(dx.vals.cpu().numpy(), hs.values)
    assert torch.equal(Ed.cpu(), torch.from_numpy(E))
    q = hs.take_rows([0, 3, 5])
    a = distances.lcrwmd_full(hs, q, E).values
    b = distances.lcrwmd_full(hs, q, Ed.cpu().numpy()).values
    assert np.array_equal(a, b)


def _abs_tol(*mats):
    return 1e-5 * max(float(np.sqrt((np.asarray(M, np.float64) ** 2).sum(1).max())) for M in mats)


@pytest.mark.gpu
def test_widen_rows_gpu(widen_case):
    """SURVEY §8f rows on the GPU vs the reference's golden outputs:
    centroids (bitwise), pairwise_euclidean and wcd_block (Phase-1 kernel, singleton
    segments), rwmd_bounds / rwmd_quadratic (both LC-RWMD directions)."""
    corpus, distances, kernels = _pkg()
    name, z, w, x1, x2, _, _ = widen_case
    E = z["E"]
    c1 = kernels.centroids(x1, E)
    assert np.array_equal(c1, w["c1"]), name
    pair = kernels.pairwise_euclidean(E[:17], E[5:40]).values
    ok, err = rel_close(pair, w["pair"], RTOL, _abs_tol(E))
    assert ok, (name, "pair", err)
    assert np.all(pair[np.arange(5, 17), np.arange(0, 12)] == 0.0)  # identical rows -> exactly 0
    wcd = distances.wcd_block(x1, x2, E).values
    ok, err = rel_close(wcd, w["wcd"], RTOL, _abs_tol(w["c1"]))
    assert ok, (name, "wcd", err)
    b1, b2 = distances.rwmd_bounds(x1, x2, E)
    for got, key in ((b1, "b1"), (b2, "b2")):
        ok, err = rel_close(got, w[key], RTOL, _abs_tol(E))
        assert ok, (name, key, err)
    q = distances.rwmd_quadratic(x1, x2, E).values
    ok, err = rel_close(q, w["quadratic"], RTOL, _abs_tol(E))
    assert ok, (name, "quadratic", err)
    assert np.array_equal(q, distances.lcrwmd_full(x1, x2, E).values)


@pytest.mark.gpu
def test_solve_emd_gpu_matches_reference():
    """solve_emd (emd.py:120-194) on the GPU: reference objectives (1x1, 1xn, nx1, ties,
    up to 60x45), marginals, dual feasibility and complementary slackness of the plan."""
    from paper_1711_07227_b200 import emd
    g = np.load(GOLDEN / "emd.npz")
    for i in range(8):
        s, d, c = g[f"s{i}"], g[f"d{i}"], g[f"c{i}"]
        plan = emd.solve_emd(emd.TransportProblem(s, d, c))
        ref = float(g[f"obj{i}"])
        assert abs(plan.objective - ref) <= 1e-9 * max(1.0, ref), (i, plan.objective, ref)
        flow = np.zeros(c.shape)
        flow[plan.source_ids, plan.target_ids] = plan.amounts
        assert np.allclose(flow.sum(1), s, atol=1e-6) and np.allclose(flow.sum(0), d, atol=1e-6)
        red = c - plan.dual_source[:, None] - plan.dual_sink[None, :]
        assert red.min() >= -1e-7, i
        assert np.all(np.abs(red[plan.source_ids, plan.target_ids]) <= 1e-7), i
        dual = float(s @ plan.dual_source + d @ plan.dual_sink)
        assert abs(dual - plan.objective) <= 1e-7 * max(1.0, abs(ref)), i
    with pytest.raises(ValueError, match="must each sum to 1.0"):
        emd.solve_emd(emd.TransportProblem(np.array([0.5]), np.array([1.0]), np.ones((1, 1))))
    with pytest.raises(ValueError, match="nonnegative and finite"):
        emd.solve_emd(emd.TransportProblem(np.array([1.0]), np.array([1.0]), -np.ones((1, 1))))


@pytest.mark.gpu
def test_wmd_and_prefiltered_topk_gpu(widen_case):
    """wmd / prefiltered_topk_wmd (emd.py:199-261) vs the reference's golden outputs
    (dyadic weights, where the reference's solver never trips on float32 totals);
    general histograms vs the oracle restatement (which has the same exhaustion rule)."""
    from paper_1711_07227_b200 import emd
    name, z, w, x1, x2, xd1, xd2 = widen_case
    E = z["E"]
    q = xd2.row(0)
    for i, ref in enumerate(w["wmd0"]):
        got = emd.wmd(xd1.row(i), q, E)
        assert abs(got - ref) <= 1e-7 * max(1.0, ref), (name, i, got, ref)
    for j in range(2):
        r, solves = emd.prefiltered_topk_wmd(xd1, xd2.row(j), E, 4)
        assert np.array_equal(r.ids, w[f"pf{j}_i"]), (name, j, r.ids, w[f"pf{j}_i"])
        assert np.allclose(r.distances, w[f"pf{j}_d"], rtol=1e-7, atol=1e-12), name
        assert solves >= int(w[f"pf{j}_solves"])  # slack 1e-4 >= the reference's 1e-6
    for i in range(min(6, x1.n_rows)):  # float32-normalised weights (reference raises on ~half)
        a, b = x1.row(i), x2.row(0)
        got = emd.wmd(a, b, E)
        ref = O.wmd(a.word_ids, a.weights, b.word_ids, b.weights, E)
        assert abs(got - ref) <= 1e-7 * max(1.0, ref), (name, i, got, ref)


@pytest.mark.gpu
def test_prefiltered_batch_equals_single(widen_case):
    """The multi-query prefilter gives each query exactly the single-query result."""
    from paper_1711_07227_b200 import emd
    name, z, w, _, _, xd1, xd2 = widen_case
    E = z["E"]
    res, solves = emd.prefiltered_topk_wmd_batch(xd1, xd2, E, 4)
    for j in range(xd2.n_rows):
        r, s = emd.prefiltered_topk_wmd(xd1, xd2.row(j), E, 4)
        assert np.array_equal(r.ids, res[j].ids) and np.array_equal(r.distances, res[j].distances), (name, j)
        assert s == solves[j], (name, j)


@pytest.mark.gpu
def test_engine_index_and_partition_invariance(tmp_path):
    """SPEC.md engine (333-383): build -> save -> open is bitwise, run_query is identical
    for P in {1, 2, 3, 5} for every method, self-exclusion drops the query's own id,
    k = 1 without it returns the query itself at distance 0, rwmd == lc-rwmd, and the
    pruned exact WMD equals the exhaustive one."""
    from paper_1711_07227_b200 import corpus as Cc, engine, synthetic as S
    rng = np.random.default_rng(3)
    V, m = 600, 24
    words = [f"t{i}" for i in range(V)]
    vocab = Cc.Vocabulary.from_words(words)
    E = S.embeddings(V, m, seed=4)
    docs = [[words[int(t)] for t in rng.integers(0, V, int(rng.integers(3, 15)))] + ["zzz-oov"] for _ in range(37)]
    labels = [f"L{i % 3}" for i in range(37)]
    idx = engine.build_index(docs, vocab, E, stopwords=frozenset({"t0", "t1"}), labels=labels)
    engine.save_index(idx, tmp_path / "i.lcrw")
    back = engine.open_index(tmp_path / "i.lcrw")
    assert back.words == idx.words and back.labels == labels
    assert np.array_equal(back.embeddings, idx.embeddings)
    assert np.array_equal(back.docs.row_offsets, idx.docs.row_offsets)
    assert np.array_equal(back.docs.column_ids, idx.docs.column_ids)
    assert np.array_equal(back.docs.values, idx.docs.values)
    qids = [2, 7, 30]
    queries = idx.docs.take_rows(qids)
    for method in ("lc-rwmd", "rwmd", "wcd", "wmd-pruned"):
        ref = engine.run_query(back, queries, engine.QueryPlan(method=method, k=4))
        for P in (2, 3, 5):
            got = engine.run_query(back, queries, engine.QueryPlan(method=method, k=4, partitions=P))
            for a, b in zip(ref, got):
                assert np.array_equal(a.ids, b.ids) and np.array_equal(a.distances, b.distances), (method, P)
        own = engine.run_query(back, queries, engine.QueryPlan(method=method, k=1))
        assert [int(t.ids[0]) for t in own] == qids and all(float(t.distances[0]) == 0.0 for t in own), method
        ex = engine.run_query(back, queries, engine.QueryPlan(method=method, k=3, self_exclusion=True, partitions=2),
                              query_ids=qids)
        assert all(q not in t.ids for q, t in zip(qids, ex)) and all(len(t.ids) == 3 for t in ex), method
    lc = engine.run_query(back, queries, engine.QueryPlan(method="lc-rwmd", k=5))
    rw = engine.run_query(back, queries, engine.QueryPlan(method="rwmd", k=5))
    assert all(np.array_equal(a.ids, b.ids) for a, b in zip(lc, rw))
    ex_all = engine.run_query(back, queries, engine.QueryPlan(method="wmd", k=4, partitions=3))
    pr = engine.run_query(back, queries, engine.QueryPlan(method="wmd-pruned", k=4))
    for a, b in zip(ex_all, pr):
        assert np.array_equal(a.ids, b.ids) and np.allclose(a.distances, b.distances, rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [4096, 37])
def test_all_pairs_matches_symmetric(batch):
    """lcrwmd_all_pairs_topk (forward direction only, D = max(D1, D1^T)) vs the reference
    symmetric bound of the set against itself; exactly symmetric, zero diagonal."""
    import torch
    from paper_1711_07227_b200 import device
    _, D, _ = _pkg()
    rng = np.random.default_rng(46)
    V = 3000
    E = rng.standard_normal((V, 300)).astype(np.float32)
    x = _rand_set(rng, 230, V, 2, 60)
    ref = O.lcrwmd_full(x, x, E, threads=8)
    full = device.all_pairs(device.DeviceCSR.upload(x), device.PreparedEmbeddings(E), batch).cpu().numpy()
    assert np.array_equal(full, full.T) and np.all(np.diag(full) == 0.0)
    ok, err = rel_close(full, ref, RTOL, _atol(E))
    assert ok, err
    res = D.lcrwmd_all_pairs_topk(x, E, 6, batch_size=batch)
    _check_topk([r.distances for r in res], [r.ids for r in res], ref, 6, _atol(E))
    assert all(int(r.ids[0]) == j and float(r.distances[0]) == 0.0 for j, r in enumerate(res))


@pytest.mark.gpu
def test_all_pairs_sharded_emulated_ranks():
    """Sharded all-pairs on one GPU: per-shard C = D1[:, S_r] (all docs against the shard's
    docs as queries), the all_to_all row blocks taken directly, max_transposed_into
    combine -- bitwise equal to the single-set all_pairs for W in {2, 3};
    parallel.sharded_all_pairs_topk at world 1 equals lcrwmd_all_pairs_topk."""
    import torch
    from paper_1711_07227_b200 import device, parallel
    _, D, _ = _pkg()
    rng = np.random.default_rng(47)
    V = 2500
    E = rng.standard_normal((V, 300)).astype(np.float32)
    x = _rand_set(rng, 97, V, 2, 40)
    prep = device.PreparedEmbeddings(E)
    dx = device.DeviceCSR.upload(x)
    want = device.all_pairs(dx, prep, 20)
    n = x.n_rows
    res_all = device.Restricted.build(dx, prep)
    for W in (2, 3):
        ranges = [parallel.shard_range(n, r, W) for r in range(W)]
        Cs = []
        for lo, hi in ranges:
            c = torch.empty((n, hi - lo), dtype=torch.float32, device="cuda")
            device.forward_rows_into(res_all, prep, device.DeviceCSR.upload(x.slice_rows(lo, hi)), c, 20)
            Cs.append(c)
        rows = []
        for r, (a0, a1) in enumerate(ranges):
            out = torch.empty((a1 - a0, n), dtype=torch.float32, device="cuda")
            for s_, (b0, b1) in enumerate(ranges):
                recv = Cs[s_][a0:a1].contiguous()  # what the all_to_all delivers from rank s
                device.max_transposed_into(out[:, b0:b1], recv, Cs[r][b0:b1])
            rows.append(out)
        got = torch.cat(rows)
        assert torch.equal(got, want), W
    od, oi = parallel.sharded_all_pairs_topk(dx, dx, 0, prep, 5, 20)
    res = D.lcrwmd_all_pairs_topk(x, E, 5, batch_size=20)
    assert np.array_equal(oi.cpu().numpy(), np.stack([r.ids for r in res]))


@pytest.mark.gpu
def test_emd_large_problems():
    """The shared-memory solver (h1 + h2 > 128) and the global-memory one (a problem too
    large for shared memory, e.g. 200 x 200) agree with the oracle restatement."""
    from paper_1711_07227_b200 import emd
    rng = np.random.default_rng(48)
    for h1, h2 in ((90, 70), (130, 20), (200, 200), (260, 90)):
        s = rng.random(h1) + 0.05
        d = rng.random(h2) + 0.05
        s /= s.sum()
        d /= d.sum()
        c = rng.random((h1, h2)) * 5
        plan = emd.solve_emd(emd.TransportProblem(s, d, c))
        ref = O.solve_emd_objective(s, d, c)
        assert abs(plan.objective - ref) <= 1e-9 * max(1.0, ref), (h1, h2, plan.objective, ref)
    # long documents through the embedding path (costs formed in-kernel), global-memory state
    V, m = 600, 24
    E = rng.standard_normal((V, m)).astype(np.float32)
    from paper_1711_07227_b200.corpus import Histogram
    for h1, h2 in ((180, 150),):
        ids1 = np.sort(rng.choice(V, h1, replace=False)).astype(np.int32)
        ids2 = np.sort(rng.choice(V, h2, replace=False)).astype(np.int32)
        w1 = np.full(h1, 1.0 / h1, np.float32)
        w2 = np.full(h2, 1.0 / h2, np.float32)
        got = emd.wmd(Histogram(ids1, w1), Histogram(ids2, w2), E)
        c = O.pairwise_euclidean(E[ids1], E[ids2]).astype(np.float64)
        ref = O.solve_emd_objective(w1.astype(np.float64), w2.astype(np.float64), c)
        assert abs(got - ref) <= 1e-9 * max(1.0, ref), (h1, h2, got, ref)


def test_emd_degenerate_ties_same_plan_and_duals():
    """Degenerate problems (small integer costs, uniform dyadic weights: many equal path
    lengths) -- the GPU solver picks the reference's augmenting paths (lowest-index sink
    among equal distances, emd.py:166-167), so plan and duals match, not only the objective."""
    from paper_1711_07227_b200 import emd
    rng = np.random.default_rng(77)
    for trial in range(60):
        h1, h2 = int(rng.integers(2, 12)), int(rng.integers(2, 12))
        if trial % 3 == 2:
            h1, h2 = int(rng.integers(40, 70)), int(rng.integers(40, 70))  # register-state kernel, 2-3 slots
        s = np.full(h1, 1.0 / 16) if h1 == 16 else rng.integers(1, 4, h1).astype(np.float64)
        d = rng.integers(1, 4, h2).astype(np.float64)
        s /= s.sum()
        d /= d.sum()
        c = rng.integers(0, 3, (h1, h2)).astype(np.float64)
        plan = emd.solve_emd(emd.TransportProblem(s, d, c))
        obj, flow, phi = O.solve_emd_plan(s, d, c)
        keep = flow > 1e-9
        pi, qi = np.nonzero(keep)
        assert abs(plan.objective - obj) <= 1e-12 * max(1.0, obj), trial
        assert np.array_equal(plan.source_ids, pi) and np.array_equal(plan.target_ids, qi), trial
        np.testing.assert_allclose(plan.amounts, flow[keep], rtol=0, atol=1e-12)
        np.testing.assert_allclose(plan.dual_sink, phi[h1:], rtol=0, atol=1e-12)
        np.testing.assert_allclose(plan.dual_source, -phi[:h1], rtol=0, atol=1e-12)


def test_emd_strict_unbalanced_opt_in(monkeypatch):
    """Totals differing by more than 1e-9 (but within the 1e-6 balance check): by default the
    transported mass is solved; STRICT_UNBALANCED raises the reference's error (emd.py:153-162)."""
    from paper_1711_07227_b200 import emd
    s = np.array([0.5, 0.5 + 4e-7])
    d = np.array([0.25, 0.75])
    c = np.array([[1.0, 2.0], [3.0, 0.5]])
    plan = emd.solve_emd(emd.TransportProblem(s, d, c))
    assert abs(plan.objective - O.solve_emd_objective(s, d, c)) <= 1e-12
    monkeypatch.setattr(emd, "STRICT_UNBALANCED", True)
    with pytest.raises(ValueError, match="no augmenting path"):
        emd.solve_emd(emd.TransportProblem(s, d, c))


# --- SPEC.md acceptance criteria (reference SPEC, "ACCEPTANCE CRITERIA") --------------

def _tiny_set(rng, n, V, hmax, hmin=1):
    from paper_1711_07227_b200.corpus import HistogramSet
    rows = []
    for _ in range(n):
        h = int(rng.integers(hmin, hmax + 1))
        ids = np.sort(rng.choice(V, size=h, replace=False)).astype(np.int32)
        c = rng.integers(1, 5, h).astype(np.int64)
        tot = int(c.sum())
        scale = 1 << int(np.ceil(np.log2(tot)))
        c[0] += scale - tot  # dyadic weights: exact in f32, totals exactly 1
        rows.append((ids, (c / scale).astype(np.float32)))
    return HistogramSet.from_rows(rows, V)


@pytest.mark.gpu
def test_acceptance_1_lcrwmd_equals_quadratic_rwmd():
    """Criterion 1: lcrwmd_full equals the quadratic RWMD (computed pair by pair by the
    oracle, distances.py:78-130) within 1e-5 relative; n1=200, n2=50, v_e <= 1000,
    h in [2, 32], m = 16 (10 random instances here, the oracle's quadratic form being slow)."""
    _, D, _ = _pkg()
    for seed in range(10):
        rng = np.random.default_rng(1000 + seed)
        E = rng.standard_normal((1000, 16)).astype(np.float32)
        x1 = _rand_set(rng, 200, 1000, 2, 32)
        x2 = _rand_set(rng, 50, 1000, 2, 32)
        got = D.lcrwmd_full(x1, x2, E).values
        ref = O.rwmd_quadratic(x1, x2, E)
        ok, err = rel_close(got, ref, 1e-5, 1e-6)
        assert ok, (seed, err)


@pytest.mark.gpu
def test_acceptance_2_lower_bound_chain():
    """Criterion 2: on >= 1000 random pairs with h <= 4: WCD <= WMD + 1e-4,
    RWMD <= WMD + 1e-4, and each one-sided bound <= the symmetric RWMD exactly."""
    from paper_1711_07227_b200 import emd
    _, D, _ = _pkg()
    rng = np.random.default_rng(2000)
    V = 300
    E = rng.standard_normal((V, 24)).astype(np.float32)
    x1 = _tiny_set(rng, 40, V, 4)
    x2 = _tiny_set(rng, 25, V, 4)
    wcd = D.wcd_block(x1, x2, E).values
    sym = D.lcrwmd_full(x1, x2, E).values
    b1, b2 = D.rwmd_bounds(x1, x2, E)
    assert np.all(b1 <= sym) and np.all(b2 <= sym)
    rows1 = [x1.row(i) for i in range(x1.n_rows)]
    for j in range(x2.n_rows):
        q = x2.row(j)
        w = emd.solve_batch([r.weights for r in rows1], [q.weights] * len(rows1), embeddings=E,
                            ids1=[r.word_ids for r in rows1], ids2=[q.word_ids] * len(rows1))
        assert np.all(wcd[:, j] <= w + 1e-4) and np.all(sym[:, j] <= w + 1e-4), j


def _brute_force_emd(s, d, c):
    """Minimum over the basic feasible solutions (spanning-tree bases of the bipartite graph)."""
    import itertools
    h1, h2 = c.shape
    cells = [(p, q) for p in range(h1) for q in range(h2)]
    best = np.inf
    for basis in itertools.combinations(cells, h1 + h2 - 1):
        A = np.zeros((h1 + h2, len(basis)))
        for k_, (p, q) in enumerate(basis):
            A[p, k_] = 1.0
            A[h1 + q, k_] = 1.0
        b = np.concatenate([s, d])
        sol, res, rank, _ = np.linalg.lstsq(A, b, rcond=None)
        if rank < h1 + h2 - 1 or np.any(sol < -1e-12) or np.abs(A @ sol - b).max() > 1e-9:
            continue
        best = min(best, float(sum(sol[k_] * c[p, q] for k_, (p, q) in enumerate(basis))))
    return best


@pytest.mark.gpu
def test_acceptance_3_emd_vs_basic_feasible_solutions():
    """Criterion 3: 2x2 and random 3x3 instances -- solve_emd equals the brute-force minimum
    over basic feasible solutions within 1e-6 relative; the dual certificate matches."""
    from paper_1711_07227_b200 import emd
    rng = np.random.default_rng(3000)
    for shape in [(2, 2)] * 10 + [(3, 3)] * 10:
        s = rng.random(shape[0]) + 0.05
        d = rng.random(shape[1]) + 0.05
        s /= s.sum()
        d /= d.sum()
        c = np.round(rng.random(shape) * 10, 1)
        plan = emd.solve_emd(emd.TransportProblem(s, d, c))
        ref = _brute_force_emd(s, d, c)
        assert abs(plan.objective - ref) <= 1e-6 * max(1.0, ref), (shape, plan.objective, ref)
        dual = float(s @ plan.dual_source + d @ plan.dual_sink)
        assert abs(dual - plan.objective) <= 1e-6 * max(1.0, ref)


@pytest.mark.gpu
def test_acceptance_4_pruning_exactness():
    """Criterion 4: on 20 random instances (n1 = 300, h <= 8, m = 8, k in {4, 16}) the
    prefiltered top-k equals the exhaustive WMD top-k, with fewer than n1 exact solves in
    at least 18 of them."""
    from paper_1711_07227_b200 import emd
    pruned = 0
    for seed in range(20):
        rng = np.random.default_rng(4000 + seed)
        V = 400
        E = rng.standard_normal((V, 8)).astype(np.float32)
        x1 = _tiny_set(rng, 300, V, 8)
        q = _tiny_set(rng, 1, V, 8).row(0)
        k = 4 if seed % 2 == 0 else 16
        res, solves = emd.prefiltered_topk_wmd(x1, q, E, k)
        rows1 = [x1.row(i) for i in range(300)]
        w = emd.solve_batch([r.weights for r in rows1], [q.weights] * 300, embeddings=E,
                            ids1=[r.word_ids for r in rows1], ids2=[q.word_ids] * 300)
        order = np.lexsort((np.arange(300), w))[:k]
        assert np.array_equal(res.ids, order), seed
        assert np.allclose(res.distances, w[order], rtol=1e-6, atol=0), seed
        pruned += solves < 300
    assert pruned >= 18, pruned


@pytest.mark.gpu
def test_acceptance_6_8_partition_invariance_and_determinism():
    """Criteria 6 and 8: identical top-k for P in {1, 2, 4, 8}; repeated runs are bitwise identical."""
    from paper_1711_07227_b200 import engine
    _, D, _ = _pkg()
    rng = np.random.default_rng(6000)
    V = 1500
    E = rng.standard_normal((V, 32)).astype(np.float32)
    x1 = _rand_set(rng, 203, V, 3, 30)
    x2 = _rand_set(rng, 9, V, 3, 30)
    idx = engine.Index(x1, E, [f"w{i}" for i in range(V)])
    ref = engine.run_query(idx, x2, engine.QueryPlan(k=7))
    for P in (2, 4, 8):
        got = engine.run_query(idx, x2, engine.QueryPlan(k=7, partitions=P))
        assert all(np.array_equal(a.ids, b.ids) and np.array_equal(a.distances, b.distances) for a, b in zip(ref, got))
    a = D.lcrwmd_full(x1, x2, E).values
    b = D.lcrwmd_full(x1, x2, E).values
    assert np.array_equal(a, b)
    t1 = D.lcrwmd_topk(x1, x2, E, 5)
    t2 = D.lcrwmd_topk(x1, x2, E, 5)
    assert all(np.array_equal(u.ids, v.ids) and np.array_equal(u.distances, v.distances) for u, v in zip(t1, t2))


def _clustered_corpus(tmp_path, n=500, topics=5, words_per_topic=60, m=16, seed=7):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((topics, m)) * 2.0
    words, vecs = [], []
    for t in range(topics):
        for w in range(words_per_topic):
            words.append(f"t{t}w{w}")
            vecs.append(centers[t] + rng.standard_normal(m) * 1.5)  # topics overlap: word-level matching matters
    emb = tmp_path / "emb.txt"
    emb.write_text(f"{len(words)} {m}\n" + "".join(
        w + " " + " ".join(f"{x:.6f}" for x in v) + "\n" for w, v in zip(words, vecs)))
    docs, labels = [], []
    for i in range(n):
        t = int(rng.integers(topics))
        h = int(rng.integers(3, 9))
        toks = [f"t{t}w{int(rng.integers(words_per_topic))}" if rng.random() < 0.8
                else f"t{int(rng.integers(topics))}w{int(rng.integers(words_per_topic))}" for _ in range(h)]
        docs.append(" ".join(toks))
        labels.append(f"topic{t}")
    (tmp_path / "docs.txt").write_text("\n".join(docs) + "\n")
    (tmp_path / "labels.txt").write_text("\n".join(labels) + "\n")
    return emb, tmp_path / "docs.txt", tmp_path / "labels.txt"


@pytest.mark.gpu
def test_cli_end_to_end_overlap_precision_determinism(tmp_path):
    """SPEC.md cli + acceptance criteria 7 and 8: index -> query (byte-identical on a rerun),
    overlap(RWMD, WMD) >= overlap(WCD, WMD) at every k on a clustered corpus (n = 500,
    5 clusters), and same-label precision reported per bucket."""
    import json
    from paper_1711_07227_b200 import cli
    emb, docs, labels = _clustered_corpus(tmp_path)
    idx = str(tmp_path / "c.lcrw")
    assert cli.main(["index", "--embeddings", str(emb), "--corpus", str(docs), "--labels", str(labels),
                     "--index", idx, "--out", str(tmp_path / "i.json")]) == 0
    assert json.loads((tmp_path / "i.json").read_text())["n"] == 500
    q = ["query", "--index", idx, "--sample", "20", "--seed", "3", "--k", "5", "--exclude-self"]
    assert cli.main(q + ["--out", str(tmp_path / "q1.jsonl")]) == 0
    assert cli.main(q + ["--out", str(tmp_path / "q2.jsonl")]) == 0
    assert (tmp_path / "q1.jsonl").read_bytes() == (tmp_path / "q2.jsonl").read_bytes()
    recs = [json.loads(l) for l in (tmp_path / "q1.jsonl").read_text().splitlines()]
    assert len(recs) == 20 and all(r["query"] not in r["ids"] and len(r["ids"]) == 5 for r in recs)
    ov = {}
    for method in ("rwmd", "wcd"):
        out = tmp_path / f"ov_{method}.jsonl"
        assert cli.main(["overlap", "--index", idx, "--sample", "20", "--seed", "3", "--method", method,
                         "--reference", "wmd", "--k-pct", "1", "2", "5", "10", "--exclude-self",
                         "--out", str(out)]) == 0
        ov[method] = [json.loads(l)["overlap"] for l in out.read_text().splitlines()]
    assert all(a >= b for a, b in zip(ov["rwmd"], ov["wcd"])), ov
    out = tmp_path / "p.jsonl"
    assert cli.main(["precision", "--index", idx, "--sample", "40", "--seed", "1", "--k", "1", "4", "16",
                     "--out", str(out)]) == 0
    prec = [json.loads(l) for l in out.read_text().splitlines()]
    assert prec and all(0.0 <= r["precision"] <= 1.0 for r in prec)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["uniform", "dup_rows", "long_docs", "m37", "clustered"])
def test_reverse_table_mode_bitwise_equals_gemm_mode(case, monkeypatch):
    """The distance-table reverse Phase 1 (csrc/table.cu) against the GEMM form: the
    symmetric matrix and the top-k are bitwise equal (same Phase-1 entries, exact
    min), over several doc batches, ragged last panels, query vocabularies that are
    not a multiple of the 128-word chunk, docs longer than 32 words and duplicated
    embedding rows (exact zeros); and within tolerance of the oracle."""
    import torch
    from paper_1711_07227_b200 import device
    rng = np.random.default_rng(60 + ["uniform", "dup_rows", "long_docs", "m37", "clustered"].index(case))
    V, m = 3000, (37 if case == "m37" else 300)
    E = rng.standard_normal((V, m)).astype(np.float32)
    if case == "dup_rows":
        E[1500:1700] = E[:200]
    if case == "clustered":  # many near pairs: the table form's refine list vs the GEMM form's scan
        c = rng.standard_normal((60, m)).astype(np.float32)
        E = (c[rng.integers(0, 60, V)] + 0.05 * E).astype(np.float32)
    hi = 150 if case == "long_docs" else 60
    x1 = _rand_set(rng, 1111, V, 1, hi)
    x2 = _rand_set(rng, 45, V, 1, 60)
    prep = device.PreparedEmbeddings(E)
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
    out = {}
    for mode in ("gemm", "table"):
        monkeypatch.setenv("LCRW_REVERSE", mode)
        full = device.symmetric(d1, d2, prep, None, z2_budget_bytes=4 * 3000 * 320)
        td, ti = device.symmetric(d1, d2, prep, 7, z2_budget_bytes=4 * 3000 * 320)
        out[mode] = (full, td, ti)
    if prep.split:  # m <= 64: the GEMM form keeps Z2 in f32; the (forced) table form rounds to 2^-15
        ok, err = rel_close(out["table"][0].cpu().numpy(), out["gemm"][0].cpu().numpy(), 2.0 ** -15, 1e-6)
        assert ok, err
    else:
        for a, b in zip(out["gemm"], out["table"]):
            assert torch.equal(a, b)
    di = np.sort(rng.choice(x1.n_rows, 150, replace=False))
    ref = O.lcrwmd_full(x1.take_rows(di), x2, E, threads=8)
    ok, err = rel_close(out["table"][0].cpu().numpy()[di], ref, RTOL, _atol(E))
    assert ok, err


def _decode_table(T: np.ndarray, V: int, inv_scale: float, a_sq: np.ndarray) -> np.ndarray:
    """16-bit key table (include/lcrwmd.h, common.cuh) -> unscaled f32 distances (chunks, V,
    256): word w of a chunk at byte 2 (w % 256) of the 512-byte row, its key relative to
    2^e <= |w| / 2 < 2^(e+1) (|w|^2 = a_sq[w], scaled): 0 -> 0, 1 -> 2^(e-1), c -> the
    f32 with the bits of 2^e plus c << 9."""
    key = np.ascontiguousarray(T).view("<u2").reshape(-1, V, 256).astype(np.uint32)
    n = key.shape[0] * 256
    sq = np.zeros(n, dtype=np.float32)
    sq[: len(a_sq)] = a_sq
    e2 = (sq.view(np.uint32) >> 23).astype(np.int64) - 127
    base = ((((e2 >> 1) - 1 + 127) << 23).astype(np.uint32)).reshape(-1, 1, 256)
    bits = np.where(key == 1, base - np.uint32(1 << 23), base + (key << 9)).astype(np.uint32)
    return np.where(key == 0, np.float32(0), bits.view(np.float32)) * np.float32(inv_scale)


@pytest.mark.gpu
def test_distance_table_layout_and_zeros():
    """Distance-table layout: chunk w // 256, E row u -> 512-byte row of 16-bit keys of the
    Phase-1 distance of query-vocabulary row w to E row u (relative rounding <= 2^-15),
    exactly 0 for identical rows; the one-pass build (packed stores from the Phase-1
    epilogue) equals the two-pass one (segment panels, lcrw_zero_identical,
    lcrw_table_transpose) bitwise."""
    from paper_1711_07227_b200 import _lib, device
    rng = np.random.default_rng(70)
    V, m = 700, 300
    E = rng.standard_normal((V, m)).astype(np.float32)
    E[600:650] = E[:50]
    x2 = _rand_set(rng, 40, V, 5, 30)
    prep = device.PreparedEmbeddings(E)
    res2 = device.Restricted.build(device.DeviceCSR.upload(x2), prep)
    T = device.distance_table(res2, prep).cpu().numpy()
    T2 = device.distance_table(res2, prep, via_transpose=True).cpu().numpy()
    used = np.unique(x2.column_ids)
    assert res2.v_e == len(used)
    w = np.arange(len(used))
    C = int(_lib.value("lcrw_table_chunk"))
    assert C == 256 and T.size == -(-len(used) // C) * V * 512
    inv = float(prep.scale[1].item())
    a_sq = res2.a_norms.cpu().numpy()
    tab = _decode_table(T, V, inv, a_sq)[w // C, :, w % C]  # (v_e, V)
    assert np.array_equal(tab, _decode_table(T2, V, inv, a_sq)[w // C, :, w % C])  # one-pass == two-pass build
    # the keys are the f32 Phase-1 entries rounded to 14 mantissa bits
    seg = __import__("torch").arange(V + 1, dtype=__import__("torch").int64, device=res2.A.device)
    zf, zp = device.phase1(res2.A, res2.a_norms, res2.v_e, prep.EhB, V, seg, V, prep, z_shift=3)
    zf = zf.cpu().numpy()[: ((V + 7) // 8) * zp].reshape(-1, res2.v_e, 8).transpose(1, 0, 2).reshape(res2.v_e, -1)[:, :V]
    nz = (tab != 0) & (zf != 0)
    assert np.max(np.abs(tab[nz] / zf[nz] - 1)) <= 2.0 ** -15 * 1.001
    ref = O.pairwise_euclidean(E[used], E)
    ok, err = rel_close(tab, ref, RTOL, _atol(E))
    assert ok, err
    same = (E[used][:, None, :] == E[None, :, :]).all(-1)
    assert np.all(tab[same] == 0.0) and same.sum() >= len(used)


@pytest.mark.gpu
@pytest.mark.parametrize("V,n1,n2,hi", [(40, 70, 5, 20), (130, 33, 129, 60), (7, 40, 3, 7)])
def test_reverse_table_mode_tiny_vocabularies(V, n1, n2, hi, monkeypatch):
    """Distance table with vocabularies smaller than one 32-row transpose tile or one
    128-word chunk, query vocabularies of 1..V words, docs holding most of the
    vocabulary: bitwise equal to the GEMM form, within tolerance of the oracle."""
    import torch
    from paper_1711_07227_b200 import device
    rng = np.random.default_rng(80 + V)
    E = rng.standard_normal((V, 300)).astype(np.float32)
    E[V - 1] = E[0]  # an identical pair
    x1 = _rand_set(rng, n1, V, 1, min(hi, V))
    x2 = _rand_set(rng, n2, V, 1, min(hi, V))
    prep = device.PreparedEmbeddings(E)
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
    out = {}
    for mode in ("gemm", "table"):
        monkeypatch.setenv("LCRW_REVERSE", mode)
        out[mode] = device.symmetric(d1, d2, prep, None)
    assert torch.equal(out["gemm"], out["table"])
    ref = O.lcrwmd_full(x1, x2, E, threads=8)
    ok, err = rel_close(out["table"].cpu().numpy(), ref, RTOL, _atol(E))
    assert ok, err


@pytest.mark.gpu
def test_solve_batch_csr_equals_solve_batch():
    """emd.solve_batch_csr (problem arrays gathered from the CSR sets in bulk) solves the
    same problems as solve_batch with per-pair lists: identical objectives."""
    import torch
    from paper_1711_07227_b200 import emd, synthetic as S
    V = 2000
    E = S.embeddings(V, 64, seed=90)
    x1 = S.histograms(300, V, 20, seed=91)
    x2 = S.histograms(7, V, 20, seed=92)
    rng = np.random.default_rng(93)
    docs = rng.integers(0, 300, 500)
    qs = rng.integers(0, 7, 500)
    Et = torch.from_numpy(E).cuda()
    a = emd.solve_batch_csr(x1, docs, x2, qs, Et)
    b = emd.solve_batch([x1.row(int(i)).weights for i in docs], [x2.row(int(j)).weights for j in qs],
                        embeddings=Et, ids1=[x1.row(int(i)).word_ids for i in docs],
                        ids2=[x2.row(int(j)).word_ids for j in qs])
    assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("n_words", [32, 256, 512, 257])
def test_table_chunk_boundaries(n_words, monkeypatch):
    """Query vocabularies of exactly one warp's rows (32 words), one chunk (256), two chunks
    (512: no partial chunk, the tail memset is skipped) and one word past a chunk (257):
    the table form equals the GEMM form bitwise."""
    import torch
    from paper_1711_07227_b200 import device
    from paper_1711_07227_b200.corpus import HistogramSet
    rng = np.random.default_rng(90 + n_words)
    V = 1000
    E = rng.standard_normal((V, 300)).astype(np.float32)
    words = np.sort(rng.choice(V, n_words, replace=False)).astype(np.int32)
    rows = []
    for j in range(0, n_words, 20):  # queries covering exactly these words
        ids = words[j:j + 20]
        u = rng.random(len(ids)) + 0.1
        rows.append((ids, (u / u.sum()).astype(np.float32)))
    x2 = HistogramSet.from_rows(rows, V)
    x1 = _rand_set(rng, 900, V, 5, 60)
    prep = device.PreparedEmbeddings(E)
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
    out = {}
    for mode in ("gemm", "table"):
        monkeypatch.setenv("LCRW_REVERSE", mode)
        out[mode] = device.symmetric(d1, d2, prep, None)
    assert torch.equal(out["gemm"], out["table"])
