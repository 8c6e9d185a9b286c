"""Pin the CPU oracle (oracle/lcrwmd_oracle.py) against the reference's own outputs.

The golden vectors were produced by importing /root/reference (see
tests/golden/make_golden.py); SPEC.md known answers are checked verbatim.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, rel_close
from oracle import lcrwmd_oracle as O

TOL = 1e-6  # dgemm vs broadcast-sum float64 round-off, absorbed by float32 rounding


def test_full_batched_onesided(golden_case):
    name, z, x1, x2 = golden_case
    E = z["E"]
    ok, err = rel_close(O.lcrwmd_full(x1, x2, E), z["full"], rtol=TOL, atol=1e-7)
    assert ok, (name, err)
    ok, err = rel_close(O.lcrwmd_batched(x1, x2, E), z["batched"], rtol=TOL, atol=1e-7)
    assert ok, (name, err)
    q = x2.row(0)
    ok, err = rel_close(O.lcrwmd_one_sided(x1, q.word_ids, q.weights, E), z["one_sided0"], rtol=TOL, atol=1e-7)
    assert ok, (name, err)
    ok, err = rel_close(O.nearest_word_distances(E, E[q.word_ids]), z["nwd0"], rtol=TOL, atol=1e-7)
    assert ok, (name, err)


def test_restrict_spmm_topk(golden_case):
    name, z, x1, x2 = golden_case
    xr, er, remap = O.restrict_vocabulary(O.as_csr(x1), z["E"])
    assert np.array_equal(xr.column_ids, z["r1_ids"])
    assert np.array_equal(er, z["r1_E"])
    assert np.array_equal(remap, z["r1_remap"])
    assert np.array_equal(O.spmm(O.as_csr(x1), z["spmm_z"]), z["spmm"])  # bitwise
    d, i = O.topk_per_query(z["full"], int(z["topk_k"]))
    assert np.array_equal(d, z["topk_d"]) and np.array_equal(i, z["topk_i"])


def test_quadratic_equivalence():
    from conftest import load_case
    z, x1, x2 = load_case("small_m16")
    ok, err = rel_close(O.rwmd_quadratic(x1, x2, z["E"]), z["quadratic"], rtol=1e-5, atol=1e-7)
    assert ok, err
    ok, err = rel_close(z["full"], z["quadratic"], rtol=1e-5, atol=1e-7)
    assert ok, err


def test_threads_bitwise(golden_case):
    name, z, x1, x2 = golden_case
    a = O.lcrwmd_full(x1, x2, z["E"], threads=1)
    b = O.lcrwmd_full(x1, x2, z["E"], threads=4)
    assert np.array_equal(a, b)


def test_topk_golden():
    z = np.load(GOLDEN / "topk.npz")
    for k in (1, 10, 128, 20_000):
        d, i = O.topk_select(z["d"], z["ids"], k)
        assert np.array_equal(d, z[f"d{k}"]) and np.array_equal(i, z[f"i{k}"])
    parts = [O.topk_select(z["d"][a:a + 2500], z["ids"][a:a + 2500], 64) for a in range(0, 10_000, 2500)]
    d, i = O.topk_merge(parts, 64)
    assert np.array_equal(d, z["merge_d"]) and np.array_equal(i, z["merge_i"])


# --- SPEC.md known answers -------------------------------------------------

def _abc():
    E = np.array([[0, 0], [1, 0], [0, 2]], dtype=np.float32)
    x1 = O.CSR(np.array([0, 2]), np.array([0, 1], np.int32), np.array([.5, .5], np.float32), 3)
    x2 = O.CSR(np.array([0, 2]), np.array([1, 2], np.int32), np.array([.5, .5], np.float32), 3)
    return E, x1, x2


def test_spec_abc_instance():
    E, x1, x2 = _abc()
    assert O.lcrwmd_full(x1, x2, E)[0, 0] == pytest.approx(1.0, abs=1e-7)
    assert O.rwmd_quadratic(x1, x2, E)[0, 0] == pytest.approx(1.0, abs=1e-7)


def test_spec_345_and_zero_law():
    z = O.nearest_word_distances(np.array([[0, 0]], np.float32), np.array([[3, 4]], np.float32))
    assert z[0] == 5.0
    E = np.random.default_rng(0).standard_normal((30, 8)).astype(np.float32)
    z = O.nearest_word_distances(E, E[[3, 7]])
    assert z[3] == 0.0 and z[7] == 0.0 and np.all(z >= 0)


def test_spec_spmv_and_topk():
    x = O.CSR(np.array([0, 1]), np.array([2], np.int32), np.array([1.0], np.float32), 4)
    assert O.spmm(x, np.array([[5], [6], [7], [8]], np.float32))[0, 0] == 7.0
    d, i = O.topk_select(np.array([3, 1, 2], np.float32), np.array([0, 1, 2]), 2)
    assert list(d) == [1, 2] and list(i) == [1, 2]
    d, i = O.topk_select(np.array([1.0, 1.0], np.float32), np.array([7, 3]), 1)
    assert list(i) == [3]
    with pytest.raises(ValueError, match="k must be >= 1"):
        O.topk_select(np.zeros(2), np.arange(2), 0)


def test_widen_rows_oracle(widen_case):
    """Oracle restatements of wcd_block, centroids, pairwise_euclidean, rwmd_bounds /
    rwmd_quadratic (distances.py:59-130, kernels.py:113-130, 201-203) vs the reference."""
    name, z, w, x1, x2, _, _ = widen_case
    E = z["E"]
    assert np.array_equal(O.centroids(x1, E), w["c1"])  # bitwise (fp64 SpMM)
    for got, key in ((O.wcd_block(x1, x2, E), "wcd"), (O.pairwise_euclidean(E[:17], E[5:40]), "pair")):
        ok, err = rel_close(got, w[key], rtol=TOL, atol=1e-7)
        assert ok, (name, key, err)
    b1, b2 = O.rwmd_bounds(x1, x2, E)
    for got, key in ((b1, "b1"), (b2, "b2"), (np.maximum(b1, b2), "quadratic")):
        ok, err = rel_close(got, w[key], rtol=TOL, atol=1e-7)
        assert ok, (name, key, err)


def test_emd_oracle():
    """solve_emd restatement (emd.py:120-194) vs the reference objective, incl. 1x1, 1xn, ties."""
    g = np.load(GOLDEN / "emd.npz")
    for i in range(8):
        got = O.solve_emd_objective(g[f"s{i}"], g[f"d{i}"], g[f"c{i}"])
        assert abs(got - float(g[f"obj{i}"])) <= 1e-9 * max(1.0, abs(float(g[f"obj{i}"]))), i


def test_wmd_prefilter_oracle(widen_case):
    """wmd and prefiltered_topk_wmd restatements (emd.py:199-261) vs the reference."""
    name, z, w, _, _, xd1, xd2 = widen_case
    E = z["E"]
    for i, ref in enumerate(w["wmd0"]):
        q, r = xd2.row(0), xd1.row(i)
        got = O.wmd(r.word_ids, r.weights, q.word_ids, q.weights, E)
        assert abs(got - ref) <= 1e-6 * max(1.0, ref), (name, i, got, ref)
    q = xd2.row(0)
    d, ids, solves = O.prefiltered_topk_wmd(xd1, q.word_ids, q.weights, E, 4)
    assert np.array_equal(ids, w["pf0_i"]), name
    assert np.allclose(d, w["pf0_d"], rtol=1e-6, atol=1e-9), name


def test_prims_restatement_bitwise():
    """The restated numpy arithmetic csrc/prims.cu implements (pairwise sums, sequential
    np.minimum) reproduces the reference's squared_norms / euclidean_into / minima bit for
    bit, and the oracle's top-k keeps the caller's dtype (tests/golden/prims.npz)."""
    z = np.load(GOLDEN / "prims.npz")
    assert np.array_equal(O.squared_norms_pairwise(z["sn_a32"]), z["sn_r32"])
    assert np.array_equal(O.squared_norms_pairwise(z["sn_a64"]), z["sn_r64"])
    for i in range(4):
        a, b = z[f"eu{i}_a"], z[f"eu{i}_b"]
        e = O.euclidean_pairwise(a, O.squared_norms_pairwise(a), b, O.squared_norms_pairwise(b))
        assert np.array_equal(e, z[f"eu{i}_o64"]), i
        assert np.array_equal(e.astype(np.float32), z[f"eu{i}_o32"]), i
    for nm in ("f", "i", "d"):
        v = z[f"mn_{nm}"]
        np.testing.assert_array_equal(O.segmented_min_seq(v, [0, v.shape[1]], axis=1)[:, 0], z[f"rmin_{nm}"])
        np.testing.assert_array_equal(O.segmented_min_seq(v, [0, v.shape[0]], axis=0)[0], z[f"cmin_{nm}"])
    np.testing.assert_array_equal(O.segmented_min_seq(z["mn_f"], z["seg0"], 0), z["smin_f0"])
    np.testing.assert_array_equal(O.segmented_min_seq(z["mn_f"], z["seg1"], 1), z["smin_f1"])
    np.testing.assert_array_equal(O.segmented_min_seq(z["mn_d"], [0, 10, 11, 40], 1), z["smin_d1"])
    np.testing.assert_array_equal(O.segmented_min_seq(z["smin_v"], z["smin_v_seg"], 0), z["smin_v_out"])
    for k in (1, 10, 700, 5000):
        for nm in ("d64", "dint", "d16"):
            d, i = O.topk_select(z[f"tk_{nm}"], z["tk_ids"], k)
            assert d.dtype == z[f"tk_{nm}"].dtype
            assert np.array_equal(d, z[f"tk_{nm}_{k}_d"]) and np.array_equal(i, z[f"tk_{nm}_{k}_i"]), (nm, k)
    d, i = O.topk_select(np.array([1.0, 1.0 + 1e-12]), np.array([7, 3]), 1)
    assert np.array_equal(i, z["tk_verdict_i"]) and i[0] == 7
