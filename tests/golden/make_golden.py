"""Generate golden vectors by running the REAL reference (movers) on seeded inputs.

Run in the build container only (it needs /root/reference):

    python tests/golden/make_golden.py

Each case is written as tests/golden/<name>.npz holding the inputs and the
reference's outputs, so the GPU box (where /root/reference does not exist)
can check both the oracle restatement and the CUDA path against them.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    from movers import corpus, distances, kernels  # noqa: E402
    return corpus, distances, kernels


def _rand_set(corpus, rng, n, vocab, hlo, hhi):
    rows = []
    for _ in range(n):
        h = int(rng.integers(hlo, hhi + 1))
        ids = np.sort(rng.choice(vocab, size=min(h, vocab), replace=False)).astype(np.int32)
        u = rng.random(len(ids)) + 0.1
        rows.append((ids, (u / u.sum()).astype(np.float32)))
    return corpus.HistogramSet.from_rows(rows, vocab)


def _pack(prefix, hs):
    return {f"{prefix}_offsets": hs.row_offsets, f"{prefix}_ids": hs.column_ids,
            f"{prefix}_vals": hs.values, f"{prefix}_ncols": np.int64(hs.n_cols)}


def case_lcrwmd(name, seed, n1, n2, vocab, m, hlo, hhi, clustered=False, dup_rows=0,
                queries_from_docs=False, quadratic=False):
    corpus, distances, kernels = _ref()
    rng = np.random.default_rng(seed)
    if clustered:
        cen = rng.standard_normal((max(2, vocab // 25), m)).astype(np.float32)
        lab = rng.integers(0, len(cen), vocab)
        E = (cen[lab] + 0.05 * rng.standard_normal((vocab, m))).astype(np.float32)
    else:
        E = rng.standard_normal((vocab, m)).astype(np.float32)
    if dup_rows:  # identical vectors under different ids: reference gives exact 0
        src = rng.choice(vocab, dup_rows, replace=False)
        dst = rng.choice(np.setdiff1d(np.arange(vocab), src), dup_rows, replace=False)
        E[dst] = E[src]
    x1 = _rand_set(corpus, rng, n1, vocab, hlo, hhi)
    if queries_from_docs:
        x2 = x1.take_rows(np.sort(rng.choice(n1, n2, replace=False)))
    else:
        x2 = _rand_set(corpus, rng, n2, vocab, hlo, hhi)
    out = {"E": E, **_pack("x1", x1), **_pack("x2", x2)}
    out["full"] = distances.lcrwmd_full(x1, x2, E).values
    out["batched"] = distances.lcrwmd_batched(x1, x2, E)
    out["one_sided0"] = distances.lcrwmd_one_sided(x1, x2.row(0), E)
    q0 = x2.row(0)
    out["nwd0"] = distances.nearest_word_distances(E, E[q0.word_ids])
    x1r, e1, remap1 = corpus.restrict_vocabulary(x1, E)
    out["r1_ids"], out["r1_E"], out["r1_remap"] = x1r.column_ids, e1, remap1
    z = rng.random((x1.n_cols, 5)).astype(np.float32)
    out["spmm_z"], out["spmm"] = z, kernels.spmm(x1, z)
    if quadratic:
        out["quadratic"] = distances.rwmd_quadratic(x1, x2, E).values
    k = 5
    ids = np.arange(n1, dtype=np.int64)
    tk_d = np.zeros((n2, min(k, n1)), np.float32)
    tk_i = np.zeros((n2, min(k, n1)), np.int64)
    for j in range(n2):
        r = kernels.topk_select(out["full"][:, j], ids, k)
        tk_d[j], tk_i[j] = r.distances, r.ids
    out["topk_k"], out["topk_d"], out["topk_i"] = np.int64(k), tk_d, tk_i
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, {k_: v.shape for k_, v in out.items() if hasattr(v, "shape")})


def case_topk():
    _, _, kernels = _ref()
    rng = np.random.default_rng(7)
    d = rng.integers(0, 50, 10_000).astype(np.float32) / 7.0  # many exact ties
    ids = rng.permutation(10_000).astype(np.int64) * 3 + 11
    out = {"d": d, "ids": ids}
    for k in (1, 10, 128, 20_000):
        r = kernels.topk_select(d, ids, k)
        out[f"d{k}"], out[f"i{k}"] = r.distances, r.ids
    parts = [kernels.topk_select(d[a:a + 2500], ids[a:a + 2500], 64) for a in range(0, 10_000, 2500)]
    mr = kernels.topk_merge(parts, 64)
    out["merge_d"], out["merge_i"] = mr.distances, mr.ids
    np.savez_compressed(OUT / "topk.npz", **out)
    print("topk")


def case_widen(name):
    """Reference outputs for the rows next to the hot path: WCD, both
    one-sided RWMD bounds, centroids, pairwise distances, exact WMD and the
    RWMD-prefiltered exact top-k, and the LCRW index file bytes."""
    import tempfile
    corpus, distances, kernels = _ref()
    from movers import emd
    z = np.load(OUT / f"{name}.npz")

    def hs(p_):
        return corpus.HistogramSet(z[f"{p_}_offsets"], z[f"{p_}_ids"], z[f"{p_}_vals"], int(z[f"{p_}_ncols"]))

    E, x1, x2 = z["E"], hs("x1"), hs("x2")
    out = {}
    out["wcd"] = distances.wcd_block(x1, x2, E).values
    out["c1"] = kernels.centroids(x1, E)
    out["pair"] = kernels.pairwise_euclidean(E[:17], E[5:40]).values
    b1, b2 = distances.rwmd_bounds(x1, x2, E)
    out["b1"], out["b2"] = b1, b2
    out["quadratic"] = distances.rwmd_quadratic(x1, x2, E).values
    # exact WMD / prefiltered top-k on dyadic-weight copies of the sets: the reference
    # solver (emd.py:153-162) raises when float32-normalised supply and demand totals
    # differ by more than 1e-9, which happens for about half of general histograms
    def dyadic(hs_, seed):
        r = np.random.default_rng(seed)
        rows = []
        for i in range(hs_.n_rows):
            q = hs_.row(i)
            c = r.integers(1, 9, len(q.word_ids)).astype(np.int64)
            c[0] += (-int(c.sum())) % 64          # total = multiple of 64 ...
            tot = int(c.sum())
            scale = 1 << int(np.ceil(np.log2(tot)))
            c[0] += scale - tot                   # ... = a power of two: weights exact in f32
            rows.append((q.word_ids, (c / scale).astype(np.float32)))
        return corpus.HistogramSet.from_rows(rows, hs_.n_cols)
    xd1, xd2 = dyadic(x1, 1), dyadic(x2, 2)
    out.update(_pack("xd1", xd1))
    out.update(_pack("xd2", xd2))
    n_w = min(6, xd1.n_rows)
    out["wmd0"] = np.array([emd.wmd(xd1.row(i), xd2.row(0), E) for i in range(n_w)])
    k = 4
    for j in range(min(2, xd2.n_rows)):
        r, solves = emd.prefiltered_topk_wmd(xd1, xd2.row(j), E, k)
        out[f"pf{j}_d"], out[f"pf{j}_i"], out[f"pf{j}_solves"] = r.distances, r.ids, np.int64(solves)
    x1r, e1, _ = corpus.restrict_vocabulary(x1, E)
    words = [f"w{i}_\u00e9" for i in range(e1.shape[0])]
    with tempfile.TemporaryDirectory() as td:
        f = Path(td) / "x.lcrw"
        corpus.write_index_file(f, x1r, e1, words)
        out["index_bytes"] = np.frombuffer(f.read_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / f"widen_{name}.npz", **out)
    print("widen", name, {k_: v.shape for k_, v in out.items() if hasattr(v, "shape")})


def case_emd():
    """solve_emd on small transport problems, including degenerate ones."""
    from movers import emd
    _ref()
    rng = np.random.default_rng(21)
    out = {}
    shapes = [(1, 1), (1, 5), (5, 1), (3, 3), (7, 4), (12, 12), (30, 25), (60, 45)]
    for i, (h1, h2) in enumerate(shapes):
        s_ = rng.random(h1) + 0.05
        d_ = rng.random(h2) + 0.05
        s_ /= s_.sum()
        d_ /= d_.sum()
        c = rng.random((h1, h2)) * 10
        if i == 3:
            c = np.round(c)  # ties
        plan = emd.solve_emd(emd.TransportProblem(s_, d_, c))
        out[f"s{i}"], out[f"d{i}"], out[f"c{i}"] = s_, d_, c
        out[f"obj{i}"] = np.float64(plan.objective)
    np.savez_compressed(OUT / "emd.npz", **out)
    print("emd", len(shapes))


def case_prims():
    """The remaining public primitives of movers.kernels (kernels.py:66-167, 210-232):
    squared_norms, euclidean_into (f32 and f64 out, m below and above numpy's 128-element
    pairwise block, duplicate rows), row_min / col_min / segmented_min (NaN, ints,
    both axes), and topk_select / topk_merge on non-f32 dtypes (f64 near-ties, exact
    ties, integers, f16)."""
    _, _, kernels = _ref()
    rng = np.random.default_rng(31)
    out = {}
    a32 = rng.standard_normal((20, 300)).astype(np.float32)
    a64 = rng.standard_normal((15, 1000))
    out["sn_a32"], out["sn_a64"] = a32, a64
    out["sn_r32"], out["sn_r64"] = kernels.squared_norms(a32), kernels.squared_norms(a64)
    for i, (r, c, m) in enumerate(((37, 29, 300), (9, 11, 700), (5, 6, 1), (8, 8, 129))):
        a = rng.standard_normal((r, m))
        b = rng.standard_normal((c, m))
        b[: min(3, c)] = a[: min(3, c)]  # identical rows: exactly 0
        o32 = np.empty((r, c), np.float32)
        o64 = np.empty((r, c), np.float64)
        kernels.euclidean_into(a, kernels.squared_norms(a), b, kernels.squared_norms(b), o32, 7, 5)
        kernels.euclidean_into(a, kernels.squared_norms(a), b, kernels.squared_norms(b), o64)
        out[f"eu{i}_a"], out[f"eu{i}_b"], out[f"eu{i}_o32"], out[f"eu{i}_o64"] = a, b, o32, o64
    mf = rng.standard_normal((13, 17)).astype(np.float32)
    mf[3, 5] = np.nan
    mf[7, :] = -0.0
    mi = rng.integers(-1000, 1000, (9, 21)).astype(np.int32)
    md = rng.standard_normal((6, 40))
    out["mn_f"], out["mn_i"], out["mn_d"] = mf, mi, md
    for nm, v in (("f", mf), ("i", mi), ("d", md)):
        out[f"rmin_{nm}"], out[f"cmin_{nm}"] = kernels.row_min(v), kernels.col_min(v)
    seg0 = np.array([0, 2, 3, 9, 13])
    seg1 = np.array([0, 1, 5, 6, 17])
    out["seg0"], out["seg1"] = seg0, seg1
    out["smin_f0"] = kernels.segmented_min(mf, seg0, axis=0)
    out["smin_f1"] = kernels.segmented_min(mf, seg1, axis=1)
    out["smin_d1"] = kernels.segmented_min(md, np.array([0, 10, 11, 40]), axis=-1)
    v1 = rng.standard_normal(50)
    out["smin_v"], out["smin_v_seg"] = v1, np.array([0, 7, 8, 30, 50])
    out["smin_v_out"] = kernels.segmented_min(v1, out["smin_v_seg"])
    # top-k on the caller's dtype
    n = 3000
    base = rng.integers(0, 40, n).astype(np.float64) / 3.0
    d64 = base + rng.integers(0, 3, n) * 1e-12  # near-ties a float32 cast would merge
    ids = rng.permutation(n).astype(np.int64) * 5 + 2
    dint = rng.integers(-20, 20, n).astype(np.int64)
    d16 = (rng.integers(0, 100, n) / 8).astype(np.float16)
    out["tk_d64"], out["tk_ids"], out["tk_dint"], out["tk_d16"] = d64, ids, dint, d16
    for k in (1, 10, 700, 5000):
        for nm, d in (("d64", d64), ("dint", dint), ("d16", d16)):
            r = kernels.topk_select(d, ids, k)
            out[f"tk_{nm}_{k}_d"], out[f"tk_{nm}_{k}_i"] = r.distances, r.ids
    r = kernels.topk_select(np.array([1.0, 1.0 + 1e-12]), np.array([7, 3]), 1)
    out["tk_verdict_d"], out["tk_verdict_i"] = r.distances, r.ids
    parts = [kernels.topk_select(d64[a:a + 700], ids[a:a + 700], 50) for a in range(0, n, 700)]
    mr = kernels.topk_merge(parts, 50)
    out["tk_merge_d"], out["tk_merge_i"] = mr.distances, mr.ids
    np.savez_compressed(OUT / "prims.npz", **out)
    print("prims", len(out))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "prims":
    case_prims()
elif __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "widen":
    for nm in ("small_m16", "m300", "clustered", "dup_rows"):
        case_widen(nm)
    case_emd()
elif __name__ == "__main__":
    case_lcrwmd("small_m16", seed=11, n1=60, n2=12, vocab=400, m=16, hlo=1, hhi=20, quadratic=True)
    case_lcrwmd("m300", seed=12, n1=48, n2=8, vocab=500, m=300, hlo=20, hhi=60)
    case_lcrwmd("clustered", seed=13, n1=40, n2=8, vocab=500, m=64, hlo=5, hhi=30, clustered=True)
    case_lcrwmd("self_queries", seed=14, n1=50, n2=10, vocab=300, m=32, hlo=2, hhi=25,
                queries_from_docs=True)
    case_lcrwmd("dup_rows", seed=15, n1=40, n2=10, vocab=200, m=24, hlo=3, hhi=20, dup_rows=12)
    case_lcrwmd("ragged_m37", seed=16, n1=70, n2=9, vocab=350, m=37, hlo=1, hhi=90)
    case_topk()
