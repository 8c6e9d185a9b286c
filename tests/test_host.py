"""CPU-only tests: host data model, ingestion, layout helpers, and that the C-ABI
library loads and exports every symbol include/lcrwmd.h declares."""

from __future__ import annotations

import ctypes
import re
import struct

import numpy as np
import pytest

from conftest import ROOT
from paper_1711_07227_b200 import corpus as C
from paper_1711_07227_b200 import synthetic as S


def test_header_symbols_exported_and_bound():
    from paper_1711_07227_b200 import _build, _lib
    _build.build()
    header = (ROOT / "include" / "lcrwmd.h").read_text()
    declared = set(re.findall(r"\b(lcrw_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    # pure host entry points work without a GPU
    assert _lib.value("lcrw_abi_version") == 1
    assert _lib.value("lcrw_padded_dim", 300) == 320
    assert _lib.value("lcrw_padded_dim", 37) == 64
    assert _lib.value("lcrw_operand_k", 300, 0) == 303 and _lib.value("lcrw_operand_k", 16, 1) == 51
    assert _lib.value("lcrw_plan_ranges", 1000, 256) == 4
    assert _lib.value("lcrw_status_string", 1) == b"invalid argument"


def test_library_rejects_bad_arguments_without_gpu():
    from paper_1711_07227_b200 import _lib
    with pytest.raises(ValueError, match="k must be >= 1"):
        _lib.call("lcrw_topk_segments", None, None, 1, 1, 0, None, None, None)
    with pytest.raises(ValueError, match="kp must be"):
        _lib.call("lcrw_phase1", None, None, 0, None, 0, 300, 300, None, 0, 1, None, None, 1, None, None, 0,
                  3, None)


def test_histogram_set_basics():
    x = S.histograms(50, 200, 10, seed=0)
    x.validate()
    assert x.n_rows == 50 and x.nnz == len(x.column_ids)
    sub = x.take_rows([3, 1, 3])
    assert np.array_equal(sub.row(0).word_ids, x.row(3).word_ids)
    assert np.array_equal(sub.row(1).weights, x.row(1).weights)
    s = x.slice_rows(10, 20)
    assert s.n_rows == 10 and np.array_equal(s.row(0).word_ids, x.row(10).word_ids)
    fr = C.HistogramSet.from_rows([(x.row(i).word_ids, x.row(i).weights) for i in range(5)], 200)
    assert np.array_equal(fr.column_ids, x.slice_rows(0, 5).column_ids)


def test_validate_errors():
    good = C.HistogramSet(np.array([0, 2]), np.array([1, 3], np.int32), np.array([.5, .5], np.float32), 5)
    good.validate()
    with pytest.raises(C.CorpusError, match="at least one word"):
        C.HistogramSet(np.array([0, 0]), np.zeros(0, np.int32), np.zeros(0, np.float32), 5).validate()
    with pytest.raises(C.CorpusError, match="strictly increasing"):
        C.HistogramSet(np.array([0, 2]), np.array([3, 1], np.int32), np.array([.5, .5], np.float32), 5).validate()
    with pytest.raises(C.CorpusError, match="weights sum"):
        C.HistogramSet(np.array([0, 2]), np.array([1, 3], np.int32), np.array([.5, .6], np.float32), 5).validate()
    with pytest.raises(C.CorpusError, match="out of range"):
        C.HistogramSet(np.array([0, 1]), np.array([7], np.int32), np.array([1.0], np.float32), 5).validate()


def test_synthetic_shapes():
    x = S.histograms(2000, 1000, 40, seed=1)
    x.validate()
    sizes = x.row_sizes
    assert 15 <= sizes.mean() <= 45 and sizes.min() >= 1
    E = S.embeddings(100, 8, seed=0)
    assert E.dtype == np.float32 and E.shape == (100, 8)


def test_build_histograms_spec_examples():
    vocab = C.Vocabulary.from_words(["cat", "dog", "the"])
    hs, kept = C.build_histograms([["cat", "cat", "dog"]], vocab)
    assert list(hs.row(0).word_ids) == [0, 1]
    assert np.allclose(hs.row(0).weights, [2 / 3, 1 / 3])
    with pytest.raises(C.IngestError) as ei:
        C.build_histograms([["cat"], ["the", "the"]], vocab, stopwords={"the"})
    assert ei.value.doc_index == 1
    hs, kept = C.build_histograms([["cat"], ["the"]], vocab, stopwords={"the"}, on_empty="skip")
    assert list(kept) == [0]


def test_load_embeddings_text_and_binary(tmp_path):
    t = tmp_path / "e.txt"
    t.write_text("3 2\na 0 0\nb 1.5 -2\na 9 9\n")
    vocab, E = C.load_embeddings(t, "text")
    assert vocab.words == ["a", "b"] and E.shape == (2, 2) and E[0, 0] == 0 and E[1, 1] == -2
    b = tmp_path / "e.bin"
    with b.open("wb") as fh:
        fh.write(b"2 3\n")
        fh.write(b"x " + struct.pack("<3f", 1, 2, 3) + b"\n")
        fh.write(b"y " + struct.pack("<3f", 4, 5, 6))
    vocab, E = C.load_embeddings(b, "binary")
    assert vocab.words == ["x", "y"] and np.array_equal(E[1], [4, 5, 6])
    bad = tmp_path / "bad.txt"
    bad.write_text("2 2\na 1\n")
    with pytest.raises(C.EmbeddingLoadError, match=r":2: expected 2 values"):
        C.load_embeddings(bad)
    with pytest.raises(ValueError, match="unknown embedding format"):
        C.load_embeddings(bad, "xml")


def test_z_panel_layout():
    from paper_1711_07227_b200.kernels import _z_panels
    z = np.arange(5 * 11, dtype=np.float32).reshape(5, 11)
    flat, zp = _z_panels(z)
    assert zp == 40
    for s in range(11):
        for r in range(5):
            assert flat[(s >> 3) * zp + r * 8 + (s & 7)] == z[r, s]


def test_no_oracle_import_in_product():
    """The product package must never import the test oracle."""
    for p in (ROOT / "paper_1711_07227_b200").rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", p.read_text(), re.M), p


@pytest.mark.parametrize("n_q,h,V", [(1000, 50, 100_000), (70, 300, 2000), (2100, 20, 5000), (3, 1, 10)])
def test_reverse_entry_plan_invariants(n_q, h, V):
    """lcrw_reverse_panels plan (include/lcrwmd.h): 16-byte aligned blocks per (group,
    tile), W cumulative list ends, every nonzero exactly once in its (group, tile,
    warp) list, lists a multiple of I long, each aligned group of I names distinct
    queries, padding = the list's scratch query G + warp with weight 0."""
    from paper_1711_07227_b200.device import plan_query_entries
    T, G, W, I = 128, 1024, 16, 4
    x = S.histograms(n_q, V, h, seed=7)
    offs, cols, vals = np.asarray(x.row_offsets), np.asarray(x.column_ids), np.asarray(x.values)
    used = np.unique(cols)
    rank = np.full(V, -1, np.int32)
    rank[used] = np.arange(len(used))
    words, tile_off = plan_query_entries(offs, cols, vals, rank, len(used), T, G, W, I)
    n_tiles = (len(used) + T - 1) // T
    n_groups = (n_q + G - 1) // G
    assert tile_off.shape == (n_groups * n_tiles + 1,) and tile_off[0] == 0 and tile_off[-1] == words.size
    assert np.all(tile_off % 4 == 0)
    seen = []
    for B in range(n_groups * n_tiles):
        g, t = divmod(B, n_tiles)
        blk = words[tile_off[B]:tile_off[B + 1]]
        ends = blk[:W].astype(np.int64)
        assert np.all(np.diff(np.concatenate([[0], ends])) % I == 0)
        assert W + 2 * ends[-1] <= blk.size < W + 2 * ends[-1] + 4
        ent = blk[W:W + 2 * ends[-1]].reshape(-1, 2)
        for w in range(W):
            lo = ends[w - 1] if w else 0
            last_row = {}  # each query's terms in ascending row order (batching-invariant fp32 sums)
            for e in range(lo, ends[w]):
                qv = int((ent[e, 0] & 0x3FFFF) >> 7)
                if qv < G:
                    rv = int(ent[e, 0] >> 25)
                    assert rv > last_row.get(qv, -1), (B, w, qv)
                    last_row[qv] = rv
            for b in range(lo, ends[w], I):
                qs = ((ent[b:b + I, 0] & 0x3FFFF) >> 7).astype(np.int64)
                real = qs < G
                assert np.all(qs[~real] == G + w)  # the warp's own scratch row
                assert len(set(qs[real].tolist())) == int(real.sum())
                assert np.all(ent[b:b + I, 1][~real] == 0)
                for e in range(b, b + I):
                    if not real[e - b]:
                        continue
                    assert ent[e, 0] & 0x7F == 0 and (ent[e, 0] >> 18) & 0x7F == 0
                    ql, rl = int((ent[e, 0] & 0x3FFFF) >> 7), int(ent[e, 0] >> 25)
                    assert ql % W == w and rl < T
                    seen.append((g * G + ql, t * T + rl, float(ent[e, 1:2].view(np.float32)[0])))
    q = np.repeat(np.arange(n_q), np.diff(offs))
    want = sorted(zip(q.tolist(), rank[cols].tolist(), vals.astype(np.float32).tolist()))
    assert sorted(seen) == want


@pytest.mark.parametrize("name", ["small_m16", "m300", "clustered", "dup_rows"])
def test_index_file_matches_reference_bytes(name, tmp_path):
    """LCRW v1 (corpus.py:17-25, 433-489): reading the reference-written file and writing
    it back reproduces the reference's bytes exactly (tests/golden/widen_*.npz)."""
    g = np.load(ROOT / "tests" / "golden" / f"widen_{name}.npz")
    ref = g["index_bytes"].tobytes()
    f = tmp_path / "ref.lcrw"
    f.write_bytes(ref)
    hs, E, words = C.read_index_file(f)
    assert hs.row_offsets.dtype == np.int64 and hs.column_ids.dtype == np.int32 and E.dtype == np.float32
    assert hs.n_cols == E.shape[0] == len(words) and words[0] == "w0_é"
    C.write_index_file(tmp_path / "ours.lcrw", hs, E, words)
    assert (tmp_path / "ours.lcrw").read_bytes() == ref


def test_index_file_errors(tmp_path):
    hs = C.HistogramSet.from_rows([(np.array([0, 2], np.int32), np.array([0.5, 0.5], np.float32))], 3)
    E = np.arange(6, dtype=np.float32).reshape(3, 2)
    with pytest.raises(C.CorpusError, match="inconsistent index"):
        C.write_index_file(tmp_path / "x", hs, E, ["a", "b"])
    C.write_index_file(tmp_path / "x", hs, E, ["a", "b", "c"])
    raw = (tmp_path / "x").read_bytes()
    (tmp_path / "m").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(C.CorpusError, match="bad magic"):
        C.read_index_file(tmp_path / "m")
    (tmp_path / "v").write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(C.CorpusError, match="unsupported format version 2"):
        C.read_index_file(tmp_path / "v")
    (tmp_path / "t").write_bytes(raw[:60])
    with pytest.raises(C.CorpusError, match="truncated"):
        C.read_index_file(tmp_path / "t")
    hs2, E2, w2 = C.read_index_file(tmp_path / "x")
    assert np.array_equal(hs2.column_ids, hs.column_ids) and np.array_equal(E2, E) and w2 == ["a", "b", "c"]


def test_read_corpus_and_labels(tmp_path):
    """corpus.py:196-237: plain text (line-number ids, blank lines skipped), JSONL, errors."""
    (tmp_path / "p.txt").write_text("Hello, World!\n\n  the CAT sat.  \n")
    ids, docs = C.read_corpus(tmp_path / "p.txt")
    assert ids == ["0", "2"] and docs == [["hello", "world"], ["the", "cat", "sat"]]
    (tmp_path / "j.jsonl").write_text('{"id": "a", "text": "x y"}\n{"text": "Z"}\n')
    ids, docs = C.read_corpus(tmp_path / "j.jsonl")
    assert ids == ["a", "1"] and docs == [["x", "y"], ["z"]]
    (tmp_path / "b.jsonl").write_text('{"id": "a", "text": "x"}\n{"id": "b"}\n')
    with pytest.raises(C.CorpusError, match=r"b.jsonl:2: bad JSONL record"):
        C.read_corpus(tmp_path / "b.jsonl")
    (tmp_path / "l.txt").write_text("pos\n\nneg \n")
    assert C.read_labels(tmp_path / "l.txt") == ["pos", "neg"]


def test_query_plan_validation():
    from paper_1711_07227_b200.engine import QueryPlan
    QueryPlan().validate()
    with pytest.raises(ValueError, match="unknown method"):
        QueryPlan(method="bm25").validate()
    with pytest.raises(ValueError, match="k must be >= 1"):
        QueryPlan(k=0).validate()
    with pytest.raises(ValueError, match="partitions must be >= 1"):
        QueryPlan(partitions=0).validate()


def test_cli_usage_and_errors(tmp_path, capsys):
    """SPEC.md cli: bad flags exit 2, runtime errors exit 1 with a diagnostic."""
    from paper_1711_07227_b200 import cli
    with pytest.raises(SystemExit) as e:
        cli.main(["query", "--method", "bm25", "--index", "x"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main([])
    assert e.value.code == 2
    assert cli.main(["query", "--index", str(tmp_path / "missing.lcrw")]) == 1
    assert "error:" in capsys.readouterr().err


def test_product_has_no_cpu_fallback():
    """Without a CUDA device every compute entry point raises instead of computing on the
    host; a missing library is reported, not worked around."""
    import subprocess
    import sys
    import torch
    from paper_1711_07227_b200 import distances, kernels
    if torch.cuda.is_available():
        pytest.skip("needs a host without a GPU")
    E = S.embeddings(40, 8, seed=0)
    x = S.histograms(5, 40, 4, seed=1)
    for call in (lambda: distances.lcrwmd_full(x, x, E), lambda: distances.lcrwmd_topk(x, x, E, 2),
                 lambda: kernels.topk_select(np.ones(4, np.float32), np.arange(4), 2)):
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            call()
    code = ("import os; os.environ['LCRW_LIB'] = '/nonexistent/liblcrwmd.so'\n"
            "from paper_1711_07227_b200 import _lib\n"
            "try:\n    _lib.load()\nexcept RuntimeError as e:\n    print('raised', e)\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.stdout.startswith("raised"), out.stdout + out.stderr


def test_reverse_mode_choice(monkeypatch):
    """Distance table only when nnz(X1) >> V, a 128-word chunk fits L2 and the table fits
    a quarter of HBM (include/lcrwmd.h); LCRW_REVERSE overrides."""
    from paper_1711_07227_b200 import device
    monkeypatch.delenv("LCRW_REVERSE", raising=False)
    hbm = 180 << 30
    assert device.reverse_mode(100_000, 39_300, 50_000_000, hbm) == "table"      # C2
    assert device.reverse_mode(3_000_000, 146_000, 75_000_000, hbm) == "gemm"    # C4: chunk >> L2
    assert device.reverse_mode(400_000, 190_000, 1_250_000, hbm) == "gemm"      # C5 shard
    assert device.reverse_mode(20_000, 2_400, 30_000, hbm) == "gemm"            # few docs: 2V > nnz
    assert device.reverse_mode(100_000, 39_300, 50_000_000, 24 << 30) == "gemm"  # table > HBM / 4
    monkeypatch.setenv("LCRW_REVERSE", "gemm")
    assert device.reverse_mode(100_000, 39_300, 50_000_000, hbm) == "gemm"
    monkeypatch.setenv("LCRW_REVERSE", "table")
    assert device.reverse_mode(3_000_000, 146_000, 75_000_000, hbm) == "table"


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the driver's reference arm: the pinned CPU oracle on the
    host cores, bounded samples extrapolated part by part) prints one JSON line with the
    contract keys and the same config object as our arm."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "3", "--ref-docs", "64", "--ref-rows", "256"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "impl", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["n_docs"] == 2000 and line["config"]["n_queries"] == 64


@pytest.mark.parametrize("n_q,h,V", [(1000, 50, 100_000), (70, 300, 2000), (2100, 20, 5000), (3, 1, 10)])
def test_native_plan_equals_numpy_plan(n_q, h, V):
    """lcrw_plan_reverse (csrc/plan.cu, host code in the library) builds exactly the words
    and block offsets of the numpy restatement plan_query_entries."""
    from paper_1711_07227_b200.device import plan_query_entries, plan_query_entries_native
    x = S.histograms(n_q, V, h, seed=9)
    offs, cols, vals = np.asarray(x.row_offsets), np.asarray(x.column_ids), np.asarray(x.values)
    used = np.unique(cols)
    rank = np.full(V, -1, np.int32)
    rank[used] = np.arange(len(used))
    w1, t1 = plan_query_entries(offs, cols, vals, rank, len(used), 128, 1024, 16, 4)
    w2, t2 = plan_query_entries_native(offs, cols, vals, rank, len(used), 128, 1024, 16, 4)
    assert np.array_equal(w1, w2) and np.array_equal(t1, t2)
