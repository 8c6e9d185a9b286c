"""Command-line surface (SPEC.md ``cli`` module): index, query, bench, overlap, precision.

    python -m paper_1711_07227_b200.cli index --embeddings E.txt --corpus docs.txt --index out.lcrw
    python -m paper_1711_07227_b200.cli query --index out.lcrw --sample 100 --method lc-rwmd --k 10
    python -m paper_1711_07227_b200.cli overlap --index out.lcrw --sample 50 --method rwmd --k-pct 1 2 5
    python -m paper_1711_07227_b200.cli precision --index out.lcrw --sample 50 --method lc-rwmd --k 1 4 16
    python -m paper_1711_07227_b200.cli bench --index out.lcrw --sample 64 --methods lc-rwmd wcd --partitions 1 2

All outputs are UTF-8 JSON lines (stdout or --out).  Bad flags exit 2 (usage),
runtime errors exit 1 with a diagnostic.  Transient queries are either a corpus
file (--corpus, tokenised over the index vocabulary) or a seeded random sample
of the resident set (--sample N --seed S, as the paper's evaluation does); the
sampled queries carry their resident ids so --exclude-self works.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from contextlib import contextmanager

import numpy as np

from . import corpus, engine


@contextmanager
def _out(path):
    if path:
        with open(path, "w", encoding="utf-8") as fh:
            yield fh
    else:
        yield sys.stdout


def _queries(args, index: engine.Index):
    """(query set, resident ids or None)."""
    if args.corpus:
        _, docs = corpus.read_corpus(args.corpus)
        return index.histograms(docs), None
    n = index.docs.n_rows
    m = min(args.sample, n)
    ids = np.sort(np.random.default_rng(args.seed).choice(n, m, replace=False))
    return index.docs.take_rows(ids), ids


def _ks(args, n: int) -> list[int]:
    if getattr(args, "k_pct", None):
        ks = [max(1, int(math.ceil(p / 100.0 * n))) for p in args.k_pct]
    else:
        ks = list(args.k)
    if max(ks) > n:
        raise ValueError(f"k = {max(ks)} exceeds the {n} resident documents")
    return ks


def cmd_index(args) -> None:
    vocab, E = corpus.load_embeddings(args.embeddings, args.format)
    stop = corpus.read_stopwords(args.stopwords) if args.stopwords else None
    labels = corpus.read_labels(args.labels) if args.labels else None
    idx = engine.build_index(args.corpus, vocab, E, stopwords=stop, labels=labels)
    engine.save_index(idx, args.index)
    with _out(args.out) as fh:
        fh.write(json.dumps({"index": args.index, "n": idx.docs.n_rows, "v_e": len(idx.words),
                             "m": int(idx.embeddings.shape[1]), "nnz": idx.docs.nnz}) + "\n")


def cmd_query(args) -> None:
    idx = engine.open_index(args.index)
    q, qids = _queries(args, idx)
    k = _ks(args, idx.docs.n_rows)[0]
    plan = engine.QueryPlan(method=args.method, k=k, batch_size=args.batch, partitions=args.partitions,
                            self_exclusion=args.exclude_self)
    res = engine.run_query(idx, q, plan, query_ids=qids)
    with _out(args.out) as fh:
        for j, r in enumerate(res):
            rec = {"query": int(qids[j]) if qids is not None else j, "method": args.method,
                   "ids": [int(i) for i in r.ids], "distances": [float(d) for d in r.distances]}
            fh.write(json.dumps(rec) + "\n")


def cmd_bench(args) -> None:
    idx = engine.open_index(args.index)
    q, _ = _queries(args, idx)
    with _out(args.out) as fh:
        engine.benchmark(idx, q, args.methods, args.partitions, k=_ks(args, idx.docs.n_rows)[0], out=fh)


def _topk(idx, q, qids, method, k, exclude):
    plan = engine.QueryPlan(method=method, k=k, self_exclusion=exclude)
    return engine.run_query(idx, q, plan, query_ids=qids)


def cmd_overlap(args) -> None:
    """|topk(method) ∩ topk(reference)| / k averaged over queries (PAPER Fig. 7)."""
    idx = engine.open_index(args.index)
    q, qids = _queries(args, idx)
    ks = _ks(args, idx.docs.n_rows)
    kmax = max(ks)
    a = _topk(idx, q, qids, args.method, kmax, args.exclude_self)
    b = _topk(idx, q, qids, args.reference, kmax, args.exclude_self)
    with _out(args.out) as fh:
        for k in ks:
            ov = float(np.mean([len(set(x.ids[:k].tolist()) & set(y.ids[:k].tolist())) / k for x, y in zip(a, b)]))
            fh.write(json.dumps({"method": args.method, "reference": args.reference, "k": k,
                                 "k_pct": 100.0 * k / idx.docs.n_rows, "overlap": ov}) + "\n")


def cmd_precision(args) -> None:
    """Fraction of same-label docs in each query's top-k, mean per label, geometric mean
    over the labels of each frequency bucket (PAPER §VI)."""
    idx = engine.open_index(args.index)
    if idx.labels is None:
        raise ValueError("precision needs an index built with --labels")
    q, qids = _queries(args, idx)
    if qids is None:
        raise ValueError("precision needs sampled resident queries (--sample)")
    labels = np.asarray(idx.labels)
    ks = _ks(args, idx.docs.n_rows)
    res = _topk(idx, q, qids, args.method, max(ks), True)
    freq = {lab: int(np.sum(labels == lab)) for lab in set(labels.tolist())}
    bounds = list(args.buckets)
    with _out(args.out) as fh:
        for k in ks:
            per_label: dict[str, list[float]] = {}
            for j, r in enumerate(res):
                lab = labels[int(qids[j])]
                per_label.setdefault(lab, []).append(float(np.mean(labels[r.ids[:k]] == lab)))
            means = {lab: float(np.mean(v)) for lab, v in per_label.items()}
            for bi in range(len(bounds) + 1):
                lo = bounds[bi - 1] if bi else 0
                hi = bounds[bi] if bi < len(bounds) else float("inf")
                vals = [v for lab, v in means.items() if lo <= freq[lab] < hi]
                if not vals:
                    continue
                gm = float(np.exp(np.mean(np.log(np.maximum(vals, 1e-12))))) if min(vals) > 0 else 0.0
                fh.write(json.dumps({"method": args.method, "k": k, "bucket": [lo, None if hi == float("inf") else hi],
                                     "labels": len(vals), "precision": gm}) + "\n")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1711_07227_b200.cli", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common_query(p, multi_k=False):
        p.add_argument("--index", required=True)
        g = p.add_mutually_exclusive_group()
        g.add_argument("--corpus")
        g.add_argument("--sample", type=int, default=100)
        p.add_argument("--seed", type=int, default=0)
        kg = p.add_mutually_exclusive_group()
        kg.add_argument("--k", type=int, nargs="+" if multi_k else 1, default=[10])
        kg.add_argument("--k-pct", type=float, nargs="+" if multi_k else 1)
        p.add_argument("--exclude-self", action="store_true")
        p.add_argument("--out")

    p = sub.add_parser("index", help="ingest + restrict + persist")
    p.add_argument("--embeddings", required=True)
    p.add_argument("--format", choices=["text", "binary"], default="text")
    p.add_argument("--corpus", required=True)
    p.add_argument("--stopwords")
    p.add_argument("--labels")
    p.add_argument("--index", required=True)
    p.add_argument("--out")
    p.set_defaults(fn=cmd_index)

    p = sub.add_parser("query", help="top-k per query (JSON lines)")
    common_query(p)
    p.add_argument("--method", choices=engine.METHODS, default="lc-rwmd")
    p.add_argument("--batch", type=int, default=32)
    p.add_argument("--partitions", type=int, default=1)
    p.set_defaults(fn=cmd_query)

    p = sub.add_parser("bench", help="timing records per (method, P)")
    common_query(p)
    p.add_argument("--methods", nargs="+", choices=engine.METHODS, default=["lc-rwmd"])
    p.add_argument("--partitions", type=int, nargs="+", default=[1])
    p.set_defaults(fn=cmd_bench)

    p = sub.add_parser("overlap", help="top-k overlap of a method with a reference method")
    common_query(p, multi_k=True)
    p.add_argument("--method", choices=engine.METHODS, default="rwmd")
    p.add_argument("--reference", choices=engine.METHODS, default="wmd")
    p.set_defaults(fn=cmd_overlap)

    p = sub.add_parser("precision", help="same-label precision at top-k (needs labels)")
    common_query(p, multi_k=True)
    p.add_argument("--method", choices=engine.METHODS, default="lc-rwmd")
    p.add_argument("--buckets", type=int, nargs="*", default=[300, 1000, 10000, 100000])
    p.set_defaults(fn=cmd_precision)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        args.fn(args)
    except (ValueError, OSError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
