#!/usr/bin/env python
"""Cost of the near-entry exact refinement (csrc/refine.cu) as the share of near
entries grows: symmetric top-10 over n docs x 1k queries (V = 100k, m = 300, h ~ 50)
with N(0,1) embeddings (nothing near; the bench's data) and clustered embeddings
(500 centres, varying spread: words of one cluster sit close to each other).

Prints one JSON line per embedding model: step time (CUDA events, table form and
GEMM form) and the sampled share of reverse Z2 entries (query word a, doc) with
0 < min_b |a - b| < 0.5 |a| (numpy, f64, on a sample).

    python tools/near_cost.py [--docs 200000] [--steps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def near_share(E, x1, x2, rng, n_docs=200, n_words=64):
    qw = np.unique(x2.column_ids)
    a_ids = rng.choice(qw, min(n_words, len(qw)), replace=False)
    docs = rng.choice(x1.n_rows, n_docs, replace=False)
    A = E[a_ids].astype(np.float64)
    an = np.linalg.norm(A, axis=1)
    near = 0
    for d in docs:
        B = E[x1.column_ids[x1.row_offsets[d]:x1.row_offsets[d + 1]]].astype(np.float64)
        dist = np.sqrt(np.maximum(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1), 0)).min(axis=1)
        near += int(((dist > 0) & (dist < 0.5 * an)).sum())
    return near / (len(a_ids) * n_docs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=200_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--spreads", default="0.2,0.3,0.4")
    ap.add_argument("--modes", default="table,gemm")
    ap.add_argument("--profile", action="store_true", help="per-kernel ms of one table-form step")
    args = ap.parse_args()
    import torch
    from paper_1711_07227_b200 import device, synthetic as S
    V, m = 100_000, 300
    x1 = S.histograms(args.docs, V, 50, seed=1)
    x2 = S.histograms(1000, V, 50, seed=2)
    models = [("normal", None)] + [("clustered", float(s)) for s in args.spreads.split(",")]
    rng = np.random.default_rng(5)
    for name, spread in models:
        E = (S.embeddings(V, m, seed=0) if spread is None
             else S.embeddings(V, m, seed=0, clustered=True, centers=500, spread=spread))
        prep = device.PreparedEmbeddings(E)
        d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)
        row = {"model": name, "spread": spread, "docs": args.docs, "queries": 1000,
               "near_share_sampled": near_share(E, x1, x2, rng)}
        for mode in args.modes.split(","):
            os.environ["LCRW_REVERSE"] = mode
            device.symmetric(d1, d2, prep, 10)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                device.symmetric(d1, d2, prep, 10)
            e1.record()
            torch.cuda.synchronize()
            row[f"{mode}_ms"] = round(e0.elapsed_time(e1) / args.steps, 2)
        if args.profile:
            from paper_1711_07227_b200 import _lib
            os.environ["LCRW_REVERSE"] = "table"
            _lib.profile_reset(True)
            device.symmetric(d1, d2, prep, 10)
            torch.cuda.synchronize()
            row["profile_ms"] = {k: round(v["ms"], 2) for k, v in _lib.profile_read().items()}
            _lib.profile_reset(False)
        os.environ.pop("LCRW_REVERSE", None)
        print(json.dumps(row), flush=True)
        del prep, d1, d2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
