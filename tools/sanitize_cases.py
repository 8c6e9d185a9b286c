"""Small invocations of every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck) on a B200:

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Cases are tiny so the sanitizer's per-access instrumentation finishes in
minutes: the distance-table and GEMM reverse forms (phase1 tcgen05 kernel with
its TMA ring / 2-CTA clusters / TMEM, table build + table_min, reverse_panels,
SpMM, top-k), all-pairs symmetrise, the primitives (prims.cu) and exact EMD
(shared-memory and global-memory state).  Prints one line per case; exits
non-zero on the first failing assertion."""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_07227_b200 import distances, emd, kernels, synthetic as S  # noqa: E402


def main(which: set[str] | None = None) -> None:
    torch.cuda.set_device(0)
    V, m = 1500, 300
    E = S.embeddings(V, m, seed=0)
    x1 = S.histograms(300, V, 30, seed=1)
    x2 = S.histograms(12, V, 30, seed=2)

    def want(name):
        return which is None or name in which

    if want("table"):
        os.environ["LCRW_REVERSE"] = "table"
        a = distances.lcrwmd_full(x1, x2, E).values
        print("table form", a.shape, flush=True)
    if want("gemm"):
        os.environ["LCRW_REVERSE"] = "gemm"
        b = distances.lcrwmd_full(x1, x2, E).values
        print("gemm form", b.shape, flush=True)
    os.environ.pop("LCRW_REVERSE", None)
    if want("topk"):
        t = distances.lcrwmd_topk(x1, x2, E, 10)
        print("topk", len(t), flush=True)
    if want("small_m"):
        Es = S.embeddings(V, 48, seed=3)
        c = distances.lcrwmd_full(x1, x2, Es).values
        print("m=48 split form", c.shape, flush=True)
    if want("allpairs"):
        r = distances.lcrwmd_all_pairs_topk(x1.slice_rows(0, 100), E, 5, batch_size=32)
        print("all-pairs", len(r), flush=True)
    if want("prims"):
        rng = np.random.default_rng(4)
        a = rng.standard_normal((37, 19))
        sq = kernels.squared_norms(a)
        out = np.empty((37, 37), dtype=np.float32)
        kernels.euclidean_into(a, sq, a, sq, out)
        kernels.segmented_min(out, np.array([0, 5, 17, 37]), axis=1)
        kernels.row_min(out)
        kernels.col_min(out)
        kernels.topk_select(rng.standard_normal(3000), np.arange(3000), 7)
        kernels.topk_select(rng.standard_normal(3000), np.arange(3000), 1500)  # sort path (k > 1024)
        print("prims", flush=True)
    if want("emd"):
        d = emd.wmd(x1.row(0), x2.row(0), E)
        big = S.histograms(2, V, 220, seed=6)  # > shared-memory problem size: global-memory state
        d2 = emd.wmd(big.row(0), big.row(1), E)
        print("emd", float(d), float(d2), flush=True)
    if want("wmd_pruned"):
        r, n_solved = emd.prefiltered_topk_wmd(x1.slice_rows(0, 60), x2.row(1), E, 3)
        print("prefiltered wmd", len(r.ids), n_solved, flush=True)
    torch.cuda.synchronize()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main(set(sys.argv[1].split(",")) if len(sys.argv) > 1 else None)
