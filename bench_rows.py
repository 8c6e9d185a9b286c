#!/usr/bin/env python
"""Measurement of the rows next to the hot path, one JSON line each.

    python bench_rows.py [--rows wmd,wcd,allpairs] [--steps K] [--warmup W]

* ``wmd``: exact top-10 word mover's distances (emd.prefiltered_topk_wmd_batch:
  LC-RWMD bounds on the tensor cores, then batched exact transport solves in
  csrc/emd.cu) for 64 queries over 20,000 docs (V = 20k, m = 300, ~40 words per
  doc -- BASELINE configs[0]'s shape, 10x the docs).  Metric: queries/s, plus the
  exact solves per second of the EMD kernel.  CPU baseline: the oracle's
  restatement of the reference's prefiltered_topk_wmd (emd.py:214-261) on a
  bounded number of queries, single process.
* ``wcd``: word centroid distances (distances.wcd_block) for 100,000 x 1,000 docs
  (V = 100k, m = 300, ~50 words); metric doc-pairs/s; CPU baseline: the oracle's
  wcd_block on a bounded row sample.

* ``allpairs``: all-pairs symmetric LC-RWMD top-10 of 50,000 docs (V = 400k,
  m = 300, ~50 words, 4k-query batches -- BASELINE configs[4]'s shape on one
  GPU) through the forward-only all_pairs path, next to the general symmetric
  pipeline on the same set.

* ``allpairs_rank``: one rank's share of BASELINE configs[4] itself (200,000
  docs, V = 400k, 8 ranks): C = D1[:, S_0] for the 25,000-doc shard against all
  200,000 docs, the max-combine into its output rows and their top-10 -- what
  each GPU computes in parallel.sharded_all_pairs_topk.  The all_to_all of the
  row blocks (17.5 GB per rank) is not part of the timed region (one GPU here);
  the received blocks are stood in for by the rank's own rows.

* ``scaling``: rank 0's share of BASELINE configs[2] (C2 over N = 1, 2, 4, 8 GPUs)
  through the sharded code path, timed on one GPU; the collectives are estimated,
  not executed (projection).

Inputs are resident in HBM for the device-timed value (CUDA events); these rows
are not part of bench.py's headline line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def timed(fn, steps, warmup):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = None
    for _ in range(steps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, out


def row_wmd(args):
    import torch
    from oracle import lcrwmd_oracle as O
    from paper_1711_07227_b200 import _lib, emd, synthetic as S
    V, m, n1, nq, h, k = 20_000, 300, 20_000, 64, 40, 10
    E = S.embeddings(V, m, seed=0)
    x1 = S.histograms(n1, V, h, seed=1)
    x2 = S.histograms(nq, V, h, seed=2)
    Et = torch.from_numpy(E).cuda()
    _lib.profile_reset(True)
    ms, (res, solves) = timed(lambda: emd.prefiltered_topk_wmd_batch(x1, x2, Et, k), args.steps, args.warmup)
    prof = _lib.profile_read()
    _lib.profile_reset(False)
    emd_ms = prof.get("emd", {"ms": 0.0})["ms"] / (args.steps + args.warmup)
    total_solves = int(np.sum(solves))
    line = {"metric": "exact WMD top-k queries/sec (RWMD-prefiltered)", "value": nq / (ms * 1e-3),
            "unit": "queries/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "dtype": "f16 bounds / fp64 transport",
            "config": {"workload": "prefiltered exact top-10 WMD, 64 queries x 20k docs, V=20k, m=300, h~40",
                       "k": k, "exact_solves_per_step": total_solves,
                       "mean_solves_per_query": total_solves / nq},
            "kernels": {"emd_ms_per_step": emd_ms, "emd_solves_per_s": total_solves / max(emd_ms * 1e-3, 1e-9)}}
    # CPU baseline: the reference algorithm (oracle restatement) on a bounded number of queries
    t0 = time.perf_counter()
    nref = 0
    while nref < nq and (nref == 0 or time.perf_counter() - t0 < args.cpu_seconds):
        q = x2.row(nref)
        O.prefiltered_topk_wmd(x1, q.word_ids, q.weights, E, k)
        nref += 1
    dt = time.perf_counter() - t0
    line["cpu_baseline"] = {"value": nref / dt, "unit": "queries/s", "cores": 1, "kind": "port",
                            "sample": f"{nref} queries x 20k docs, oracle prefiltered_topk_wmd ({dt:.1f} s)"}
    for j in range(nref):  # the checked sample must agree with the GPU result
        q = x2.row(j)
        d, i, _ = O.prefiltered_topk_wmd(x1, q.word_ids, q.weights, E, k)
        assert np.array_equal(i, res[j].ids), ("wmd mismatch", j)
    print(json.dumps(line), flush=True)


def row_wcd(args):
    import torch
    from oracle import lcrwmd_oracle as O
    from paper_1711_07227_b200 import device, synthetic as S
    V, m, n1, n2, h = 100_000, 300, 100_000, 1000, 50
    E = S.embeddings(V, m, seed=0)
    x1 = S.histograms(n1, V, h, seed=1)
    x2 = S.histograms(n2, V, h, seed=2)
    Et = torch.from_numpy(E).cuda()
    d1, d2 = device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2)

    def step():
        return device.pairwise(device.centroids(d1, Et), device.centroids(d2, Et))

    ms, out = timed(step, args.steps, args.warmup)
    line = {"metric": "WCD doc-pairs/sec", "value": n1 * n2 / (ms * 1e-3), "unit": "doc-pairs/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "fp64 centroids / f16 Gram", "config": {"workload": "wcd_block 100k x 1k docs, V=100k, m=300"}}
    t0 = time.perf_counter()
    ns = 2000
    ref = O.wcd_block(x1.slice_rows(0, ns), x2, E)
    dt = time.perf_counter() - t0
    got = out[:ns].cpu().numpy()
    err = float(np.max(np.abs(got - ref) / (np.abs(ref) + 1e-3)))
    line["max_rel_err_sample"] = err
    line["cpu_baseline"] = {"value": ns * n2 / dt, "unit": "doc-pairs/s", "cores": 1, "kind": "port",
                            "sample": f"first {ns} docs x 1000, oracle wcd_block ({dt:.1f} s)"}
    print(json.dumps(line), flush=True)


def row_allpairs(args):
    """All-pairs symmetric LC-RWMD top-10 (BASELINE configs[4] shape on one GPU: V = 400k,
    h ~ 50, 4k-query batches): forward-only all_pairs vs the general symmetric pipeline
    on the same set."""
    import torch
    from paper_1711_07227_b200 import device, synthetic as S
    V, m, n, h, k, batch = 400_000, 300, args.allpairs_n, 50, 10, 4096
    E = S.embeddings(V, m, seed=0)
    x = S.histograms(n, V, h, seed=1)
    Et = torch.from_numpy(E).cuda()
    dx = device.DeviceCSR.upload(x)

    def step():
        prep = device.PreparedEmbeddings(Et)
        D = device.all_pairs(dx, prep, batch)
        od = torch.empty((n, k), dtype=torch.float32, device=D.device)
        oi = torch.empty((n, k), dtype=torch.int64, device=D.device)
        device.topk_matrix_rows(D, n, n, n, 0, k, od, oi)
        return od, oi

    ms, (od, oi) = timed(step, args.steps, args.warmup)
    del od, oi
    torch.cuda.empty_cache()

    def general():
        prep = device.PreparedEmbeddings(Et)
        return device.symmetric(dx, dx, prep, k)

    gms, _ = timed(general, 1, 1)
    line = {"metric": "all-pairs symmetric RWMD doc-pairs/sec", "value": n * n / (ms * 1e-3), "unit": "doc-pairs/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "f16 operands, fp32 accumulate, fp64 SpMM",
            "config": {"workload": f"all-pairs symmetric LC-RWMD top-10 of {n} docs, V=400k, m=300, h~50, "
                                   f"query batches of {batch} (BASELINE configs[4] shape, one GPU)"},
            "general_symmetric_path": {"ms_per_step": gms, "value": n * n / (gms * 1e-3),
                                       "note": "device.symmetric(x, x): forward + reverse per query group"}}
    print(json.dumps(line), flush=True)


def row_allpairs_rank(args):
    """Per-rank compute of sharded all-pairs at configs[4] scale (see module docstring)."""
    import torch
    from paper_1711_07227_b200 import device, parallel, synthetic as S
    V, m, n, h, k, world = 400_000, 300, 200_000, 50, 10, 8
    lo, hi = parallel.shard_range(n, 0, world)
    n_r = hi - lo
    E = S.embeddings(V, m, seed=0)
    x = S.histograms(n, V, h, seed=1)
    Et = torch.from_numpy(E).cuda()
    dx = device.DeviceCSR.upload(x)
    dloc = device.DeviceCSR.upload(x.slice_rows(lo, hi))
    C = torch.empty((n, n_r), dtype=torch.float32, device="cuda")
    Dr = torch.empty((n_r, n), dtype=torch.float32, device="cuda")
    od = torch.empty((n_r, k), dtype=torch.float32, device="cuda")
    oi = torch.empty((n_r, k), dtype=torch.int64, device="cuda")
    sizes = [parallel.shard_range(n, r, world)[1] - parallel.shard_range(n, r, world)[0] for r in range(world)]
    assert all(sz == n_r for sz in sizes)
    t = {}

    def step():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        prep = device.PreparedEmbeddings(Et)
        device.forward_rows_into(device.Restricted.build(dx, prep), prep, dloc, C, 4096)
        e[1].record()
        at = 0
        for sz in sizes:  # C[S_0] (n_r x n_r) stands in for the received block D1[S_0, S_s]
            device.max_transposed_into(Dr[:, at:at + sz], C[lo:hi], C[at:at + sz])
            at += sz
        device.topk_matrix_rows(Dr, n_r, n, n, 0, k, od, oi)
        e[2].record()
        t.setdefault("fwd", []).append(e)
        return od

    ms, _ = timed(step, args.steps, args.warmup)
    torch.cuda.synchronize()
    ev = t["fwd"][-args.steps:]
    fwd = sum(a[0].elapsed_time(a[1]) for a in ev) / len(ev)
    comb = sum(a[1].elapsed_time(a[2]) for a in ev) / len(ev)
    xch_bytes = (n - n_r) * n_r * 4
    # the other orientation (the shard's rows against all docs as queries), timed once:
    # Phase 1 is v_e(shard) x H(all) there, with v_e(shard) ~ v_e(all)
    del Dr
    Dold = torch.empty((n_r, n), dtype=torch.float32, device="cuda")
    prep = device.PreparedEmbeddings(Et)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    device.forward_rows_into(device.Restricted.build(dloc, prep), prep, dx, Dold, 4096)
    e1.record()
    torch.cuda.synchronize()
    old_ms = e0.elapsed_time(e1)
    del Dold
    line = {"metric": "all-pairs symmetric RWMD doc-pairs/sec (per-rank compute, configs[4] shard)",
            "value": n * n / (ms * 1e-3), "unit": "doc-pairs/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "f16 operands, fp32 accumulate, fp64 SpMM",
            "config": {"workload": "rank 0 of 8 for all-pairs top-10 of 200k docs, V=400k, m=300, h~50 "
                                   "(BASELINE configs[4]); value = n^2 / per-rank compute time, all_to_all excluded",
                       "n_docs": n, "shard_docs": n_r, "world": world},
            "split_ms": {"forward_C": fwd, "combine_topk": comb},
            "exchange_bytes_per_rank": xch_bytes,
            "rows_orientation_forward_ms": old_ms}
    print(json.dumps(line), flush=True)


def row_scaling(args):
    """Per-rank compute of BASELINE configs[2] (C2 sharded over N GPUs) on one B200: for N in
    1, 2, 4, 8 the step rank 0 runs in parallel.sharded_topk -- its vocabulary slice of the
    forward Phase 1 (Z1 rows [0, V/N)), the forward SpMM and the whole reverse direction on
    its 1M/N docs (the distance table is built by every rank: replicated E and X2), the
    max-combine and its per-query top-10.  The two collectives (the Z1 all-gather, 400 MB,
    and the gather of the 1k x 10 lists) are not executed: one GPU.  They are reported as
    bytes with an NVLink 5 estimate (all-gather of (N-1)/N x 400 MB at 600 GB/s per GPU).
    Projection, clearly not a multi-GPU measurement."""
    import torch
    from paper_1711_07227_b200 import device, parallel, synthetic as S
    V, m, n1, n2, h, k = 100_000, 300, 1_000_000, 1000, 50, 10
    E = S.embeddings(V, m, seed=0)
    x1 = S.histograms(n1, V, h, seed=1)
    x2 = S.histograms(n2, V, h, seed=2)
    Et = torch.from_numpy(E).cuda()
    dx2 = device.DeviceCSR.upload(x2)
    out = []
    base_ms = None
    for world in (1, 2, 4, 8):
        lo, hi = parallel.shard_range(n1, 0, world)
        dx1 = device.DeviceCSR.upload(x1.slice_rows(lo, hi))
        prep0 = device.PreparedEmbeddings(Et)
        # the other ranks' Z1 slices (the all-gather's result), computed outside the timed step
        slices = [parallel.z1_slice(dx2, prep0, r, world)[0] for r in range(world)]
        zall = torch.stack(slices).contiguous()
        R = parallel.vocab_slice(V, 0, world)[2]
        del slices

        def step():
            prep = device.PreparedEmbeddings(Et)
            zl, _ = parallel.z1_slice(dx2, prep, 0, world)  # this rank's slice (the all-gather's input)
            d1 = parallel.d1_from_slices(dx1, zall, R, n2)
            return device.symmetric(dx1, dx2, prep, k, d1=d1, id_offset=lo)

        ms, _ = timed(step, args.steps, args.warmup)
        if base_ms is None:
            base_ms = ms
        ag_bytes = (world - 1) / world * 4.0 * V * n2 if world > 1 else 0.0
        ag_ms = ag_bytes / 600e9 * 1e3
        proj = ms + ag_ms
        out.append({"n_gpus": world, "rank0_ms": ms, "allgather_bytes": ag_bytes, "allgather_ms_est": ag_ms,
                    "projected_step_ms": proj, "projected_pairs_per_s": n1 * n2 / (proj * 1e-3),
                    "projected_efficiency": base_ms / (world * proj)})
        del dx1, zall
    line = {"metric": "symmetric RWMD doc-pairs/sec, C2 sharded over N GPUs (per-rank compute on one B200)",
            "value": out[-1]["projected_pairs_per_s"], "unit": "doc-pairs/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "dtype": "f16 operands, fp32 accumulate",
            "config": {"workload": "rank 0's share of BASELINE configs[2] (1M docs x 1k queries, V=100k, m=300, "
                                   "top-10) for N = 1, 2, 4, 8; collectives not executed (one GPU), all-gather "
                                   "time estimated at 600 GB/s", "scaling": "strong"},
            "per_n": out}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="wmd,wcd")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--allpairs-n", type=int, default=50_000)
    args = ap.parse_args()
    for r in args.rows.split(","):
        {"wmd": row_wmd, "wcd": row_wcd, "allpairs": row_allpairs, "allpairs_rank": row_allpairs_rank,
         "scaling": row_scaling}[r](args)


if __name__ == "__main__":
    main()
