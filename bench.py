#!/usr/bin/env python
"""Benchmark: symmetric LC-RWMD doc-pair distances/sec (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|mid|c4|c5]

Other --config values run one GPU's share of BASELINE configs[3] (c4: V = 3M,
h ~ 150) and [4] (c5: a 4k-query batch on a 25k-doc shard, V = 400k); the
all-pairs path for configs[4] is measured by bench_rows.py.

Workload (BASELINE.json configs[1] = SURVEY "C2"): 1M resident docs x 1k query
docs, vocabulary 100k, m = 300, ~50 unique words/doc, top-k = 10, synthetic
(N(0,1) embeddings, uniform word ids, (u+0.1)/sum weights; seeds fixed).

One step = the whole symmetric LC-RWMD top-k from HBM-resident raw inputs
(E f32, both CSR sets): f16 operand preparation + identity classes,
restriction of both sides, forward Phase 1 + SpMM, reverse Phase 1 (at C2 the
distance-table form: table build + per-doc gathers; --reverse gemm forces the
GEMM form) + reverse SpMM with the max-combine over doc batches, per-query
top-k.  Inputs (X1 = 400 MB, D1 = 4 GB,
Z2 batches of GBs) are far larger than the 126 MB L2, so no flush is needed.

`value` is device-timed (CUDA events on the launching stream, max over
ranks); `e2e` calls the public API distances.lcrwmd_topk with pinned host
arrays, so it includes the host->device copies of X1, X2, E and the
device->host read of the (n2, k) result.  `roofline` is the dominant kernel,
timed live with events inside the timed region: table_min_kernel against the
L2 gather ceiling measured by tools/l2gather.cu (profiles/l2_gather_peak.json),
or, on the GEMM form, the reverse phase1_kernel against the sustained tensor
peak; `phase1_tensor` reports every Phase-1 GEMM launch against that peak.

With --gpus N > 1 (torchrun, NCCL) resident docs are sharded by contiguous
rows; Phase 1 of the forward direction is split by vocabulary slice with Z1
all-gathered, the reverse direction is local, and per-shard top-k lists are
gathered to rank 0 and merged (paper_1711_07227_b200/parallel.py).  Total work
is fixed (strong scaling of C2, as BASELINE.json configs[2] describes).

--impl reference times the reference algorithm (the pinned CPU oracle port,
oracle/lcrwmd_oracle.py, all host threads) on bounded samples of each part of
the same workload, extrapolated part by part to the full step (CpuSample);
rank 0 only.  `--gpus N` outside torchrun re-launches itself as N ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c2": dict(n_docs=1_000_000, n_queries=1000, vocab=100_000, dim=300, h=50, k=10,
               l2="inputs larger than L2 (X1 400 MB, D1 4 GB, distance table 11.8 GB); no flush",
               workload="symmetric LC-RWMD top-10, 1M docs x 1k queries, V=100k, m=300, h~50 (BASELINE configs[1])"),
    "c1": dict(n_docs=2000, n_queries=64, vocab=20_000, dim=300, h=40, k=10,
               workload="symmetric LC-RWMD top-10, 2000 docs x 64 queries, V=20k, m=300, h~40 (BASELINE configs[0])"),
    "mid": dict(n_docs=100_000, n_queries=256, vocab=50_000, dim=300, h=50, k=10,
                workload="symmetric LC-RWMD top-10, 100k docs x 256 queries, V=50k, m=300, h~50 (dev size)"),
    # one GPU's share of BASELINE configs[3] (V = 3M, h ~ 150; 4M docs over 8 GPUs -> 500k per GPU)
    "c4": dict(n_docs=500_000, n_queries=1000, vocab=3_000_000, dim=300, h=150, k=10,
               l2="inputs larger than L2 (E 3.6 GB, X1 600 MB, Z1 12 GB); no flush",
               workload="symmetric LC-RWMD top-10, 500k docs (one of 8 shards of 4M) x 1k queries, V=3M, m=300, "
                        "h~150 (BASELINE configs[3] per GPU)"),
    # one 4k-query batch of BASELINE configs[4] on one GPU's 25k-doc shard (200k docs over 8 GPUs)
    "c5": dict(n_docs=25_000, n_queries=4096, vocab=400_000, dim=300, h=50, k=10,
               l2="inputs larger than L2 (E 480 MB, Z1 of the batch 6.6 GB); no flush",
               workload="symmetric LC-RWMD top-10, 25k docs (one of 8 shards of 200k) x a 4k-query batch, V=400k, "
                        "m=300, h~50 (BASELINE configs[4] per GPU and batch)"),
}
METRIC = "symmetric RWMD doc-pair distances/sec"
UNIT = "doc-pairs/s"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def make_data(cfg):
    from paper_1711_07227_b200 import synthetic as S
    E = S.embeddings(cfg["vocab"], cfg["dim"], seed=0)
    x1 = S.histograms(cfg["n_docs"], cfg["vocab"], cfg["h"], seed=1)
    x2 = S.histograms(cfg["n_queries"], cfg["vocab"], cfg["h"], seed=2)
    return E, x1, x2


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                try:
                    rows.append((float(f[0]), float(f[1]), float(f[2]), f[3:7]))
                except ValueError:
                    pass
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3]) if v.lower().startswith("active")})
        loaded = [r[0] for r in rows if r[2] > 200.0] or [r[0] for r in rows]
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port, all host threads): bounded samples of each part of the
# step, each extrapolated to the full workload by its own work model
# ---------------------------------------------------------------------------
class CpuSample:
    """The reference algorithm's step (lcrwmd_full + per-query top-k, distances.py:244-264,
    kernels.py:210-223) on the host cores, timed as four parts on bounded samples and
    extrapolated part by part (each oracle loop is linear in its row count):

      forward Phase 1   R restricted-vocabulary rows x all query words  -> x v_e1 / R
      forward SpMM      n_s docs x all queries                          -> x n1 / n_s
      reverse direction n_s docs as queries against the query set       -> x n1 / n_s
      max + top-k       the n_s x n2 block, per query                   -> x n1 / n_s

    (a plain "first n docs" sample would under-count the forward pass, whose vocabulary
    restriction -- hence Phase-1 work -- grows with n until it saturates at ~V)."""

    def __init__(self, E, x1, x2, k, rows: int, docs: int, threads: int):
        from oracle import lcrwmd_oracle as O
        self.O, self.E, self.x1, self.x2, self.k, self.threads = O, E, x1, x2, k, threads
        self.used1 = np.unique(np.asarray(x1.column_ids))
        self.v_e1 = int(self.used1.size)
        self.rows = min(rows, self.v_e1)
        self.docs = min(docs, x1.n_rows)
        self.xs = O.as_csr(x1.slice_rows(0, self.docs))
        self.x2c = O.as_csr(x2)
        self.t2 = np.ascontiguousarray(E[np.asarray(x2.column_ids)])
        self.e_rows = np.ascontiguousarray(E[self.used1[: self.rows]])
        self.x2r, self.e2, _ = O.restrict_vocabulary(self.x2c, E)
        self.xsr, _, _ = O.restrict_vocabulary(self.xs, E)
        rng = np.random.default_rng(0)
        self.z1 = rng.random((self.xsr.n_cols, x2.n_rows), dtype=np.float32)  # SpMM cost: any values

    def step(self) -> dict:
        O, th = self.O, self.threads
        t = {}
        t0 = time.perf_counter()
        O.phase1(self.e_rows, self.t2, np.asarray(self.x2c.row_offsets), threads=th)
        t["fwd_phase1"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        d1 = O.spmm(self.xsr, self.z1, threads=th)
        t["fwd_spmm"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        d2t = O.one_direction(self.x2r, self.e2, self.E, self.xs, threads=th)
        t["reverse"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.topk_per_query(np.maximum(d1, d2t.T), self.k)
        t["max_topk"] = time.perf_counter() - t0
        return t

    def extrapolate(self, t: dict) -> float:
        """Seconds for the full workload (n1 docs x n2 queries)."""
        f_docs = self.x1.n_rows / self.docs
        return (t["fwd_phase1"] * self.v_e1 / self.rows
                + (t["fwd_spmm"] + t["reverse"] + t["max_topk"]) * f_docs)

    def describe(self, t: dict) -> str:
        return (f"extrapolated from bounded samples of the same workload (oracle/lcrwmd_oracle.py, "
                f"{self.threads} threads): forward Phase 1 on {self.rows} of {self.v_e1} restricted vocabulary rows x "
                f"all {self.x2.nnz} query words ({t['fwd_phase1']:.2f} s, x{self.v_e1 / self.rows:.1f}); "
                f"forward SpMM, reverse direction and max+top-{self.k} on {self.docs} of {self.x1.n_rows} docs "
                f"({t['fwd_spmm']:.2f} + {t['reverse']:.2f} + {t['max_topk']:.2f} s, "
                f"x{self.x1.n_rows / self.docs:.0f})")


def cpu_sample_rate(E, x1, x2, k, target_s: float, rows: int = 2048, docs: int = 512):
    from oracle import lcrwmd_oracle as O
    threads = O.default_threads()
    smp = CpuSample(E, x1, x2, k, rows, docs, threads)
    tot = {}
    t_start = time.perf_counter()
    reps = 0
    while True:
        for n_, v in smp.step().items():
            tot[n_] = tot.get(n_, 0.0) + v
        reps += 1
        if time.perf_counter() - t_start >= target_s:
            break
    avg = {n_: v / reps for n_, v in tot.items()}
    secs = smp.extrapolate(avg)
    return {"value": x1.n_rows * x2.n_rows / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "extrapolated": True, "seconds_full_step": secs, "parts_s": avg,
            "sample": smp.describe(avg) + f"; {reps} repetition(s)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1711_07227_b200 import _lib, device, distances, parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.force_sharded:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    E, x1, x2 = make_data(cfg)
    k = cfg["k"]
    n1, n2 = x1.n_rows, x2.n_rows
    lo, hi = parallel.shard_range(n1, rank, world)
    x1s = x1.slice_rows(lo, hi)

    # HBM-resident inputs for the device-timed value
    Ed = device.to_device(E, torch.float32)
    dx1 = device.DeviceCSR.upload(x1s, "x1")
    dx2 = device.DeviceCSR.upload(x2, "x2")

    def step():
        prep = device.PreparedEmbeddings(Ed)
        if world == 1 and not args.force_sharded:
            return device.symmetric(dx1, dx2, prep, k, z2_budget_bytes=args.z2_mb << 20)
        return parallel.sharded_topk(dx1, lo, n1, dx2, prep, k)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    _lib.profile_reset(True)
    calls0 = dict(_lib.CALLS)
    clocks = ClockSampler(local)
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    ev0.record()
    for _ in range(args.steps):
        out = step()
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    calls = {n: c - calls0.get(n, 0) for n, c in _lib.CALLS.items()}
    ksum = _lib.profile_read()
    _lib.profile_reset(False)
    # reverse pipeline: 6 kernels per doc batch (gather, 2 plan, phase1, zeros, reverse_panels), counted
    # from its reverse_panels launches; calibrated against the ncu launch list (profiles/)
    rev_batches = ksum.get("reverse_panels", {"launches": 0})["launches"]
    table_mode = "table_min" in ksum
    per_batch = _lib.REVERSE_KERNELS_PER_BATCH_TABLE if table_mode else _lib.REVERSE_KERNELS_PER_BATCH
    launches = (_lib.launches(calls) + per_batch * rev_batches) // args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- end to end through the public API (pinned host buffers) ----
    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()

    from paper_1711_07227_b200.corpus import HistogramSet
    hx1 = HistogramSet(pinned(x1s.row_offsets), pinned(x1s.column_ids), pinned(x1s.values), x1s.n_cols)
    hx2 = HistogramSet(pinned(x2.row_offsets), pinned(x2.column_ids), pinned(x2.values), x2.n_cols)
    hE = pinned(E)
    h2d = sum(a.nbytes for a in (hx1.row_offsets, hx1.column_ids, hx1.values, hx2.row_offsets,
                                 hx2.column_ids, hx2.values, hE))
    d2h = n2 * k * (4 + 8)

    def e2e_step():
        if world == 1 and not args.force_sharded:
            return distances.lcrwmd_topk_arrays(hx1, hx2, hE, k)
        return parallel.sharded_topk_host(hx1, lo, n1, hx2, hE, k)

    e2e_step()
    e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(e_steps):
        e2e_step()
    t1.record()
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1) / e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        barrier()

    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    pk, pk_kind = peaks()
    tpath = ROOT / "profiles" / "roofline_traffic.json"
    traffic_all = json.loads(tpath.read_text()) if tpath.exists() and args.config == "c2" else {}
    v_e2 = int(np.unique(x2.column_ids).size)
    # algorithmic FLOPs of a Phase-1 GEMM: 2 * rows * cols * m, K = m unpadded
    rev_flops = 2.0 * v_e2 * x1s.nnz * cfg["dim"]
    fwd_flops = 2.0 * int(np.unique(x1s.column_ids).size) * x2.nnz * cfg["dim"]
    table_flops = 2.0 * v_e2 * cfg["vocab"] * cfg["dim"]
    # table_min gathers, per doc word and 256-word table chunk, one 512-byte row of 16-bit keys
    # (2 B per (query-vocabulary word, doc word) distance) and writes one 4-byte Z2 entry per
    # (query-vocabulary word, doc)
    from paper_1711_07227_b200 import _lib as _L, device as _dev
    n_chunks = -(-v_e2 // int(_L.value("lcrw_table_chunk")))
    table_bytes = float(_dev.TABLE_ROW_BYTES) * n_chunks * x1s.nnz + 4.0 * v_e2 * x1s.n_rows
    table_entries = float(v_e2) * x1s.nnz
    spmm_bytes = 8.0 * (x1s.n_rows + 1) + 8.0 * x1s.nnz + 4.0 * x1s.nnz * n2
    # reverse_panels streams every Z2 panel once (4 * v_e2 bytes per doc) and reads D1; with the
    # fused top-k (k <= 32) D is not written
    rev_bytes = 4.0 * v_e2 * x1s.n_rows + (4.0 if k <= 32 else 8.0) * n2 * x1s.n_rows
    work = {"phase1": fwd_flops, "phase1_rev": rev_flops, "table_build": table_flops, "spmm": spmm_bytes,
            "reverse_panels": rev_bytes, "table_min": table_bytes}
    peak_tf = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    pairs = n1 * n2
    value = pairs / (ms * 1e-3)
    # every tcgen05 Phase-1 launch of the step (forward, reverse GEMM or the distance-table
    # build) against the tensor peak: the north star's Phase-1 GEMM evidence on either path
    p1_flops = {"phase1": fwd_flops, "phase1_rev": rev_flops, "table_build": table_flops}
    p1_ms = sum(ksum[n]["ms"] for n in p1_flops if n in ksum) / args.steps
    p1_work = sum(f for n, f in p1_flops.items() if n in ksum)
    # Phase 2 (the forward CSR SpMM and the reverse SpMM + max-combine) against the HBM peak,
    # algorithmic bytes as SURVEY §8(d) defines them (reads of X, Z gathers / Z2 stream, D1, D)
    p2 = {"spmm": spmm_bytes, "reverse_panels": rev_bytes}
    p2_ms = sum(ksum[n]["ms"] for n in p2 if n in ksum) / args.steps
    p2_bytes = sum(b for n, b in p2.items() if n in ksum)
    hbm = pk.get("hbm_gbs")
    phase2_hbm = {"kernels": [n for n in p2 if n in ksum], "ms_per_step": p2_ms,
                  "achieved": p2_bytes / (p2_ms * 1e-3) / 1e9 if p2_ms else None, "peak": hbm, "unit": "GB/s",
                  "frac": p2_bytes / (p2_ms * 1e-3) / 1e9 / hbm if p2_ms and hbm else None,
                  "per_kernel_frac": {n: p2[n] / (ksum[n]["ms"] / args.steps * 1e-3) / 1e9 / hbm
                                      for n in p2 if n in ksum and hbm},
                  "note": "spmm's Z1 gathers are served partly by L2 (Z1 in L2-resident 128-query panels), so "
                          "its algorithmic rate can exceed the HBM peak"}
    phase1_tensor = {"kernels": [n for n in p1_flops if n in ksum], "ms_per_step": p1_ms,
                     "achieved": p1_work / (p1_ms * 1e-3) / 1e12 if p1_ms else None, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": p1_work / (p1_ms * 1e-3) / 1e12 / peak_tf if p1_ms else None,
                     "note": "algorithmic 2*rows*cols*m FLOP of the Phase-1 GEMMs launched per step; the table "
                             "build is store-bound (7.9 GB of table at C2), the GEMM-path reverse Phase 1 "
                             "(--reverse gemm) runs at 0.93-0.97 of the sustained peak"}
    if table_mode:  # dominant kernel: the distance-table gathers, bound by L2 bandwidth
        tm = ksum["table_min"]
        achieved = table_bytes / (tm["ms"] / args.steps * 1e-3) / 1e9
        l2path = ROOT / "profiles" / "l2_gather_peak.json"
        l2 = json.loads(l2path.read_text()) if l2path.exists() else {"gbs": float("nan"), "source": "missing"}
        tr = traffic_all.get("table_min_kernel")
        roofline = {"kernel": "table_min_kernel (reverse Phase 1: per-doc min over 512-B rows of 16-bit keys of "
                              "an L2-resident 256-word distance-table chunk)",
                    "bound": "l2", "achieved": achieved, "peak": l2["gbs"], "unit": "GB/s",
                    "frac": achieved / l2["gbs"],
                    "traffic": tr["dram_bytes_per_launch"] if tr else None,
                    "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/roofline_traffic.json)",
                    "traffic_launch_docs": tr.get("launch_docs") if tr else None,
                    "traffic_over_algorithmic": tr.get("traffic_over_algorithmic") if tr else None,
                    "ncu_lts_throughput_pct": tr.get("lts_throughput_pct") if tr else None,
                    "ncu_l2_hit_rate_pct": tr.get("lts_hit_rate_pct") if tr else None,
                    "algorithmic_bytes_per_launch": table_bytes * args.steps / tm["launches"],
                    "algorithmic_bytes_note": "mean over the step's launches (full doc batches + the remainder); "
                                              "traffic_over_algorithmic compares ncu's DRAM bytes with the "
                                              "algorithmic bytes of that same full-batch launch",
                    "peak_source": f"measured L2 gather ceiling on B200 ({l2['source']})",
                    "hbm_peak_gbs": pk.get("hbm_gbs"), "achieved_over_hbm_peak": achieved / pk.get("hbm_gbs", 1.0),
                    "per_launch_ms": tm["ms"] / max(tm["launches"], 1),
                    "distances_per_s": table_entries / (tm["ms"] / args.steps * 1e-3),
                    "launches_per_step": tm["launches"] / args.steps, "share_of_step": tm["ms"] / args.steps / ms}
    else:
        rev = ksum.get("phase1_rev", {"ms": float("nan"), "launches": 1})
        achieved_tf = rev_flops / (rev["ms"] / args.steps * 1e-3) / 1e12
        tr = traffic_all.get("phase1_kernel")
        roofline = {"kernel": "phase1_kernel (reverse direction, tcgen05 f16 GEMM + fused segmented min)",
                    "bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": achieved_tf / peak_tf, "traffic": tr["dram_bytes_per_launch"] if tr else None,
                    "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/roofline_traffic.json)",
                    "peak_source": f"{pk_kind} bf16_tflops_sustained (dense f16 = bf16 rate)",
                    "per_launch_ms": rev["ms"] / max(rev["launches"], 1),
                    "launches_per_step": rev["launches"] / args.steps, "share_of_step": rev["ms"] / args.steps / ms}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16 operands, fp32 accumulate",
        "data": "synthetic (N(0,1) embeddings, uniform word ids; seeds 0/1/2)",
        "config": bench_config(cfg, world),
        "e2e": {"value": pairs / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "paper_1711_07227_b200.distances.lcrwmd_topk (pinned host arrays)"},
        "roofline": roofline,
        "kernels": {n: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                        ("tflops" if n.startswith(("phase1", "table_build")) else "gbs_algorithmic"):
                            (work.get(n, 0.0) / (v["ms"] / args.steps * 1e-3) /
                             (1e12 if n.startswith(("phase1", "table_build")) else 1e9))}
                    for n, v in ksum.items()},
        "phase1_tensor": phase1_tensor,
        "phase2_hbm": phase2_hbm,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample_rate(E, x1, x2, k, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on the host cores
# ---------------------------------------------------------------------------
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import lcrwmd_oracle as O
    E, x1, x2 = make_data(cfg)
    k = cfg["k"]
    threads = O.default_threads()
    smp = CpuSample(E, x1, x2, k, args.ref_rows, args.ref_docs, threads)
    for _ in range(args.warmup):
        smp.step()
    tot = {}
    for _ in range(args.steps):
        for n_, v in smp.step().items():
            tot[n_] = tot.get(n_, 0.0) + v
    avg = {n_: v / args.steps for n_, v in tot.items()}
    secs = smp.extrapolate(avg)
    value = x1.n_rows * x2.n_rows / secs
    sample = smp.describe(avg) + "; the reference is pure Python (no compiled build): its algorithm restated in " \
                                 "numpy, pinned to the reference's outputs (tests/golden)"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True, "impl": "reference",
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (N(0,1) embeddings, uniform word ids; seeds 0/1/2)",
            "config": bench_config(cfg, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "extrapolated": True,
                             "sample": sample, "parts_s": avg},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_config(cfg, world: int) -> dict:
    """The config object both arms print (identical keys and values)."""
    return {"workload": cfg["workload"], "n_docs": cfg["n_docs"], "n_queries": cfg["n_queries"],
            "vocab": cfg["vocab"], "dim": cfg["dim"], "h": cfg["h"], "k": cfg["k"],
            "parallelism": f"docs sharded x{world}",
            "l2": cfg.get("l2", "small inputs (not a headline config); no flush")}


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: re-run this command as N ranks
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-docs", type=int, default=512,
                    help="sampled resident docs per reference-arm step (SpMM, reverse, top-k parts)")
    ap.add_argument("--ref-rows", type=int, default=2048,
                    help="sampled restricted-vocabulary rows per reference-arm step (forward Phase 1 part)")
    ap.add_argument("--z2-mb", type=int, default=4096, help="reverse Z2 batch budget (MiB)")
    ap.add_argument("--reverse", choices=["auto", "gemm", "table"], default="auto",
                    help="reverse Phase-1 form (sets LCRW_REVERSE): auto picks the distance table when "
                         "nnz(X1) >> V, gemm is the tcgen05 GEMM + fused segmented min throughout")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the multi-GPU code path (NCCL process group) even with one rank")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}; using WORLD_SIZE",
              file=sys.stderr)
    if args.reverse != "auto":
        os.environ["LCRW_REVERSE"] = args.reverse
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
