"""The sharded pipeline as real processes on the GPU box: world 2 and 3, every rank on
cuda:0 (the box has one GPU, and NCCL refuses two ranks on one device), collectives
over gloo on the CUDA tensors.  parallel.sharded_topk (vocabulary-slice Phase 1, the
Z1 all-gather, the local reverse pass with the fused top-k, the gather of the per-rank
lists to rank 0 and their merge) and parallel.sharded_all_pairs_topk (the all_to_all
of C's row blocks, uneven shards) must give rank 0 exactly the single-process result
(partition invariance).  The NCCL calls are the same torch.distributed
calls (allgather_slices, gather_candidates, exchange_blocks, gather_rows_uneven)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_1711_07227_b200 import synthetic as S
    V = 6000
    E = S.embeddings(V, 300, seed=51)
    x1 = S.histograms(2999, V, 40, seed=52)
    x2 = S.histograms(45, V, 40, seed=53)
    return E, x1, x2


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1711_07227_b200 import device, parallel
        E, x1, x2 = _case()
        lo, hi = parallel.shard_range(x1.n_rows, rank, world)
        prep = device.PreparedEmbeddings(E)
        out = parallel.sharded_topk(device.DeviceCSR.upload(x1.slice_rows(lo, hi)), lo, x1.n_rows,
                                    device.DeviceCSR.upload(x2), prep, 10)
        dx_all = device.DeviceCSR.upload(x1.slice_rows(0, 700))
        n = dx_all.n_rows
        alo, ahi = parallel.shard_range(n, rank, world)
        ap = parallel.sharded_all_pairs_topk(dx_all.slice_rows(alo, ahi), dx_all, alo, prep, 7, batch=128)
        if rank == 0:
            q.put(("ok", out[0].cpu().numpy(), out[1].cpu().numpy(), ap[0].cpu().numpy(), ap[1].cpu().numpy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("err", traceback.format_exc(), None, None, None))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_processes_match_single_process(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1711_07227_b200 import device
    E, x1, x2 = _case()
    prep = device.PreparedEmbeddings(E)
    rd, ri = device.symmetric(device.DeviceCSR.upload(x1), device.DeviceCSR.upload(x2), prep, 10)
    dx_all = device.DeviceCSR.upload(x1.slice_rows(0, 700))
    full = device.all_pairs(dx_all, prep, batch=128)
    n = dx_all.n_rows
    ad = torch.empty((n, 7), dtype=torch.float32, device=full.device)
    ai = torch.empty((n, 7), dtype=torch.int64, device=full.device)
    device.topk_matrix_rows(full, n, n, n, 0, 7, ad, ai)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
    assert res[0] == "ok", res[1]
    assert np.array_equal(res[1], rd.cpu().numpy()) and np.array_equal(res[2], ri.cpu().numpy())
    assert np.array_equal(res[3], ad.cpu().numpy()) and np.array_equal(res[4], ai.cpu().numpy())
