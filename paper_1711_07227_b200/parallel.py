"""Multi-GPU LC-RWMD: resident docs sharded across ranks (one process per GPU).

Decomposition ("spreading X1 across GPUs"; SPEC.md:357-383
contiguous shards + topk_merge):

* docs (rows of X1): contiguous shards, one per rank (``shard_range``);
  E, X2 and the query batch are replicated;
* forward Phase 1: rank r computes Z1 for its vocabulary slice
  [r*R, (r+1)*R) of the full vocabulary, R = ceil(V / world), and the slices
  are all-gathered over NVLink (NCCL) into [world][panels][R][W]; the SpMM of
  the local doc shard reads it through the blocked addressing of lcrw_spmm;
* reverse direction (the dominant cost): fully local -- each rank's docs are
  the "queries" of the reverse pass against the replicated X2;
* top-k: local per-query top-k, NCCL gather to rank 0, merge there
  (kernels.py:226-232);
* all-pairs (X1 == X2, BASELINE configs[4]): forward bounds of EVERY doc
  against the local docs as queries, C_r = D1[:, S_r] -- Phase 1 is then
  v_e(all) x H(local), so the dominant work divides by the world size (the
  other orientation, local rows against all queries, keeps v_e(local) ~ v_e and
  does not scale) -- one all_to_all of C_r's contiguous row blocks, the
  max-combine with the own block transposed into the local output rows, local
  top-k, gather (``sharded_all_pairs_topk``).  Results are identical for any world size: every
  pair distance is computed by the same arithmetic, and the merge is exact.

The collective glue (``allgather_slices``, ``gather_candidates``) is
device-agnostic so it is exercised with the gloo backend on CPU in
tests/test_parallel_gloo.py; the compute steps are the CUDA kernels.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import device
from .device import DeviceCSR, PreparedEmbeddings


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of ``rank``."""
    return n * rank // world, n * (rank + 1) // world


def vocab_slice(V: int, rank: int, world: int) -> tuple[int, int, int]:
    """(v0, v1, R): this rank's vocabulary rows and the padded slice height."""
    R = (V + world - 1) // world
    v0 = min(V, rank * R)
    return v0, min(V, v0 + R), R


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def allgather_slices(local: torch.Tensor, group=None) -> torch.Tensor:
    """[world, *local.shape] from equal-shaped per-rank slices: one
    ``all_gather_into_tensor`` into a contiguous buffer (ncclAllGather on NCCL; the same
    call runs on gloo in tests/test_parallel_gloo.py), issued whenever a process group
    is initialised, world 1 included."""
    if not (dist.is_available() and dist.is_initialized()):
        return local.unsqueeze(0)
    world = dist.get_world_size(group)
    out = torch.empty((world, *local.shape), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out.view(-1), local.contiguous().view(-1), group=group)
    return out


def exchange_blocks(C: torch.Tensor, sizes: list[int], group=None) -> list[torch.Tensor]:
    """All-pairs exchange (BASELINE configs[4]): this rank holds the forward
    bounds of ALL docs against its own docs, C = D1[:, S_r] (n, n_r) row-major; rank s
    needs the row block C[S_s] = D1[S_s, S_r] (contiguous, no packing).  One
    all_to_all; returns the blocks received from every rank s, each (n_r, n_s) =
    D1[S_r, S_s] (rank s's C rows for our docs)."""
    rank, world = _world()
    n_r = int(C.shape[1])
    offs = [0]
    for sz in sizes:
        offs.append(offs[-1] + sz)
    if world == 1:
        return [C[offs[0]:offs[1]]]
    send = C.contiguous().view(-1)
    my = sizes[rank]
    recv = torch.empty(sum(sz * my for sz in sizes), dtype=C.dtype, device=C.device)
    dist.all_to_all_single(recv, send, output_split_sizes=[my * sz for sz in sizes],
                           input_split_sizes=[sz * n_r for sz in sizes], group=group)
    out, at = [], 0
    for sz in sizes:
        out.append(recv[at:at + my * sz].view(my, sz))
        at += my * sz
    return out


def gather_candidates(d: torch.Tensor, i: torch.Tensor, group=None):
    """Gather per-rank (n_q, k) top-k lists to rank 0 as (n_q, world * k); None elsewhere.
    The gather is issued whenever a process group is initialised (world 1 included)."""
    if not (dist.is_available() and dist.is_initialized()):
        return d, i
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    gd = [torch.empty_like(d) for _ in range(world)] if rank == 0 else None
    gi = [torch.empty_like(i) for _ in range(world)] if rank == 0 else None
    dist.gather(d.contiguous(), gd, dst=0, group=group)
    dist.gather(i.contiguous(), gi, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat(gd, dim=1).contiguous(), torch.cat(gi, dim=1).contiguous()


# ---------------------------------------------------------------------------
# CUDA pipeline
# ---------------------------------------------------------------------------

def z1_slice(dx2: DeviceCSR, prep: PreparedEmbeddings, rank: int, world: int,
             near: "device.NearPairs | None" = None) -> tuple[torch.Tensor, int]:
    """This rank's forward Phase-1 slice: Z1 rows [v0, v1) as (panels, R, W), zero padded,
    W = 1 << device.spmm_z_shift(n_q) segments per panel.  ``near``: the near word pairs
    of dx2's query side (device.QuerySide), refining the slice's near entries (and built
    by it when it marks any)."""
    n_q = dx2.n_rows
    v0, v1, R = vocab_slice(prep.V, rank, world)
    rows = v1 - v0
    dev = dx2.cols.device
    zs = device.spmm_z_shift(n_q)
    W = 1 << zs
    panels = (n_q + W - 1) // W
    zl = torch.zeros((panels, R, W), dtype=torch.float32, device=dev)
    if rows > 0:
        B, _ = device.gather_rows(prep, dx2.cols, "B")
        Z, zp = device.phase1(prep.EhA[v0:v1], prep.norms[v0:v1], rows, B, dx2.nnz, dx2.offsets, n_q, prep,
                              z_shift=zs)
        remap = torch.full((prep.V,), -1, dtype=torch.int32, device=dev)
        remap[v0:v1] = torch.arange(rows, dtype=torch.int32, device=dev)
        rep, nxt = prep.representatives(dx2.cols)
        device.zero_identical(dx2.offsets, n_q, rep, nxt, remap, Z, zp, zs)
        a_ids = torch.arange(v0, v1, dtype=torch.int32, device=dev)
        if near is None:
            device.refine_near(Z, zp, zs, rows, n_q, dx2.offsets, dx2.cols, a_ids, prep.norms[v0:v1], prep)
        else:
            near.forward(Z, zp, zs, rows, a_ids, prep.norms[v0:v1], remap, dx2.offsets, dx2.cols, n_q)
        zl[:, :rows, :] = Z.view(panels, rows, W)
    return zl, R


def d1_from_slices(dx1: DeviceCSR, zall: torch.Tensor, R: int, n_q: int) -> torch.Tensor:
    """Forward SpMM of the local shard against all-gathered slices [world][panels][R][W]."""
    n1 = dx1.n_rows
    W = zall.shape[-1]
    zs = W.bit_length() - 1
    panels = zall.shape[1]
    out = torch.empty(((n_q + 7) // 8) * 8 * max(n1, 1), dtype=torch.float32, device=zall.device)
    if n_q % 8:  # padding queries of the last panel (read 8 at a time by lcrw_reverse_panels)
        out[(n_q // 8) * 8 * max(n1, 1):].zero_()
    device.spmm(dx1.offsets, dx1.cols, dx1.vals, n1, zall, W * R, n_q, out, 8, 8 * n1,
                z_block_rows=R, z_block_stride=panels * R * W, z_shift=zs, dist=True)
    return out


def forward_d1(dx1: DeviceCSR, dx2: DeviceCSR, prep: PreparedEmbeddings, group=None,
               near: "device.NearPairs | None" = None) -> torch.Tensor:
    """D1 (panels, local docs) with Phase 1 split by vocabulary slice + Z1 all-gather."""
    rank, world = _world()
    zl, R = z1_slice(dx2, prep, rank, world, near)
    zall = allgather_slices(zl, group)  # [world][panels][R][W]
    return d1_from_slices(dx1, zall, R, dx2.n_rows)


def sharded_topk(dx1: DeviceCSR, doc_base: int, n1_total: int, dx2: DeviceCSR, prep: PreparedEmbeddings, k: int,
                 group=None):
    """Per-query top-k over all ranks' docs; (n_q, k) on rank 0, None elsewhere."""
    rank, world = _world()
    # the query side first: its near word pairs serve this rank's forward slice and reverse pass
    qside = device.QuerySide.build(dx2, prep, dx1.nnz) if dx2.n_rows <= device.QUERY_SLICE else None
    d1 = forward_d1(dx1, dx2, prep, group, qside.near if qside is not None else None)
    ld, li = device.symmetric(dx1, dx2, prep, k, d1=d1, id_offset=doc_base, prepared=qside)
    if ld.shape[1] < k:  # shard smaller than k: pad with sentinels so gather shapes agree
        pd = torch.full((ld.shape[0], k), float("inf"), dtype=ld.dtype, device=ld.device)
        pi = torch.full((li.shape[0], k), torch.iinfo(torch.int64).max, dtype=li.dtype, device=li.device)
        pd[:, : ld.shape[1]] = ld
        pi[:, : li.shape[1]] = li
        ld, li = pd, pi
    ld = ld.contiguous()
    li = li.contiguous()
    g = gather_candidates(ld, li, group)
    if g is None:
        return None
    cd, ci = g
    n_q = dx2.n_rows
    d, i = device.topk_rows(cd, ci, n_q, cd.shape[1], k)
    kk = min(k, n1_total)
    return d[:, :kk], i[:, :kk]


def sharded_topk_host(x1_shard, doc_base: int, n1_total: int, x2, E, k: int, group=None):
    """End-to-end variant from host arrays (pinned for async copies)."""
    prep = PreparedEmbeddings(E)
    out = sharded_topk(DeviceCSR.upload(x1_shard, "x1"), doc_base, n1_total, DeviceCSR.upload(x2, "x2"), prep, k,
                       group)
    if out is None:
        return None
    return out[0].cpu().numpy(), out[1].cpu().numpy()


def sharded_all_pairs_topk(dx_local: DeviceCSR, dx_all: DeviceCSR, lo: int, prep: PreparedEmbeddings, k: int,
                           batch: int = 4096, group=None):
    """All-pairs symmetric top-k with docs sharded over ranks (BASELINE configs[4]):
    C = D1[:, S_r], the forward bounds of every doc against the local docs as queries
    (in ``batch``-query passes), one all_to_all of C's row blocks, then
    D[S_r, S_s] = max(D1[S_r, S_s] received, C[S_s]^T) into the local output rows,
    per-row top-k with global ids, gathered to rank 0 as (n, k); None elsewhere."""
    rank, world = _world()
    n = dx_all.n_rows
    sizes = [hi_ - lo_ for lo_, hi_ in (shard_range(n, r, world) for r in range(world))]
    n_r = dx_local.n_rows
    C = torch.empty((n, max(n_r, 1)), dtype=torch.float32, device=dx_all.cols.device)
    if n_r:
        device.forward_rows_into(device.Restricted.build(dx_all, prep), prep, dx_local, C, batch)
    if world == 1:  # C is D1 itself: symmetrise in place
        device._lib.call("lcrw_symmetrize_max", device._p(C), n, n, device._stream())
        D = C
    else:
        blocks = exchange_blocks(C[:, :n_r], sizes, group)
        D = torch.empty((max(n_r, 1), n), dtype=torch.float32, device=C.device)
        at = 0
        for s, sz in enumerate(sizes):
            if n_r and sz:
                device.max_transposed_into(D[:n_r, at:at + sz], blocks[s], C[at:at + sz, :n_r])
            at += sz
        del C, blocks
    kk = min(k, n)
    od = torch.empty((max(n_r, 1), k), dtype=torch.float32, device=D.device)
    oi = torch.empty((max(n_r, 1), k), dtype=torch.int64, device=D.device)
    device.topk_matrix_rows(D, n_r, n, n, 0, k, od, oi)
    od, oi = od[:n_r, :kk].contiguous(), oi[:n_r, :kk].contiguous()
    if world == 1:
        return od, oi
    return gather_rows_uneven(od, oi, sizes, group)


def gather_rows_uneven(d: torch.Tensor, i: torch.Tensor, sizes: list[int], group=None):
    """Gather per-rank (sizes[r], k) row blocks to rank 0 as one (sum(sizes), k) pair; None
    elsewhere.  gather needs equal shapes on every rank, so each block is padded to
    max(sizes) rows and rank 0 trims the padding."""
    rank, world = _world()
    mx = max(sizes) if sizes else 0
    k = int(d.shape[1])

    def padded(t, fill):
        if t.shape[0] == mx:
            return t.contiguous()
        out = torch.full((mx, k), fill, dtype=t.dtype, device=t.device)
        out[: t.shape[0]] = t
        return out

    pd = padded(d, float("inf"))
    pi = padded(i, -1)
    gd = [torch.empty_like(pd) for _ in range(world)] if rank == 0 else None
    gi = [torch.empty_like(pi) for _ in range(world)] if rank == 0 else None
    dist.gather(pd, gd, dst=0, group=group)
    dist.gather(pi, gi, dst=0, group=group)
    if rank != 0:
        return None
    return (torch.cat([g[:sz] for g, sz in zip(gd, sizes)]), torch.cat([g[:sz] for g, sz in zip(gi, sizes)]))
