"""Multi-rank host logic on CPU (gloo, world_size 2): vocabulary-slice all-gather
of Z1, blocked Z addressing, per-shard top-k gather + merge == global top-k
(partition invariance).  Compute steps use the CPU oracle as the
stand-in for the CUDA kernels; the collective code is the product's."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _panels(z: np.ndarray, R: int) -> np.ndarray:
    """(rows, n_q) -> (panels, R, 8) zero padded, the per-rank slice layout."""
    rows, nq = z.shape
    P = (nq + 7) // 8
    out = np.zeros((P, R, 8), np.float32)
    zz = np.zeros((rows, P * 8), np.float32)
    zz[:, :nq] = z
    out[:, :rows, :] = zz.reshape(rows, P, 8).transpose(1, 0, 2)
    return out


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import lcrwmd_oracle as O
        from paper_1711_07227_b200 import parallel, synthetic as S

        V, k = 900, 4
        E = S.embeddings(V, 24, seed=1)
        x1 = S.histograms(150, V, 12, seed=2)
        x2 = S.histograms(11, V, 12, seed=3)
        # --- Z1 vocabulary slice, all-gather, blocked addressing
        v0, v1, R = parallel.vocab_slice(V, rank, world)
        t = E[x2.column_ids]
        zfull = O.phase1(E, t, x2.row_offsets)  # (V, n_q)
        zl = torch.from_numpy(_panels(zfull[v0:v1], R))
        zall = parallel.allgather_slices(zl).numpy()  # [world][P][R][8]
        for w in range(V):
            b, r = divmod(w, R)
            got = zall[b, :, r, :].reshape(-1)[: x2.n_rows]
            assert np.array_equal(got, zfull[w]), w
        # --- docs sharded; local symmetric top-k with global ids; gather + merge
        lo, hi = parallel.shard_range(x1.n_rows, rank, world)
        full = O.lcrwmd_full(x1, x2, E)
        d_loc, i_loc = O.topk_per_query(full[lo:hi], k)
        d_t = torch.from_numpy(np.ascontiguousarray(d_loc))
        i_t = torch.from_numpy(np.ascontiguousarray(i_loc + lo))
        g = parallel.gather_candidates(d_t, i_t)
        if rank == 0:
            cd, ci = (x.numpy() for x in g)
            want_d, want_i = O.topk_per_query(full, k)
            for j in range(x2.n_rows):
                md, mi = O.topk_select(cd[j], ci[j], k)
                assert np.array_equal(md, want_d[j]) and np.array_equal(mi, want_i[j]), j
        else:
            assert g is None
        # --- all-pairs (X1 == X2): this rank holds C = D1[:, S_r] (every doc against its
        # docs as queries); one all_to_all of C's row blocks; max(received, C[S_s]^T)
        # over this rank's rows equals the symmetric all-pairs matrix
        n = 23
        sizes = [hi_ - lo_ for lo_, hi_ in (parallel.shard_range(n, r, world) for r in range(world))]
        xa = S.histograms(n, V, 12, seed=5)
        D1 = O.lcrwmd_batched(xa, xa, E)  # forward bounds (n, n)
        a0, a1 = parallel.shard_range(n, rank, world)
        mine = torch.from_numpy(np.ascontiguousarray(D1[:, a0:a1]))
        blocks = parallel.exchange_blocks(mine, sizes)
        for s_ in range(world):
            b0, b1 = parallel.shard_range(n, s_, world)
            assert np.array_equal(blocks[s_].numpy(), D1[a0:a1, b0:b1]), s_
        sym = np.maximum(D1, D1.T)
        got = np.concatenate([np.maximum(blocks[s_].numpy(), mine.numpy()[slice(*parallel.shard_range(n, s_, world))].T)
                              for s_ in range(world)], axis=1)
        assert np.array_equal(got, sym[a0:a1])
        assert np.allclose(sym, O.lcrwmd_full(xa, xa, E), rtol=1e-6, atol=1e-7)
        # uneven per-rank row blocks (n = 23 over 2 ranks: 11 + 12) gathered to rank 0
        # (sharded_all_pairs_topk's final step): padded to equal shapes, trimmed on rank 0
        kk = 4
        rows_d = np.sort(sym[a0:a1], axis=1)[:, :kk].astype(np.float32)
        rows_i = np.tile(np.arange(kk, dtype=np.int64), (a1 - a0, 1)) + a0
        g = parallel.gather_rows_uneven(torch.from_numpy(rows_d), torch.from_numpy(rows_i), sizes)
        if rank == 0:
            gd, gi = (x.numpy() for x in g)
            assert gd.shape == (n, kk) and np.array_equal(gd, np.sort(sym, axis=1)[:, :kk].astype(np.float32))
            want_i = np.concatenate([np.tile(np.arange(kk), (sz, 1)) + lo_ for sz, (lo_, _) in
                                     zip(sizes, (parallel.shard_range(n, r, world) for r in range(world)))])
            assert np.array_equal(gi, want_i)
        else:
            assert g is None
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_sharded_glue_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", f"rank {r}:\n{msg}"


def test_shard_ranges_partition():
    from paper_1711_07227_b200 import parallel
    for n in (0, 1, 7, 1000):
        for w in (1, 2, 3, 8):
            rs = [parallel.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            vs = [parallel.vocab_slice(n, r, w) for r in range(w)]
            assert sum(v1 - v0 for v0, v1, _ in vs) == n
