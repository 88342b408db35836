"""Multi-GPU row-panel orchestration (paper_1405_7470_b200/dist.py) exercised on
CPU with the gloo backend, world_size 2 and 3: panel/chunk arithmetic, the
chunked broadcast of B from rank 0, per-block products written into disjoint
column blocks of C, and concatenated panels equal to the full product.  The
per-block product is the float64 oracle (test infrastructure) -- the CUDA
kernels are covered by the GPU tests; here only the host-side logic is."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1405_7470_b200.dist import (block_owner, chunk_bounds, chunk_grid, chunk_streams, choose_chunks,
                                       panel_bounds, rowpanel_gemm)


def test_panel_bounds_cover_rows_exactly():
    for M in (0, 1, 7, 8192, 1000, 1001):
        for g in (1, 2, 3, 4, 8):
            spans = [panel_bounds(M, g, r) for r in range(g)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
    assert panel_bounds(8192, 8, 3) == (3072, 4096)     # tile-aligned panels at n=8192
    with pytest.raises(ValueError):
        panel_bounds(10, 2, 2)


def test_chunk_bounds_aligned_and_covering():
    for N in (1, 127, 128, 1000, 3000, 8192):
        for c in (1, 2, 3, 4, 8, 64):
            b = chunk_bounds(N, c)
            assert b[0][0] == 0 and b[-1][1] == N
            assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
            assert all(c0 % 128 == 0 for c0, _ in b)
            assert len(b) <= max(1, c)
    assert chunk_bounds(8192, 4) == [(0, 2048), (2048, 4096), (4096, 6144), (6144, 8192)]
    assert chunk_bounds(0, 4) == []


def test_chunk_policy():
    # n = 8192 panels for g = 8 / 4 / 2 / 1 ranks
    assert [choose_chunks(8192 // g, 8192) for g in (8, 4, 2, 1)] == [8, 4, 2, 2]
    assert [chunk_streams(8192 // g, choose_chunks(8192 // g, 8192)) for g in (8, 4, 2, 1)] == [4, 2, 1, 1]
    assert choose_chunks(1024, 1000) == 1 and choose_chunks(1024, 0) == 1
    # grids sized to a block's own tiles, never beyond the chip
    assert chunk_grid(1024, 1024, 148, "3xtf32") == 32      # 16 pair tiles
    assert chunk_grid(8192, 8192, 148, "3xtf32") == 148
    assert chunk_grid(1024, 1024, 148, "ffma") == 32
    assert chunk_grid(1, 1, 148, "ffma") == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, N, K, chunks, q, owners=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    try:
        r0, r1 = panel_bounds(M, world, rank)
        A = torch.from_numpy(synth.matrix(r1 - r0, K, seed=3, matrix_id=0, row0=r0))
        bounds = chunk_bounds(N, chunks)
        blocks = []
        for c, (c0, c1) in enumerate(bounds):
            if rank == block_owner(c, world, 0, owners):
                blocks.append(torch.from_numpy(synth.matrix(K, c1 - c0, seed=3, matrix_id=1, col0=c0)))
            else:
                blocks.append(torch.full((K, c1 - c0), float("nan")))
        C = torch.full((r1 - r0, N), float("nan"))

        def gemm_fn(a, b, c):
            m, k = a.shape
            n = b.shape[1]
            ref, _ = oracle.gemm(m, n, k, a.contiguous().numpy().reshape(-1), k, 0,
                                 b.contiguous().numpy().reshape(-1), n, 0)
            c.copy_(torch.from_numpy(ref.astype(np.float32)))

        rowpanel_gemm(A, blocks, C, bounds, gemm_fn=gemm_fn, owners=owners)
        # every rank now holds all of B (the broadcast), and its panel of C
        B_full = torch.cat(blocks, dim=1)
        if rank == 0:
            q.put(("ok", B_full.numpy(), None, C.numpy()))
        else:
            q.put(("ok_rank", rank, bool(torch.isnan(B_full).any()), C.numpy()))
    except Exception as e:   # surface worker failures to the parent
        q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,N,K,chunks,owners", [(2, 256, 384, 96, 3, False), (3, 200, 300, 64, 2, False),
                                                       (2, 130, 128, 33, 1, False), (3, 256, 768, 40, 3, True),
                                                       (2, 300, 1024, 24, 4, True)])
def test_rowpanel_gloo(world, M, N, K, chunks, owners):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, chunks, q, owners)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    errs = [r for r in results if r[0] == "err"]
    assert not errs, errs
    A = synth.matrix(M, K, seed=3, matrix_id=0)
    B = synth.matrix(K, N, seed=3, matrix_id=1)
    Cref, _ = oracle.gemm(M, N, K, A.reshape(-1), K, 0, B.reshape(-1), N, 0)
    panels = {}
    for r in results:
        if r[0] == "ok":
            assert np.array_equal(r[1], B)                  # rank 0 kept B intact
            panels[0] = r[3]
        else:
            assert not r[2], "broadcast left NaNs in B on a receiving rank"
            panels[r[1]] = r[3]
    C = np.concatenate([panels[r] for r in range(world)], axis=0)
    assert np.array_equal(C, Cref.astype(np.float32))
