"""Multi-GPU row-panel orchestration (paper_1405_7470_b200/dist.py) exercised on
CPU with the gloo backend, world_size 2 and 3: panel / K-chunk arithmetic, the
chunked broadcast of B's K-row chunks from their owners, the per-chunk arrival
signal issued after each chunk's broadcast and in chunk order, and concatenated
panels equal to the full product.  The product itself is the float64 oracle
(test infrastructure) -- the CUDA kernels and the gated product are covered by
the GPU tests (tests/test_gated_gpu.py); here only the host-side logic is."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1405_7470_b200.dist import (check_kchunks, choose_kchunks, chunk_owner, gemm_rowpanel, kchunk_bounds,
                                       owned_chunks, panel_bounds, panel_opts)


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


def test_kchunk_bounds_cover_k_with_equal_chunks():
    for K in (1, 31, 32, 33, 777, 1000, 4096, 8192):
        for c in (1, 2, 3, 4, 8, 16, 64):
            b = kchunk_bounds(K, c)
            assert b[0][0] == 0 and b[-1][1] == K
            assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
            assert len(b) <= max(1, c)
            w = check_kchunks(b, K)                     # equal widths, >= 32, multiple of 32
            assert w >= 32 and (len(b) == 1 or w % 32 == 0)
    assert kchunk_bounds(8192, 16)[1] == (512, 1024)
    assert kchunk_bounds(0, 4) == []
    with pytest.raises(ValueError):
        check_kchunks([(0, 16), (16, 32)], 32)         # below the gate's 32-row minimum
    with pytest.raises(ValueError):
        check_kchunks([(0, 64), (64, 96), (96, 192)], 192)   # unequal widths


def test_chunk_policy_and_ownership():
    assert choose_kchunks(1024, 8192, "3xtf32") == 16
    assert choose_kchunks(1024, 8192, "ffma") == 8
    assert choose_kchunks(1024, 300, "3xtf32") == 1
    assert [chunk_owner(c, 4) for c in range(6)] == [0] * 6
    assert [chunk_owner(c, 4, owners=True) for c in range(6)] == [0, 1, 2, 3, 0, 1]
    # every chunk has exactly one owner; owners spread them evenly
    for g in (1, 2, 3, 8):
        for owners in (False, True):
            got = sorted(c for r in range(g) for c in owned_chunks(16, g, r, 0, owners))
            assert got == list(range(16))
    assert owned_chunks(16, 8, 0, owners=True) == [0, 8]       # 1/8 of B per rank
    o = panel_opts(148)
    assert o.plan_sms == 140 and o.num_ctas == 0 and list(o.reserved) == [0, 0, 0]


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
        Bfull = torch.from_numpy(synth.matrix(K, N, seed=3, matrix_id=1))
        bounds = kchunk_bounds(K, chunks)
        B = torch.full((K, N), float("nan"))
        for c in owned_chunks(len(bounds), world, rank, 0, owners):
            k0, k1 = bounds[c]
            B[k0:k1] = Bfull[k0:k1]
        events = []

        def signal_fn(c, k0, k1):
            # the chunk has arrived when its flag is raised
            events.append((c, bool(torch.isnan(B[k0:k1]).any())))

        def gemm_fn(a, b, c, _gate):
            m, k = a.shape
            n = b.shape[1]
            ref, _ = oracle.gemm(m, n, k, a.contiguous().numpy().reshape(-1), k, 0,
                                 b.contiguous().numpy().reshape(-1), n, 0)
            c.copy_(torch.from_numpy(ref.astype(np.float32)))

        C, info = gemm_rowpanel(A, B, chunks=chunks, owners=owners, gemm_fn=gemm_fn, signal_fn=signal_fn)
        assert info["chunks"] == len(bounds)
        q.put(("ok", rank, bool(torch.equal(B, Bfull)), events, C.numpy()))
    except Exception as e:   # surface worker failures to the parent
        q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,N,K,chunks,owners", [(2, 256, 384, 96, 3, False), (3, 200, 300, 64, 2, False),
                                                       (2, 130, 128, 33, 1, False), (3, 256, 200, 160, 5, True),
                                                       (2, 300, 100, 130, 4, True)])
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
    nb = len(kchunk_bounds(K, chunks))
    panels = {}
    for _, rank, b_ok, events, C in results:
        assert b_ok, f"rank {rank}: B incomplete after the broadcast"
        assert [c for c, _ in events] == list(range(nb)), "chunks signalled out of order"
        assert not any(nan for _, nan in events), "a chunk was signalled before it arrived"
        panels[rank] = C
    C = np.concatenate([panels[r] for r in range(world)], axis=0)
    assert np.array_equal(C, Cref.astype(np.float32))
