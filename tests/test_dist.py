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

from paper_1405_7470_b200.dist import (check_kchunks, choose_kchunks, chunk_owner, gemm_rowpanel, gemm_rowpanel_host,
                                       default_reserve, kchunk_bounds, owned_chunks, panel_bounds, panel_opts,
                                       transfers)


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
    assert choose_kchunks(1024, 8192, "3xtf32") == 8
    assert choose_kchunks(1024, 8192, "ffma") == 8
    assert choose_kchunks(1024, 300, "3xtf32") == 1
    assert [chunk_owner(c, 4) for c in range(6)] == [0] * 6
    assert [chunk_owner(c, 4, mode="owners") for c in range(6)] == [0, 1, 2, 3, 0, 1]
    assert [chunk_owner(c, 4, mode="allgather") for c in range(6)] == [0, 1, 2, 3, 0, 1]
    with pytest.raises(ValueError):
        chunk_owner(0, 4, mode="nvls")
    # every chunk has exactly one owner; owners spread them evenly
    for g in (1, 2, 3, 8):
        for mode in ("root", "owners", "allgather"):
            got = sorted(c for r in range(g) for c in owned_chunks(16, g, r, 0, mode))
            assert got == list(range(16))
    assert owned_chunks(16, 8, 0, mode="owners") == [0, 8]       # 1/8 of B per rank


def test_transfer_plan():
    b16 = kchunk_bounds(8192, 16)
    assert transfers(b16, 8, mode="root") == [("bcast", [c]) for c in range(16)]
    assert transfers(b16, 8, mode="allgather") == [("allgather", list(range(8))), ("allgather", list(range(8, 16)))]
    assert transfers(b16, 1, mode="allgather") == [("bcast", [c]) for c in range(16)]
    # a partial last round and a short last chunk fall back to broadcasts
    b5 = kchunk_bounds(160, 5)          # 5 chunks of 32
    assert transfers(b5, 2, mode="allgather") == [("allgather", [0, 1]), ("allgather", [2, 3]), ("bcast", [4])]
    b4 = kchunk_bounds(130, 4)          # widths 64, 64, 2 -> 3 chunks
    assert [w for w, _ in [(k1 - k0, 0) for k0, k1 in b4]] == [64, 64, 2]
    assert transfers(b4, 2, mode="allgather") == [("allgather", [0, 1]), ("bcast", [2])]
    # every chunk exactly once, in increasing order
    for g in (2, 3, 4):
        flat = [c for _, cs in transfers(kchunk_bounds(1000, 7), g, mode="allgather") for c in cs]
        assert flat == sorted(flat) == list(range(len(kchunk_bounds(1000, 7))))
    assert default_reserve("3xtf32") == 32 and default_reserve("ffma") == 8
    o = panel_opts(148, default_reserve("3xtf32"))
    assert o.plan_sms == 116 and o.num_ctas == 0 and list(o.reserved) == [0, 0, 0]
    assert panel_opts(148, 8).plan_sms == 140


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, N, K, chunks, q, mode="root"):
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
        for c in owned_chunks(len(bounds), world, rank, 0, mode):
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

        C, info = gemm_rowpanel(A, B, chunks=chunks, bcast=mode, gemm_fn=gemm_fn, signal_fn=signal_fn)
        assert info["chunks"] == len(bounds)
        q.put(("ok", rank, bool(torch.equal(B, Bfull)), events, C.numpy()))
    except Exception as e:   # surface worker failures to the parent
        q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,N,K,chunks,mode", [(2, 256, 384, 96, 3, "root"), (3, 200, 300, 64, 2, "root"),
                                                     (2, 130, 128, 33, 1, "root"), (3, 256, 200, 160, 5, "owners"),
                                                     (2, 300, 100, 130, 4, "owners"), (2, 256, 96, 256, 8, "allgather"),
                                                     (3, 200, 64, 224, 7, "allgather"), (2, 100, 50, 130, 4, "allgather")])
def test_rowpanel_gloo(world, M, N, K, chunks, mode):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, chunks, q, mode)) for r in range(world)]
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


def _host_worker(rank, world, port, M, N, K, chunks, q, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    try:
        r0, r1 = panel_bounds(M, world, rank)
        A = torch.from_numpy(synth.matrix(r1 - r0, K, seed=4, matrix_id=0, row0=r0))
        bounds = kchunk_bounds(K, chunks)
        # the host holds only this rank's chunks of B (the rest NaN): nothing else may be read
        B = torch.full((K, N), float("nan"))
        for c in owned_chunks(len(bounds), world, rank, 0, mode):
            k0, k1 = bounds[c]
            B[k0:k1] = torch.from_numpy(synth.matrix(k1 - k0, N, seed=4, matrix_id=1, row0=k0))
        C = torch.full((r1 - r0, N), float("nan"))

        def gemm_fn(a, b, c, _gate):
            m, k = a.shape
            n = b.shape[1]
            ref, _ = oracle.gemm(m, n, k, a.contiguous().numpy().reshape(-1), k, 0,
                                 b.contiguous().numpy().reshape(-1), n, 0)
            c.copy_(torch.from_numpy(ref.astype(np.float32)))

        info = gemm_rowpanel_host(A, B, C, chunks=chunks, bcast=mode, device="cpu", gemm_fn=gemm_fn)
        q.put(("ok", rank, info["h2d_bytes"], info["d2h_bytes"], bool(torch.isnan(info["B"]).any()), C.numpy()))
    except Exception as e:
        q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M,N,K,chunks,mode", [(2, 256, 96, 256, 8, "owners"), (3, 200, 64, 224, 7, "allgather"),
                                                     (2, 130, 50, 130, 4, "owners")])
def test_rowpanel_host_gloo(world, M, N, K, chunks, mode):
    """The host-buffer step (dist.gemm_rowpanel_host) planned on CPU under
    gloo: each rank "uploads" its A panel and only the chunks it owns -- its
    host B holds nothing else (NaN) -- the plan completes B everywhere, the
    panels concatenate to the oracle product, and the per-rank H2D bytes are
    4 (rows K + owned chunk rows N): 4 (M K + K N) over all ranks, B once."""
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, world, port, M, N, K, chunks, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    errs = [r for r in results if r[0] == "err"]
    assert not errs, errs
    A = synth.matrix(M, K, seed=4, matrix_id=0)
    B = synth.matrix(K, N, seed=4, matrix_id=1)
    Cref, _ = oracle.gemm(M, N, K, A.reshape(-1), K, 0, B.reshape(-1), N, 0)
    panels, h2d_total, d2h_total = {}, 0, 0
    for _, rank, h2d, d2h, nan_left, C in results:
        assert not nan_left, f"rank {rank}: B incomplete after the plan"
        panels[rank] = C
        h2d_total += h2d
        d2h_total += d2h
    C = np.concatenate([panels[r] for r in range(world)], axis=0)
    assert np.array_equal(C, Cref.astype(np.float32))
    assert h2d_total == 4 * (M * K + K * N) and d2h_total == 4 * M * N
