"""GPU parity of the K-gated product (lpy_gemm_f32_gated, include/lpy.h) and of
the CUDA branch of the row-panel step (paper_1405_7470_b200/dist.py) against
the float64 oracle, plus the gate's own contract:

  * with every flag already raised the gated product is BITWISE the ungated
    one with the same opts (the gate moves reads in time, not arithmetic);
  * operands that arrive late are read only after their chunk's flag: B starts
    as NaN and each K-row chunk is written, then signalled, by a second stream
    after a device-side delay -- any early read would poison C;
  * a flag that never comes traps the kernel after timeout_ms (the deadlock
    detector), in a child process so this process's context survives;
  * gemm_rowpanel on a world-1 NCCL group (broadcast in K-row chunks, the
    signal kernel, the gated product on a plan of num_sms - dist.default_reserve) matches the
    oracle element by element and the ungated product bitwise, for chunk
    counts 2 / 8 / 16, every bcast mode, both paths; the host-buffer step
    (gemm_rowpanel_host) gives the same bits, with its PCIe byte accounting.
"""
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

import oracle
import paper_1405_7470_b200 as lpy
import synth
from gpu_util import TOL, check
from paper_1405_7470_b200 import dist as ldist

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(M, N, K, seed=0):
    return (synth.matrix(M, K, seed=seed, matrix_id=synth.MATRIX_A),
            synth.matrix(K, N, seed=seed, matrix_id=synth.MATRIX_B))


def _opts(plan):
    o = lpy.GemmOpts()
    o.plan_sms = plan
    return o


def _sms():
    return torch.cuda.get_device_properties(0).multi_processor_count


@pytest.mark.parametrize("path", ["ffma", "3xtf32"])
@pytest.mark.parametrize("M,N,K,chunk_k", [(1024, 2048, 2048, 256), (300, 500, 780, 32), (256, 8192, 4096, 512),
                                           (1000, 3000, 776, 100)])
def test_gated_ready_flags_bitwise_ungated(path, M, N, K, chunk_k):
    A, B = _inputs(M, N, K, seed=5)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    plan = _sms() - 8
    nflags = -(-K // chunk_k)
    flags = torch.full((nflags,), 7, dtype=torch.int32, device="cuda")
    ref = lpy.gemm(dA, dB, path=path, opts=_opts(plan))
    for epoch in (7, 5, 0xFFFFFFF9):          # 7 - 0xFFFFFFF9 wraps to 14 >= 0: ready
        got = lpy.gemm(dA, dB, path=path, opts=_opts(plan), gate=lpy.KGate(flags.data_ptr(), chunk_k, epoch, 0))
        torch.cuda.synchronize()
        assert torch.equal(got, ref), f"gated product differs (epoch {epoch:#x})"
    check(ref.cpu().numpy(), A, B)


@pytest.mark.parametrize("path", ["ffma", "3xtf32"])
@pytest.mark.parametrize("M,N,K,chunk_k", [(4, 4, 40, 32), (1, 8, 64, 32), (128, 4, 96, 32), (200, 300, 48, 4096),
                                           (257, 132, 4100, 64)])
def test_gated_edge_shapes(path, M, N, K, chunk_k):
    """Gate edges: a short last chunk (K = 40 over 32-row chunks), one chunk
    longer than K, a single-row and a 4-column product (16-byte rows: a gated
    operand cannot go through the repack), and many small chunks
    over a K that is not a multiple of the k-block -- the flags are raised one
    by one from a second stream after a delay; bitwise the ungated product."""
    A, B = _inputs(M, N, K, seed=17)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    nflags = -(-K // chunk_k)
    flags = torch.zeros(nflags, dtype=torch.int32, device="cuda")
    plan = _sms() - 8
    side = torch.cuda.Stream()
    torch.cuda._sleep(1)
    torch.cuda.synchronize()
    out = lpy.gemm(dA, dB, path=path, opts=_opts(plan), gate=lpy.KGate(flags.data_ptr(), chunk_k, 3, 0))
    with torch.cuda.stream(side):
        torch.cuda._sleep(2_000_000)
        for c in range(nflags):
            lpy.kgate_signal(flags, c, 3, stream=side)
    ref = lpy.gemm(dA, dB, path=path, opts=_opts(plan))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    check(out.cpu().numpy(), A, B)


@pytest.mark.parametrize("path", ["ffma", "3xtf32"])
@pytest.mark.parametrize("la,lb,lc", [(1, 0, 0), (0, 1, 0), (1, 1, 1), (0, 0, 1)])
def test_gated_layouts_bitwise_ungated(path, la, lb, lc):
    """The gate is on k, which every layout and the column-major-C swap
    (C^T = B^T A^T) keep: any layout of A, B, C gives the ungated bits."""
    M, N, K, chunk_k = 1000, 1100, 1024, 128
    A, B = _inputs(M, N, K, seed=8)
    dA = torch.from_numpy(A).cuda() if la == 0 else torch.from_numpy(A.T.copy()).cuda().t()
    dB = torch.from_numpy(B).cuda() if lb == 0 else torch.from_numpy(B.T.copy()).cuda().t()
    def new_out():   # (a column-major C is the transposed problem: compare like with like)
        return torch.empty((M, N), device="cuda") if lc == 0 else torch.empty((N, M), device="cuda").t()
    out, ref = new_out(), new_out()
    flags = torch.ones(K // chunk_k, dtype=torch.int32, device="cuda")
    plan = _sms() - 8
    lpy.gemm(dA, dB, out=out, path=path, opts=_opts(plan), gate=lpy.KGate(flags.data_ptr(), chunk_k, 1, 0))
    lpy.gemm(dA, dB, out=ref, path=path, opts=_opts(plan))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    check(out.cpu().numpy(), A, B)


@pytest.mark.parametrize("path", ["ffma", "3xtf32"])
@pytest.mark.parametrize("lc", [0, 1])
def test_gate_orders_reads_after_arrival(path, lc):
    """B is NaN until a second stream writes chunk c and raises flags[c]
    after a ~20 ms device-side delay; the product must see only arrived data."""
    M, N, K, chunk_k = 512, 1024, 2048, 256
    A, B = _inputs(M, N, K, seed=9)
    dA = torch.from_numpy(A).cuda()
    src = torch.from_numpy(B).cuda()
    dB = torch.full_like(src, float("nan"))
    flags = torch.zeros(K // chunk_k, dtype=torch.int32, device="cuda")
    out = torch.empty((M, N), dtype=torch.float32, device="cuda") if lc == 0 else \
        torch.empty((N, M), dtype=torch.float32, device="cuda").t()
    side = torch.cuda.Stream()
    # load torch's spin kernel now: its first launch (lazy module loading)
    # would wait for the device, i.e. for the product spinning on its flags
    torch.cuda._sleep(1)
    torch.cuda.synchronize()
    lpy.gemm(dA, dB, out=out, path=path, opts=_opts(_sms() - 8),
             gate=lpy.KGate(flags.data_ptr(), chunk_k, 1, 0))
    with torch.cuda.stream(side):
        torch.cuda._sleep(40_000_000)          # ~20 ms at 1.9 GHz: the product is waiting by then
        for c in range(K // chunk_k):
            dB[c * chunk_k:(c + 1) * chunk_k].copy_(src[c * chunk_k:(c + 1) * chunk_k])
            lpy.kgate_signal(flags, c, 1, stream=side)
    torch.cuda.synchronize()
    C = out.cpu().numpy()
    assert np.isfinite(C).all(), "the product read B before its chunk arrived"
    check(C, A, B)


def test_gate_timeout_traps_in_child():
    code = textwrap.dedent(f"""
        import sys, torch
        sys.path.insert(0, {ROOT!r})
        import paper_1405_7470_b200 as lpy
        A = torch.rand(256, 512, device="cuda"); B = torch.rand(512, 256, device="cuda")
        flags = torch.zeros(4, dtype=torch.int32, device="cuda")
        o = lpy.GemmOpts(); o.plan_sms = 64
        lpy.gemm(A, B, path="3xtf32", opts=o, gate=lpy.KGate(flags.data_ptr(), 128, 1, 300))
        try:
            torch.cuda.synchronize()
        except Exception as e:
            print("TRAPPED", type(e).__name__, str(e).splitlines()[0]); sys.exit(0)
        print("NO_TRAP"); sys.exit(1)
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert "TRAPPED" in r.stdout, (r.stdout, r.stderr[-2000:])


def test_gated_validation_on_device():
    A = torch.rand(64, 64, device="cuda")
    B = torch.rand(64, 64, device="cuda")
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    gate = lpy.KGate(flags.data_ptr(), 32, 1, 0)
    # an operand that would need the aligned repack cannot be gated
    Ab = torch.rand(64 * 65 + 1, device="cuda")[1:].view(64, 65)[:, :64]
    with pytest.raises(lpy.LpyError, match="NOT_SUPPORTED"):
        lpy.gemm(Ab, B, gate=gate)
    with pytest.raises(lpy.LpyError, match="INVALID_VALUE"):
        lpy.gemm(A, B, opts=_opts(_sms() + 1))
    with pytest.raises(lpy.LpyError, match="MISALIGNED"):
        lpy.gemm(A, B, gate=lpy.KGate(flags.data_ptr() + 2, 32, 1, 0))
    assert lpy.lpy_kgate_signal(0, 1, None) == 3        # NULL flag
    assert lpy.lpy_kgate_signal(flags.data_ptr() + 1, 1, None) == 4


@pytest.fixture(scope="module", autouse=True)
def _destroy_world1_group():
    """Tear down the world-1 NCCL group the row-panel tests create."""
    yield
    import torch.distributed as dist
    if dist.is_initialized():
        torch.cuda.synchronize()
        ldist._state.clear()        # cached communicators / streams of the group being destroyed
        dist.destroy_process_group()


def _world1():
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


def _sampled_cols(N, tile=256):
    # every output-tile boundary column across the whole of j, and j = N - 1
    edges = sorted({c for t in range(0, N, tile) for c in (t, t + tile - 1) if c < N} | {N - 1})
    return np.array(edges)


@pytest.mark.parametrize("path", ["3xtf32", "ffma"])
@pytest.mark.parametrize("chunks,mode", [(2, "root"), (8, "owners"), (16, "allgather")])
def test_rowpanel_cuda_world1(path, chunks, mode):
    dist = _world1()
    M, N, K = 1024, 2048, 4096                    # a g=8 panel of n = 8192 in miniature
    A, B = _inputs(M, N, K, seed=11)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C, info = ldist.gemm_rowpanel(dA, dB, chunks=chunks, path=path, bcast=mode)
    assert info["chunks"] == chunks and info["total_ms"] > 0 and info["bcast_ms"] > 0
    # bitwise the ungated product planned for the same SMs
    ref = lpy.gemm(dA, dB, path=path, opts=ldist.panel_opts(_sms(), ldist.default_reserve(path)))
    torch.cuda.synchronize()
    assert torch.equal(C, ref)
    # B survived its (world-1) broadcast
    assert torch.equal(dB.cpu(), torch.from_numpy(B))
    # element-wise against the oracle on sampled rows x every tile-boundary column
    rows = np.array(sorted({0, 1, 127, 128, 255, 256, 511, 512, 767, 1023}))
    cols = _sampled_cols(N)
    ii, jj = np.meshgrid(rows, cols, indexing="ij")
    Cref, D = oracle.gemm_elems(M, N, K, A.reshape(-1), K, 0, B.reshape(-1), N, 0, ii.reshape(-1), jj.reshape(-1))
    err = oracle.normalized_error(C.cpu().numpy()[ii, jj].reshape(-1), Cref, D)
    assert err <= TOL
    # repeated steps raise the epoch and reuse the flags (no reset)
    for _ in range(3):
        C2, _ = ldist.gemm_rowpanel(dA, dB, chunks=chunks, path=path, bcast=mode, timings=False)
    torch.cuda.synchronize()
    assert torch.equal(C2, ref)


@pytest.mark.parametrize("path", ["3xtf32", "ffma"])
def test_rowpanel_host_world1_and_emulated(path):
    _world1()
    M, N, K = 1024, 2048, 4096
    A, B = _inputs(M, N, K, seed=12)
    hA = torch.from_numpy(A).pin_memory()
    hB = torch.from_numpy(B).pin_memory()
    hC = torch.empty((M, N), dtype=torch.float32).pin_memory()
    ws = ldist.HostWorkspace()
    info = ldist.gemm_rowpanel_host(hA, hB, hC, chunks=8, path=path, workspace=ws)
    ref = lpy.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), path=path,
                   opts=ldist.panel_opts(_sms(), ldist.default_reserve(path)))
    torch.cuda.synchronize()
    assert torch.equal(hC, ref.cpu())
    assert info["h2d_bytes"] == 4 * (M * K + K * N) and info["d2h_bytes"] == 4 * M * N
    # emulating rank 0 of 8: only its own chunks (0 of 8) cross PCIe, the rest
    # are taken as delivered (the workspace holds them from the call above)
    hC.fill_(float("nan"))
    info = ldist.gemm_rowpanel_host(hA, hB, hC, chunks=8, path=path, workspace=ws, emulate_world=8)
    assert info["h2d_bytes"] == 4 * (M * K + (K // 8) * N)
    assert torch.equal(hC, ref.cpu())


@pytest.mark.slow
@pytest.mark.parametrize("path", ["3xtf32", "ffma"])
def test_rowpanel_full_size_emulated_g8(path):
    """BASELINE config 4 at full size in the launch configuration bench.py
    times for N>1 (here rank 0 of an emulated 8-rank split on a world-1 NCCL
    group): the 1024 x 8192 x 8192 row panel through gemm_rowpanel (16 or 8
    K-row chunks, the gated product planned for num_sms - dist.default_reserve).  Sampled
    elements -- every 256-column tile boundary on the panel's first, middle
    and last rows, plus 2000 random ones -- against the oracle, and the whole
    panel bitwise the ungated product with the same plan."""
    _world1()
    n, rows = 8192, 1024
    A = synth.matrix(rows, n, seed=0, matrix_id=synth.MATRIX_A)
    B = synth.matrix(n, n, seed=0, matrix_id=synth.MATRIX_B)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C, info = ldist.gemm_rowpanel(dA, dB, path=path)
    ref = lpy.gemm(dA, dB, path=path, opts=ldist.panel_opts(_sms(), ldist.default_reserve(path)))
    torch.cuda.synchronize()
    assert torch.equal(C, ref)
    assert info["chunks"] == ldist.choose_kchunks(rows, n, path)
    rng = np.random.default_rng(1)
    cols = _sampled_cols(n)
    ii = np.concatenate([np.repeat([0, 511, rows - 1], cols.size), rng.integers(0, rows, 2000)])
    jj = np.concatenate([np.tile(cols, 3), rng.integers(0, n, 2000)])
    Cref, D = oracle.gemm_elems(rows, n, n, A.reshape(-1), n, 0, B.reshape(-1), n, 0, ii, jj)
    assert oracle.normalized_error(C.cpu().numpy()[ii, jj], Cref, D) <= TOL


@pytest.mark.parametrize("path", ["3xtf32", "ffma"])
def test_rowpanel_graph_replay(path):
    """dist.RowPanelGraph: the step captured as a CUDA graph (flag reset ->
    signals on one branch, the gated product spinning on them on the other)
    replays bitwise the eager step, and inputs changed in place between
    replays are picked up (the graph reads the same buffers)."""
    _world1()
    M, N, K = 1024, 2048, 4096
    A, B = _inputs(M, N, K, seed=13)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty((M, N), device="cuda")
    ref, _ = ldist.gemm_rowpanel(dA, dB, chunks=8, path=path)
    g = ldist.RowPanelGraph(dA, dB, out, chunks=8, path=path)
    for _ in range(3):
        out.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
    dA.mul_(-1.0)                                   # new inputs, same buffers: C must flip sign
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, -ref)
