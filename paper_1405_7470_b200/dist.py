"""Multi-GPU row-panel product (BASELINE.json north_star).

C's rows are split into contiguous panels, one per rank (one process per GPU);
rank r owns rows [r*ceil(M/g), min(M, (r+1)*ceil(M/g))) of A and C
(reading A14).  Row panels are independent given the whole of B,
C[rows_r, :] = A[rows_r, :] B, so the only exchange is ONE broadcast of B
(4*K*N bytes) over NCCL / NVLink; C stays sharded.

The product is fused with its broadcast through the K-gate (include/lpy.h
lpy_gemm_f32_gated).  Every output tile walks k in order (the reduction
sum(k, a[i,k]*b[k,j])), so a tile needs the k-th rows of B only
when it reaches k.  B (row-major K x N) is therefore broadcast in chunks of
K ROWS -- each one contiguous in memory, so NCCL sends B itself, no re-blocking
copy -- and after each chunk's broadcast a signal kernel on the communication
stream publishes flags[c] = epoch.  ONE persistent product over the whole
panel (the paper's split_iname of the k loop into chunks, whose
prefetch waits for the chunk) runs at the same time on the caller's
stream and its TMA producers wait for each chunk's flag before loading it: the
first tiles start as soon as the first chunk has landed, and the panel is one
launch with one tile schedule (stream-K balanced over its SM share) instead of
per-block products that each under-fill the GPU.

Scheduling contract: the product spins on flags while it holds its SMs, so it
is planned for `num_sms - reserve_sms` SMs (opts.plan_sms), leaving the rest to
NCCL's collective kernels (capped at reserve_sms - 1 CTAs through the
communicator's maxCTAs, comm_group) and the signal kernel.

Pieces are injectable (`bcast_fn`, `gemm_fn`, `signal_fn`) so the orchestration
runs on CPU under gloo in the tests (tests/test_dist.py); on CUDA the defaults
are torch.distributed.broadcast and the library's gated product and signal.
"""
from __future__ import annotations

import math
import os
import threading

RESERVE_SMS = {"3xtf32": 32, "ffma": 8}   # SMs left to the collectives per path (profiles/r02_bcast_emul.txt)


def default_reserve(path: str) -> int:
    """SMs a rank's gated product leaves to the chunk collectives.  Measured on
    one GPU with each chunk moved through HBM by persistent CTAs on the free SMs
    (the per-rank work of a ring broadcast; profiles/r02_bcast_emul.txt): the
    3xTF32 panel (0.5 ms) is paced by those copies below ~32 SMs (step 0.78 /
    0.73 / 0.65 / 0.64 ms with 16 / 24 / 32 / 40), the FFMA panel (2.4 ms) by its
    own product (2.55 / 2.57 / 2.83 / 3.23 ms with 8 / 16 / 24 / 32)."""
    return RESERVE_SMS.get(path, 32)
FLAG_WORDS = 4096        # flag array per device (chunks per call <= this)


def panel_bounds(M: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of C owned by `rank` (contiguous panels of ceil(M/world))."""
    if world < 1 or not 0 <= rank < world or M < 0:
        raise ValueError("bad panel request")
    h = math.ceil(M / world) if M else 0
    r0 = min(M, rank * h)
    return r0, min(M, r0 + h)


def kchunk_bounds(K: int, chunks: int, align: int = 32) -> list[tuple[int, int]]:
    """K-row ranges [k0, k1) covering [0, K): `chunks` ranges (fewer if K is
    small) of equal length rounded up to a multiple of `align` (>= 32, the
    K-gate's minimum), the last one possibly shorter."""
    if K <= 0:
        return []
    chunks = max(1, min(chunks, math.ceil(K / align)))
    w = math.ceil(math.ceil(K / chunks) / align) * align
    out, k0 = [], 0
    while k0 < K:
        out.append((k0, min(K, k0 + w)))
        k0 += w
    return out


def choose_kchunks(rows: int, K: int, path: str) -> int:
    """Broadcast chunks of B for a rank's (rows x N) panel: enough that the
    first chunk (the wait before the first tiles start) is a small share of
    the step, few enough that the host's per-collective cost (a
    torch.distributed call is ~10-30 us of host time, enqueued one after
    another on the communication stream) stays well inside the broadcast it
    overlaps: 8 chunks (1024 rows, 33.5 MB at n = 8192: the first arrives in
    ~50 us at 700 GB/s, all 8 are enqueued within ~0.25 ms); never chunks
    shorter than 256 rows of K."""
    del rows, path
    return max(1, min(8, K // 256))


BCAST_MODES = ("root", "owners", "allgather")


def chunk_owner(c: int, world: int, root: int = 0, mode: str = "root") -> int:
    """Rank holding K-row chunk c of B before the step: `root` in mode "root"
    (north_star's broadcast of B), else c mod world -- B starts sharded by
    K-row chunks and every rank sends the chunks it holds ("owners": one NCCL
    broadcast per chunk from its owner; "allgather": one NCCL all-gather per
    round of `world` consecutive chunks, SURVEY 8(f)-3's all-gather from
    pre-sharded B, which NCCL can run as NVLS on NVSwitch).  Either way the send
    load -- and on the host-buffer path the PCIe upload -- is spread over all
    ranks."""
    if mode not in BCAST_MODES:
        raise ValueError(f"bcast mode {mode!r} not in {BCAST_MODES}")
    return root if mode == "root" else c % world


def owned_chunks(nchunks: int, world: int, rank: int, root: int = 0, mode: str = "root") -> list[int]:
    """The K-row chunks of B `rank` holds before the step (and, on the
    host-buffer path, uploads)."""
    return [c for c in range(nchunks) if chunk_owner(c, world, root, mode) == rank]


def transfers(bounds, world: int, root: int = 0, mode: str = "root") -> list[tuple[str, list[int]]]:
    """The communication plan of one step: ("bcast", [c]) broadcasts chunk c
    from its owner; ("allgather", [c0 .. c0+world-1]) all-gathers a round of
    `world` consecutive equal chunks, chunk c0+r coming from rank r, in place
    (the round's rows of B are contiguous and rank r's piece sits at offset r
    in them, as NCCL's in-place all-gather wants).  A round that would be
    partial, or hold a shorter last chunk, falls back to per-chunk broadcasts.
    Chunks are delivered in increasing order (the gate polls them in order)."""
    n = len(bounds)
    if mode != "allgather" or world == 1:
        return [("bcast", [c]) for c in range(n)]
    w = bounds[0][1] - bounds[0][0] if bounds else 0
    plan, c = [], 0
    while c < n:
        rnd = list(range(c, c + world))
        if rnd[-1] < n and all(bounds[x][1] - bounds[x][0] == w for x in rnd):
            plan.append(("allgather", rnd))
            c += world
        else:
            plan.append(("bcast", [c]))
            c += 1
    return plan


def check_kchunks(bounds, K: int) -> int:
    """Validate explicit chunk ranges (contiguous from 0 to K, equal lengths
    >= 32 except a shorter last one) and return the chunk length."""
    if not bounds:
        return 32
    if len(bounds) == 1 and bounds[0] == (0, K):
        return max(32, K)              # one chunk: all of K (the gate's chunk_k >= 32)
    w = bounds[0][1] - bounds[0][0]
    ok = w >= 32 and bounds[0][0] == 0 and bounds[-1][1] == K
    for i, (k0, k1) in enumerate(bounds):
        ok = ok and k0 == i * w and (k1 - k0 == w or (i == len(bounds) - 1 and 0 < k1 - k0 <= w))
    if not ok:
        raise ValueError(f"bad K chunks {bounds[:4]}... for K={K}")
    return w


class _Flags:
    """Per-device arrival flags (int32 words, compared as uint32 by the
    kernels) and the epoch counter: each call raises the epoch, so flags are
    never reset (lpy_kgate)."""

    def __init__(self, device):
        import torch
        self.flags = torch.zeros(FLAG_WORDS, dtype=torch.int32, device=device)
        self.epoch = 0
        self.warm = set()          # (group, plan kinds) whose kernels a step has already launched
        self.lock = threading.Lock()

    def next_epoch(self) -> int:
        with self.lock:
            self.epoch = (self.epoch + 1) & 0xFFFFFFFF or 1
            return self.epoch


_state: dict = {}


def _flags_for(device) -> _Flags:
    key = ("flags", str(device))
    if key not in _state:
        _state[key] = _Flags(device)
    return _state[key]


def _comm_stream(device):
    import torch
    key = ("comm", str(device))
    if key not in _state:
        _state[key] = torch.cuda.Stream(device=device)
    return _state[key]


def comm_group(reserve_sms: int, group=None):
    """The NCCL process group the chunk collectives run on: the ranks of
    `group` (default: all), with NCCL told to launch at most reserve_sms - 1
    CTAs per collective (ncclConfig maxCTAs) -- the SMs the gated product
    leaves, less one for the signal kernel -- so a collective never queues CTAs
    behind the spinning product.  Created once per (ranks, reserve): all ranks
    must reach the first call for a given reserve together (new_group is
    collective), as the row-panel step guarantees."""
    import torch.distributed as dist
    if dist.get_backend(group) != "nccl":
        return group
    ranks = tuple(dist.get_process_group_ranks(group)) if group is not None else tuple(range(dist.get_world_size()))
    key = ("comm_group", ranks, int(reserve_sms))
    if key not in _state:
        opts = dist.ProcessGroupNCCL.Options()
        opts.config.max_ctas = max(1, int(reserve_sms) - 1)
        opts.config.min_ctas = 1
        _state[key] = dist.new_group(ranks=list(ranks), backend="nccl", pg_options=opts)
    return _state[key]


def panel_opts(sms: int, reserve_sms: int = 32):
    """GemmOpts of the gated panel product: planned for the SMs the broadcast
    leaves it (results depend on plan_sms, never on the grid)."""
    from . import GemmOpts
    o = GemmOpts()
    o.plan_sms = max(2, sms - reserve_sms)
    return o


def gemm_rowpanel(A_panel, B, group=None, root=0, chunks=None, path="auto", out=None,
                  reserve_sms=None, bcast="root", broadcast=True, comm_stream=None,
                  timings=True, bcast_fn=None, gather_fn=None, gemm_fn=None, signal_fn=None,
                  before_chunk=None, flags=None, epoch=None):
    """One distributed product step on this rank: C_panel = A_panel @ B with B
    broadcast in K-row chunks while the gated product consumes them.

    A_panel : (rows_r, K) fp32, this rank's rows of A (row- or column-major).
    B       : (K, N) contiguous row-major fp32; its chunks are valid on their
              owner (chunk_owner: `root` with bcast="root", else c mod world)
              on entry and on every rank on exit.
    bcast   : "root" | "owners" | "allgather" (chunk_owner, transfers).
    reserve_sms: SMs the product leaves to the collectives (None: default_reserve
              of the path); on NCCL the collectives run on comm_group(reserve_sms),
              whose communicator launches at most reserve_sms - 1 CTAs.
    out     : optional (rows_r, N) fp32 output (row- or column-major).
    chunks  : number of K-row chunks (None: choose_kchunks) or explicit
              kchunk_bounds-style [(k0, k1), ...] ranges (each >= 32 rows but
              the last, equal lengths).
    before_chunk(c): optional hook run on the communication stream before
              chunk c's broadcast (the host-buffer step waits for the owner's
              upload there).
    flags, epoch: an explicit flag array (int32 CUDA tensor) and epoch instead
              of the device's shared ones (RowPanelGraph: a captured step resets
              its own flags and always uses epoch 1).
    Returns (C_panel, info): with timings=True (CUDA) the step is synchronised
    and info = {"bcast_ms": start -> last chunk broadcast, "gemm_ms": start ->
    product done, "total_ms": start -> both done, "chunks": n} (the two overlap:
    gemm_ms includes waiting for chunks); with timings=False info holds the
    start/bcast/gemm CUDA events instead and nothing is synchronised (the
    caller's stream is joined to all the work).  On CPU (gloo tests) the chunks
    are broadcast and signalled in order and then gemm_fn runs.
    """
    import torch
    import torch.distributed as dist

    if A_panel.dim() != 2 or B.dim() != 2 or A_panel.shape[1] != B.shape[0]:
        raise ValueError(f"shape mismatch {tuple(A_panel.shape)} @ {tuple(B.shape)}")
    if not B.is_contiguous():
        raise ValueError("B must be contiguous row-major: its K-row chunks are broadcast in place")
    rows, K = A_panel.shape
    N = B.shape[1]
    resolved = path
    if path == "auto" and A_panel.is_cuda:
        from . import PATH_AUTO, lpy_select_path
        _, ch = lpy_select_path(rows, N, K, PATH_AUTO)
        resolved = {1: "ffma", 2: "3xtf32"}[ch]
    if isinstance(chunks, (list, tuple)):
        bounds = [tuple(b) for b in chunks]
    else:
        bounds = kchunk_bounds(K, chunks or choose_kchunks(rows, K, resolved))
    chunk_k = check_kchunks(bounds, K)
    if len(bounds) > FLAG_WORDS:
        raise ValueError(f"at most {FLAG_WORDS} chunks")
    if reserve_sms is None:
        reserve_sms = default_reserve(resolved)
    if A_panel.is_cuda and broadcast and bcast_fn is None and gather_fn is None:
        group = comm_group(reserve_sms, group)
    world = dist.get_world_size(group) if broadcast else 1
    # a broadcast among one rank moves nothing: skipped (the chunks are still
    # signalled, so a world-1 step runs the same gated product)
    broadcast = broadcast and world > 1
    src = [chunk_owner(c, world, root, bcast) for c in range(len(bounds))]
    plan = transfers(bounds, world, root, bcast)
    if bcast_fn is None:
        def bcast_fn(t, s):
            dist.broadcast(t, src=s, group=group)
    if gather_fn is None:
        def gather_fn(out_rows, piece):
            dist.all_gather_into_tensor(out_rows, piece, group=group)
    rank = dist.get_rank(group) if broadcast else 0

    def run_plan(signal):
        for kind, cs in plan:
            if before_chunk is not None:
                for c in cs:
                    before_chunk(c)
            if broadcast and kind == "bcast":
                k0, k1 = bounds[cs[0]]
                bcast_fn(B[k0:k1], src[cs[0]])
            elif broadcast:
                k0, k1 = bounds[cs[0]][0], bounds[cs[-1]][1]
                p0, p1 = bounds[cs[rank]]
                gather_fn(B[k0:k1], B[p0:p1])
            for c in cs:
                signal(c)
    if out is None:
        out = torch.empty((rows, N), dtype=torch.float32, device=A_panel.device)

    if not A_panel.is_cuda:
        # CPU (gloo) path: the same sequence without overlap
        run_plan(lambda c: signal_fn(c, *bounds[c]) if signal_fn is not None else None)
        if gemm_fn is None:
            raise ValueError("CPU tensors need an injected gemm_fn (the product is CUDA-only)")
        gemm_fn(A_panel, B, out, None)
        return out, {"chunks": len(bounds)}

    from . import KGate, gemm as lpy_gemm, kgate_signal
    dev = A_panel.device
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fl = _flags_for(dev)
    flag_t = flags if flags is not None else fl.flags
    if epoch is None:
        epoch = fl.next_epoch()
    caller = torch.cuda.current_stream(dev)
    comm = comm_stream or _comm_stream(dev)
    capturing = torch.cuda.is_current_stream_capturing()
    ev = {k: torch.cuda.Event(enable_timing=not capturing) for k in ("start", "bcast", "gemm")}
    # fork the communication stream off the caller's work so far -- recorded
    # BEFORE the product is enqueued, so the chain never waits for the product
    ev["start"].record(caller)
    comm.wait_event(ev["start"])
    gate = KGate(flag_t.data_ptr(), chunk_k, epoch, 0)
    opts = panel_opts(sms, reserve_sms)

    def product():
        if gemm_fn is not None:
            gemm_fn(A_panel, B, out, (opts, gate))
        elif K > 0 and rows > 0 and N > 0:
            lpy_gemm(A_panel, B, out=out, path=path, opts=opts, gate=gate)
        elif rows > 0 and N > 0:
            lpy_gemm(A_panel, B, out=out, path=path)      # K == 0: C := 0, nothing to wait for
        ev["gemm"].record(caller)

    def chain():
        with torch.cuda.stream(comm):
            run_plan(lambda c: signal_fn(c, *bounds[c]) if signal_fn is not None
                     else kgate_signal(flag_t, c, epoch, stream=comm))
            ev["bcast"].record(comm)

    # Enqueue order.  The first step of a kind (group, collectives used) on a
    # device enqueues the whole chain first: every kernel it launches (NCCL's,
    # the signal) is then loaded before the
    # product spins (lazy module loading would otherwise block those first
    # launches behind it, include/lpy.h).  Later steps enqueue the product
    # first, so it is running -- its first tiles waiting on chunk 0 -- while
    # the host is still enqueuing the chain.
    # (LPY_DIST_CHAIN_FIRST=1 keeps the chain-first order on every step: a
    # profiler that serialises kernels -- ncu -- would otherwise run the product
    # alone while its flags are still pending, and its deadlock detector traps)
    key = (id(group), broadcast, tuple(sorted({kind for kind, _ in plan})), signal_fn is None)
    if key in fl.warm and os.environ.get("LPY_DIST_CHAIN_FIRST", "0") != "1" and not capturing:
        product()
        chain()
    else:
        chain()
        product()
        fl.warm.add(key)
    caller.wait_stream(comm)
    if not timings or capturing:
        return out, {"events": ev, "chunks": len(bounds)}
    torch.cuda.synchronize(dev)
    b = ev["start"].elapsed_time(ev["bcast"])
    g = ev["start"].elapsed_time(ev["gemm"])
    return out, {"bcast_ms": b, "gemm_ms": g, "total_ms": max(b, g), "chunks": len(bounds)}


class RowPanelGraph:
    """One row-panel step (gemm_rowpanel) captured as a CUDA graph and replayed:
    the chunk collectives, their signals and the gated product are enqueued by
    ONE graph launch instead of ~10-30 us of host time per torch.distributed
    call (the task's "capture launch-bound inner loops in CUDA graphs").  The
    graph owns its flag array: its first node zeroes the flags, then the
    communication branch (collectives + signals, epoch 1) and the product
    branch run concurrently, the product spinning on the flags as in the eager
    step.  A first eager step before the capture initialises the collectives'
    communicator and loads every kernel.  Inputs and output are fixed at
    construction (A_panel, B, out are reused by every replay).  NCCL
    collectives inside CUDA graphs need the communicator to exist before the
    capture, which the eager step guarantees."""

    def __init__(self, A_panel, B, out, group=None, root=0, chunks=None, path="auto",
                 reserve_sms=None, bcast="root"):
        import torch
        self.kw = dict(group=group, root=root, chunks=chunks, path=path, out=out, reserve_sms=reserve_sms,
                       bcast=bcast)
        self.A, self.B, self.out = A_panel, B, out
        gemm_rowpanel(A_panel, B, timings=False, **self.kw)          # warm: comm init, kernel loads
        torch.cuda.synchronize()
        self.flags = torch.zeros(FLAG_WORDS, dtype=torch.int32, device=A_panel.device)
        self.comm = torch.cuda.Stream(device=A_panel.device)
        self.graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(device=A_panel.device)
        cap.wait_stream(torch.cuda.current_stream(A_panel.device))
        with torch.cuda.graph(self.graph, stream=cap):
            self.flags.zero_()
            _, self.info = gemm_rowpanel(A_panel, B, timings=False, comm_stream=self.comm, flags=self.flags,
                                         epoch=1, **self.kw)
        torch.cuda.synchronize()

    def replay(self):
        self.graph.replay()
        return self.out


class HostWorkspace:
    """Device buffers of the host-buffer step, kept across calls (a serving
    loop re-uses them; the caching allocator would too, but emulation needs
    B's non-owned chunks to persist)."""

    def __init__(self):
        self.bufs = {}

    def get(self, name, shape, device):
        import torch
        t = self.bufs.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.device != device:
            t = torch.empty(shape, dtype=torch.float32, device=device)
            self.bufs[name] = t
        return t


def gemm_rowpanel_host(A_panel, B, C_panel, group=None, root=0, chunks=None, path="auto", bcast="owners",
                       reserve_sms=None, workspace=None, emulate_world=None, broadcast=True,
                       device=None, gemm_fn=None):
    """End-to-end step from HOST buffers (pinned CPU tensors): the multi-GPU
    counterpart of lpy_gemm_f32_host.  Each rank uploads its A panel and only
    the K-row chunks of B it owns (chunk_owner: c mod world with bcast
    "owners" or "allgather", so each rank moves ~1/g of B over PCIe instead of
    all of it), the chunks
    are broadcast over NCCL / NVLink as they land while the gated product
    consumes them, and the C panel is downloaded into `C_panel`.  Synchronises
    before returning.  Returns {"h2d_bytes", "d2h_bytes", "chunks"} (this
    rank's PCIe traffic).

    emulate_world (diagnostics at world 1 only): plan ownership as if there
    were that many ranks -- rank 0 uploads only its own chunks and the others
    are taken as already delivered (the workspace must hold them from an
    earlier call with emulate_world=None); the broadcast is a no-op.

    device="cpu" (tests, gloo): the same plan on CPU "device" buffers -- the
    uploads are plain copies of the owned chunks into a NaN-filled B, the
    chunks go through gemm_rowpanel's CPU branch and `gemm_fn` computes the
    panel -- so the ownership, the PCIe byte accounting and the broadcast plan
    are exercised without a GPU (tests/test_dist.py).
    """
    import torch
    import torch.distributed as dist

    rows, K = A_panel.shape
    N = B.shape[1]
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ws = workspace or _state.setdefault(("host_ws", str(dev)), HostWorkspace())
    world = dist.get_world_size(group) if broadcast else 1
    rank = dist.get_rank(group) if broadcast else 0
    plan_world = emulate_world if (emulate_world and world == 1) else world
    resolved = path
    if path == "auto":
        from . import PATH_AUTO, lpy_select_path
        _, ch = lpy_select_path(rows, N, K, PATH_AUTO)
        resolved = {1: "ffma", 2: "3xtf32"}[ch]
    if isinstance(chunks, (list, tuple)):
        bounds = [tuple(b) for b in chunks]
    else:
        bounds = kchunk_bounds(K, chunks or choose_kchunks(rows, K, resolved))
    check_kchunks(bounds, K)
    mine = set(owned_chunks(len(bounds), plan_world, rank, root, bcast))
    if dev.type == "cpu":
        dA = A_panel.clone()
        dB = torch.full((K, N), float("nan"))
        h2d_bytes = 4 * rows * K
        for c in sorted(mine):
            k0, k1 = bounds[c]
            dB[k0:k1] = B[k0:k1]
            h2d_bytes += 4 * (k1 - k0) * N
        dC, _ = gemm_rowpanel(dA, dB, group=group, root=root, chunks=bounds, path=path, bcast=bcast,
                              broadcast=world > 1, gemm_fn=gemm_fn)
        C_panel.copy_(dC)
        return {"h2d_bytes": h2d_bytes, "d2h_bytes": 4 * rows * N, "chunks": len(bounds), "B": dB}
    dA = ws.get("A", (rows, K), dev)
    dB = ws.get("B", (K, N), dev)
    dC = ws.get("C", (rows, N), dev)
    caller = torch.cuda.current_stream(dev)
    key = ("h2d", str(dev))
    if key not in _state:
        _state[key] = torch.cuda.Stream(device=dev)
    h2d = _state[key]
    comm = _comm_stream(dev)
    h2d.wait_stream(caller)
    ev_a = torch.cuda.Event()
    ev_b = [torch.cuda.Event() for _ in bounds]
    h2d_bytes = 0
    with torch.cuda.stream(h2d):
        # A first: the product needs all of its k range from the first chunk on
        dA.copy_(A_panel, non_blocking=True)
        h2d_bytes += 4 * rows * K
        ev_a.record(h2d)
        for c, (k0, k1) in enumerate(bounds):
            if c in mine:
                dB[k0:k1].copy_(B[k0:k1], non_blocking=True)
                h2d_bytes += 4 * (k1 - k0) * N
            ev_b[c].record(h2d)

    caller.wait_event(ev_a)
    gemm_rowpanel(dA, dB, group=group, root=root, chunks=bounds, path=path, out=dC,
                  reserve_sms=reserve_sms, bcast=bcast, broadcast=world > 1, comm_stream=comm,
                  timings=False, before_chunk=lambda c: comm.wait_event(ev_b[c]))
    C_panel.copy_(dC, non_blocking=True)
    caller.synchronize()
    return {"h2d_bytes": h2d_bytes, "d2h_bytes": 4 * rows * N, "chunks": len(bounds)}
