"""Multi-GPU row-panel product (BASELINE.json north_star).

C's rows are split into contiguous panels, one per rank (one process per GPU);
rank r owns rows [r*ceil(M/g), min(M, (r+1)*ceil(M/g))) of A and C
(reading A14).  Row panels are independent given the whole of B,
C[rows_r, :] = A[rows_r, :] B, so the only exchange is ONE broadcast of B
(4*K*N bytes) from the root over NCCL / NVLink; C stays sharded.

To overlap the broadcast with the product, B is held in column-blocked
storage: `chunks` contiguous blocks, block c a row-major K x w_c matrix
(the same logical B, different storage -- the paper's layout tags).
Block c is broadcast on a dedicated communication stream; as soon as it has
arrived, C[:, cols_c] = A_panel B_c (an lpy_gemm_f32 call writing a disjoint
column block of C, ldc = N) runs on one of `compute_streams` streams, so the
product of a block overlaps the broadcast of the next, and the block products
run concurrently on several streams, each with a persistent grid sized to its
own tiles (`chunk_grid`), so together they fill the GPU.  Chunk widths are
multiples of 256 (the 3xTF32 pair tile) so each block is 16-byte aligned.

The GEMM itself is injected (`gemm_fn`) so the orchestration can be tested
on CPU with the gloo backend (tests/test_dist.py).
"""
from __future__ import annotations

import math


def panel_bounds(M: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of C owned by `rank` (contiguous panels of ceil(M/world))."""
    if world < 1 or not 0 <= rank < world or M < 0:
        raise ValueError("bad panel request")
    h = math.ceil(M / world) if M else 0
    r0 = min(M, rank * h)
    return r0, min(M, r0 + h)


def chunk_bounds(N: int, chunks: int, align: int = 256) -> list[tuple[int, int]]:
    """Column blocks [c0, c1) covering [0, N): `chunks` blocks (fewer if N is
    small) whose widths are multiples of `align` except possibly the last."""
    if N <= 0:
        return []
    chunks = max(1, min(chunks, math.ceil(N / align)))
    w = math.ceil(math.ceil(N / chunks) / align) * align
    out, c0 = [], 0
    while c0 < N:
        out.append((c0, min(N, c0 + w)))
        c0 += w
    return out


def choose_chunks(rows: int, N: int, sms: int = 148, tile: int = 256, max_chunks: int = 8) -> int:
    """Number of B column blocks for a rank's (rows x N) panel.  The step takes
    about T_bcast / chunks + T_products(chunks); measured on one B200 at n=8192
    (scripts/panel_probe.py, profiles/r01_panel_probe.txt) the products lose
    2-3% at 8 blocks for a 1024-row panel but 8-11% for 2048/4096-row panels,
    where the broadcast is also a smaller share of the step, so: 8 blocks for
    panels of <= 1024 rows, 4 up to 2048, else 2 (blocks >= 1024 columns)."""
    del sms
    want = 8 if rows <= 1024 else 4 if rows <= 2048 else 2
    return max(1, min(max_chunks, want, N // (4 * tile)))


def chunk_streams(rows: int, chunks: int) -> int:
    """Concurrent compute streams for the block products (same measurement):
    4 for 1024-row panels, 2 up to 2048, 1 beyond (then one block's product
    fills the GPU by itself)."""
    want = 4 if rows <= 1024 else 2 if rows <= 2048 else 1
    return max(1, min(want, chunks))


def chunk_tile_n(path: str) -> int:
    """Output-tile width (opts.tile_n) for a block product: full-width tiles
    (256 x 256 per CTA pair on 3xTF32, 128 x 256 per CTA on FFMA) whatever
    share of the GPU the block's grid gets; the automatic choice would look at
    the block alone and pick narrower tiles to fill all SMs."""
    del path
    return 256


def chunk_grid(rows: int, cols: int, sms: int, path: str) -> int:
    """Persistent grid (CTAs) for one block product sized to its own tiles
    of width chunk_tile_n (256 x 256 per CTA pair on 3xTF32, 128 x 256 per CTA
    on FFMA), so concurrent block products share the SMs instead of each
    claiming all."""
    tn = chunk_tile_n(path)
    if path == "3xtf32":
        return 2 * max(1, min(sms // 2, math.ceil(rows / 256) * math.ceil(cols / tn)))
    return max(1, min(sms, math.ceil(rows / 128) * math.ceil(cols / tn)))


def block_owner(c: int, world: int, root: int = 0, owners: bool = False) -> int:
    """Rank holding column block c of B before the step: `root` for the
    north_star's broadcast of B, or rank c mod world when B starts sharded
    by column blocks (`owners=True`: every rank broadcasts the blocks it holds,
    so the send load -- and B's generation -- is spread over all ranks; an
    all-gather of the blocks expressed as per-block broadcasts, since NCCL's
    all-gather needs equal contiguous pieces and the blocks are column blocks)."""
    return c % world if owners else root


def rowpanel_gemm(A_panel, B_blocks, C_panel, bounds, group=None, root=0, gemm_fn=None,
                  comm_stream=None, compute_streams=None, broadcast=True, owners=False):
    """One distributed product step on this rank.

    A_panel : (rows_r, K) tensor, this rank's rows of A.
    B_blocks: list of (K, w_c) contiguous tensors, the column blocks of B; block
              c valid on block_owner(c) (root, or c mod world with owners=True),
              receive buffers elsewhere.  Broadcast in order.
    C_panel : (rows_r, N) row-major tensor; column block c is written by
              gemm_fn(A_panel, B_blocks[c], C_panel[:, c0:c1]).
    bounds  : chunk_bounds(N, len(B_blocks)).
    On CUDA the caller's current stream is joined to all the work before return
    (the step is complete in stream order).  Returns the "block arrived" events
    (CUDA) or None (CPU).
    """
    import torch
    import torch.distributed as dist

    if gemm_fn is None:
        from . import gemm as gemm_fn_default

        def gemm_fn(a, b, c):
            gemm_fn_default(a, b, out=c)
    world = dist.get_world_size(group) if broadcast else 1
    src = [block_owner(c, world, root, owners) for c in range(len(B_blocks))]
    if not A_panel.is_cuda:
        # CPU (gloo) path: same order, no overlap
        for c, ((c0, c1), blk) in enumerate(zip(bounds, B_blocks)):
            if broadcast:
                dist.broadcast(blk, src=src[c], group=group)
            gemm_fn(A_panel, blk, C_panel[:, c0:c1])
        return None

    caller = torch.cuda.current_stream()
    comm = comm_stream or torch.cuda.Stream()
    streams = compute_streams or [torch.cuda.Stream()
                                  for _ in range(chunk_streams(A_panel.shape[0], len(B_blocks)))]
    comm.wait_stream(caller)
    for st in streams:
        st.wait_stream(caller)
    events = []
    for c, blk in enumerate(B_blocks):
        if broadcast:
            with torch.cuda.stream(comm):
                dist.broadcast(blk, src=src[c], group=group)
        ev = torch.cuda.Event()
        ev.record(comm)
        events.append(ev)
    for i, ((c0, c1), blk, ev) in enumerate(zip(bounds, B_blocks, events)):
        st = streams[i % len(streams)]
        st.wait_event(ev)
        with torch.cuda.stream(st):
            gemm_fn(A_panel, blk, C_panel[:, c0:c1])
    caller.wait_stream(comm)
    for st in streams:
        caller.wait_stream(st)
    return events
