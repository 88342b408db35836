#!/usr/bin/env python
"""Benchmark: fp32 C = A*B (Loo.py's reduction example)
on B200 through the C-ABI, BASELINE.json's metric

    "fp32 GEMM GFLOP/s at n=4096/8192 on 1/2/4/8 B200; % of FMA/TF32 roofline"

One step = one whole distributed product over the n=8192 square workload
(BASELINE config 4): at N=1 one lpy_gemm_f32 call; at N>1 each rank owns a
row panel of A and C, B is broadcast from rank 0 with NCCL inside the step in
chunks of K rows, and one K-gated product per rank consumes each chunk as it
lands (dist.gemm_rowpanel).  `value` = 2 n^3 per step /
max-over-ranks device time (strong scaling: total work fixed).

Prints ONE JSON line on rank 0 (contract in the task statement; fields
documented in DESIGN.md "Measurement").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 8192] [--path auto|ffma|3xtf32]
  python bench.py --impl reference ...   # the float64 CPU oracle, timed on host cores
"""
from __future__ import annotations

import argparse
import json
import os
import faulthandler
import statistics
import subprocess
import sys
import time

faulthandler.enable()

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fp32 GEMM GFLOP/s at n=4096/8192 on 1/2/4/8 B200; % of FMA/TF32 roofline"
UNIT = "GFLOP/s"
L2_BYTES = 126 * 2 ** 20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


def roofline_peak(path: str):
    """(bound, peak TFLOP/s, note) for the dominant kernel of `path`.

    3xtf32: tensor bound; TF32 peak = measured bf16 burst x the guide's nominal
            tf32/bf16 ratio (1.1 / 2.25), divided by 3 because every fp32
            product costs three tf32 MMAs (frac = tensor-pipe utilisation).
    ffma  : plain fp32 FMA ("alu") bound: 148 SM x 128 FP32 lanes x 2 flop x
            max SM clock."""
    peaks, src = load_peaks()
    if path == "3xtf32":
        tf32 = peaks["bf16_tflops"] * (1.1 / 2.25)
        return "tensor", tf32 / 3.0, (f"TF32 = {src} bf16 burst {peaks['bf16_tflops']} x 1.1/2.25 = "
                                       f"{tf32:.1f} TFLOP/s; /3 for 3 tf32 MMAs per fp32 product")
    mhz = peaks.get("sm_max_mhz", 1965.0)
    return "alu", 148 * 128 * 2 * mhz * 1e6 / 1e12, f"148 SM x 128 FP32 lanes x 2 x {mhz} MHz ({src} clock)"


def profile_traffic(path: str, n: int):
    """DRAM bytes (read + write) per launch of `path`'s kernel at size n from the
    newest committed `ncu --set full` summary (profiles/rNN_ncu_full_<path>_n<n>.txt),
    or (None, None)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_full_{path}_n{n}.txt")))
    if not files:
        return None, None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    total = 0.0
    seen = 0
    with open(files[-1]) as f:
        for line in f:
            parts = line.split()
            if parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum") and len(parts) >= 3:
                total += float(parts[1]) * scale.get(parts[2], 1)
                seen += 1
    return (int(total), os.path.relpath(files[-1], ROOT)) if seen == 2 else (None, None)


class ClockSampler:
    """Samples SM clock + throttle reasons with `nvidia-smi -lms` during the
    timed region (the profiling guide's clocks line)."""

    FIELDS = ("index,pci.bus_id,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int, period_ms: int = 20):
        import shutil
        import tempfile
        self.period = period_ms
        self.proc = None
        self.bus = None
        try:
            import torch
            p = torch.cuda.get_device_properties(device_index)
            self.bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
        except Exception:
            pass
        self.smi = shutil.which("nvidia-smi")
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        if self.smi:
            cmd = [self.smi, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                   f"-lms", str(self.period)]
            self.proc = subprocess.Popen(cmd, stdout=self.out, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.smi:
            return None
        self.out.flush()
        rows = []
        with open(self.out.name) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 10:
                    rows.append(parts)
        os.unlink(self.out.name)
        mine = [r for r in rows if self.bus and r[1].upper().endswith(self.bus[-12:])]
        rows = mine or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm = []
        for r in rows:
            try:
                sm.append(float(r[2]))
            except ValueError:
                pass
            for name, val in zip(names, r[6:10]):
                if val.lower() == "active":
                    reasons.add(name)
        loaded = [x for x in sm if x > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": float(rows[0][3]) if rows[0][3].replace('.', '').isdigit() else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# --------------------------------------------------------------------------- CPU oracle
def host_cores() -> int:
    """The host cores this process may run on.  The oracle is timed on all of
    them: torchrun sets OMP_NUM_THREADS=1 for every rank, but at N > 1 only
    rank 0 runs the oracle while the others wait."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return max(1, os.cpu_count() or 1)


def oracle_sample(n: int, seconds: float, dist_name: str, nthreads: int = 0):
    """Time the float64 oracle on a bounded sample of the n x n x n product:
    the first R rows of C (R sized to ~`seconds`).  Returns (GFLOP/s, sample
    description, threads)."""
    import numpy as np
    import oracle
    import synth
    B = synth.matrix(n, n, seed=0, matrix_id=synth.MATRIX_B, dist=dist_name).reshape(-1)
    threads = nthreads or oracle.max_threads()
    R = max(1, threads)
    A = synth.matrix(R, n, seed=0, matrix_id=synth.MATRIX_A, dist=dist_name).reshape(-1)
    t0 = time.perf_counter()
    oracle.gemm_rows(R, n, n, A, n, 0, B, n, 0, 0, R, nthreads=threads)
    dt = time.perf_counter() - t0
    rows = int(max(R, min(n, R * max(1.0, seconds / max(dt, 1e-6)))))
    rows = (rows // threads) * threads or threads
    A = synth.matrix(rows, n, seed=0, matrix_id=synth.MATRIX_A, dist=dist_name).reshape(-1)
    t0 = time.perf_counter()
    oracle.gemm_rows(rows, n, n, A, n, 0, B, n, 0, 0, rows, nthreads=threads)
    dt = time.perf_counter() - t0
    gflops = 2.0 * rows * n * n / dt / 1e9
    return gflops, dt, f"first {rows} rows of C for n={n} (all of B), float64 i-k-j loop", threads


JSON_OUT = {"fd": None}


def emit(line: dict) -> None:
    """Print the one JSON line on the real stdout (saved before NCCL could
    write to fd 1)."""
    fd = JSON_OUT["fd"]
    if fd is None:
        print(json.dumps(line), flush=True)
    else:
        sys.stdout.flush()
        os.write(fd, (json.dumps(line) + "\n").encode())


def cpu_model() -> str | None:
    """The host CPU's model name (lscpu's "Model name"), from /proc/cpuinfo."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, timed on this box's host cores."""
    if rank != 0:
        return
    import oracle
    n = args.n
    # each step a bounded sample: the whole --steps K --warmup W run stays near
    # --ref-total seconds (a few minutes at most), at least 0.2 s of work per step
    per_step = max(0.2, min(args.ref_seconds, args.ref_total / max(1, args.steps + args.warmup)))
    # calibrate the sample once, then time each step on that fixed sample
    gf, dt, sample, threads = oracle_sample(n, per_step, "uniform", nthreads=host_cores())
    times = []
    import numpy as np
    import synth
    rows = int(sample.split()[1])
    B = synth.matrix(n, n, seed=0, matrix_id=synth.MATRIX_B).reshape(-1)
    A = synth.matrix(rows, n, seed=0, matrix_id=synth.MATRIX_A).reshape(-1)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.gemm_rows(rows, n, n, A, n, 0, B, n, 0, 0, rows, nthreads=threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times)
    value = 2.0 * rows * n * n * len(times) / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded SplitMix64 uniform[-1,1) fp32 inputs",
        "config": {"workload": f"n={n} square C=A*B, row-major (BASELINE config 4), "
                               f"bounded sample: {rows} rows of C per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def host_inputs(n, r0, r1, chunk_rows):
    """Host (numpy) A panel rows [r0, r1) and the K-row chunks of B listed in
    `chunk_rows` [(k0, k1), ...] (None: all of B) -- the seeded synthetic
    inputs; every rank draws only what it holds."""
    import numpy as np
    import synth
    A = synth.matrix(r1 - r0, n, seed=0, matrix_id=synth.MATRIX_A, row0=r0)
    if chunk_rows is None:
        return A, synth.matrix(n, n, seed=0, matrix_id=synth.MATRIX_B)
    B = np.full((n, n), np.nan, dtype=np.float32)
    for k0, k1 in chunk_rows:
        B[k0:k1] = synth.matrix(k1 - k0, n, seed=0, matrix_id=synth.MATRIX_B, row0=k0)
    return A, B


def time_path(args, path, rank, world, device, dist_on):
    """Device-resident step.  N = 1: one lpy_gemm_f32 call.  N > 1 (or
    --force-dist): the fused row-panel step, dist.gemm_rowpanel -- B broadcast
    from its owner(s) in K-row chunks on a communication stream while ONE
    K-gated product per rank consumes the chunks as they land."""
    import torch
    import paper_1405_7470_b200 as lpy
    from paper_1405_7470_b200.dist import (choose_kchunks, gemm_rowpanel, kchunk_bounds, owned_chunks,
                                          panel_bounds, panel_opts, chunk_owner, transfers)
    n = args.n
    pw = args.emulate_ranks if (args.emulate_ranks and world == 1) else world   # panel split
    r0, r1 = panel_bounds(n, pw, rank)
    rows = r1 - r0
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    mode = args.bcast
    from paper_1405_7470_b200.dist import comm_group, default_reserve
    reserve = args.reserve_sms or default_reserve(path)
    bounds = kchunk_bounds(n, args.chunks or choose_kchunks(rows, n, path)) if dist_on else [(0, n)]
    mine = owned_chunks(len(bounds), world, rank, 0, mode) if dist_on else [0]
    Ah, Bh = host_inputs(n, r0, r1, [bounds[c] for c in mine] if dist_on and world > 1 else None)
    A = torch.from_numpy(Ah).to(device)
    B = torch.from_numpy(Bh).to(device)
    del Bh
    C = torch.empty((rows, n), dtype=torch.float32, device=device)

    graph = None
    if dist_on and args.graph:
        # the whole step (collectives + signals + gated product) as one CUDA graph
        from paper_1405_7470_b200.dist import RowPanelGraph
        graph = RowPanelGraph(A, B, C, chunks=bounds, path=path, reserve_sms=reserve, bcast=mode)

    before_chunk = None
    if dist_on and world == 1 and args.emulate_bcast_gbs > 0:
        # Diagnostics (world 1): stand in for the broadcast's arrival of chunk c
        # with, on the communication stream, a device-side wait and a copy of
        # the chunk into B by `reserve_sms` persistent CTAs (liblpy_probe.so's
        # persistent copy: the way a collective's channel CTAs move bytes, on
        # the SMs the gated product leaves free, through HBM as a receive
        # would), paced so the chunk rate does not exceed --emulate-bcast-gbs
        # (0 < rate; a huge rate = copies back to back) -- a projection of a
        # g-rank step, not a bench value.  (A first version copied with torch's
        # elementwise kernel: its many small blocks on 16 SMs moved ~0.4 TB/s
        # and measured that kernel rather than the overlap.)
        import ctypes
        probe = ctypes.CDLL(os.path.join(os.path.dirname(lpy.library_path()), "liblpy_probe.so"))
        probe.lpy_probe_persistent_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                                    ctypes.c_int, ctypes.c_void_p]
        probe.lpy_probe_bulk_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int,
                                              ctypes.c_void_p]
        copy_mode = os.environ.get("LPY_EMUL_COPY", "threads")
        bulk = copy_mode == "bulk"        # TMA bulk copies instead of thread copies
        # cudaMemcpyAsync pulls (a dist copy-engine pull mode's stand-in) -- but on one GPU the
        # device-to-device copies ran on SMs (profiles/r02_ce_emul.txt), so this does not model
        # NVLink copy-engine pulls
        ce = copy_mode == "ce"
        Bsrc = B.clone()
        clock_hz = 1.9e9

        owned_only = args.bcast == "allgather"    # NVLS all-gather: a rank's SMs move only its own shard

        def before_chunk(c, _b=bounds):
            k0, k1 = _b[c]
            nbytes = 4 * (k1 - k0) * B.shape[1]
            wait_s = nbytes / (args.emulate_bcast_gbs * 1e9)
            if wait_s > 2e-6:
                torch.cuda._sleep(int(wait_s * clock_hz))
            if ce:
                # the rank pulls every chunk it does not own from its owner with its copy
                # engines (dist "ce" mode: each chunk c is owned by rank c mod g)
                if c % args.emulate_ranks != 0:
                    B[k0:k1].copy_(Bsrc[k0:k1], non_blocking=True)
                return
            if owned_only and c % args.emulate_ranks != 0:
                return          # delivered by the switch: no SM work on this rank
            ctas = max(1, reserve - 1)
            if bulk:
                rc = probe.lpy_probe_bulk_copy(B[k0:k1].data_ptr(), Bsrc[k0:k1].data_ptr(), nbytes, ctas,
                                               torch.cuda.current_stream().cuda_stream)
            else:
                rc = probe.lpy_probe_persistent_copy(B[k0:k1].data_ptr(), Bsrc[k0:k1].data_ptr(),
                                                     (k1 - k0) * B.shape[1], ctas,
                                                     torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc

    def step():
        if not dist_on:
            lpy.gemm(A, B, out=C, path=path)
        elif graph is not None:
            graph.replay()
        else:
            gemm_rowpanel(A, B, chunks=bounds, path=path, out=C, bcast=mode, reserve_sms=reserve,
                          timings=False, before_chunk=before_chunk)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0.record()
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            per.append((e0, e1))
        t1.record()
        torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    kernel_ms = [a.elapsed_time(b) for a, b in per]
    multi = None
    if dist_on:
        import torch.distributed as dist

        def max_ms(ms):
            t = torch.tensor([ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        def timed(fn, reps):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return max_ms(a.elapsed_time(b) / reps)

        total_ms = max_ms(total_ms)
        reps = max(3, min(args.steps, 10))
        # the two halves of a step, each timed alone (max over ranks): B's
        # chunked broadcast (4*K*N bytes from the owners) and this rank's
        # product planned for the same SMs, ungated (bitwise the gated one)
        opts = panel_opts(sms, reserve)
        plan = transfers(bounds, world, 0, mode)
        cg = comm_group(reserve)

        def comm_only():
            for kind, cs in plan:
                if kind == "bcast":
                    k0, k1 = bounds[cs[0]]
                    dist.broadcast(B[k0:k1], src=chunk_owner(cs[0], world, 0, mode), group=cg)
                else:
                    p0, p1 = bounds[cs[rank]]
                    dist.all_gather_into_tensor(B[bounds[cs[0]][0]:bounds[cs[-1]][1]], B[p0:p1], group=cg)
        bcast_ms = timed(comm_only, reps)
        gemm_ms = timed(lambda: lpy.gemm(A, B, out=C, path=path, opts=opts), reps)
        nbytes = 4 * n * n
        multi = {"total_ms": round(total_ms / args.steps, 4), "bcast_ms": round(bcast_ms, 4),
                 "gemm_ms": round(gemm_ms, 4), "bcast_bytes": nbytes,
                 "bcast_algbw_gbs": round(nbytes / (bcast_ms * 1e-3) / 1e9, 1), "chunks": len(bounds),
                 "chunk_k": bounds[0][1] - bounds[0][0], "plan_sms": opts.plan_sms,
                 "reserve_sms": reserve, "bcast": args.bcast, "graph": bool(args.graph),
                 "emulate_bcast_gbs": args.emulate_bcast_gbs or None}
        dist.barrier()
        step()                      # the output parity checks below is a full step's
        torch.cuda.synchronize()
    # sampled parity of this run's output against the oracle, on EVERY rank
    # (max over ranks): the reference regenerates A's panel and all of B from
    # the seeded generator on the host, independent of the broadcast
    parity = None
    if not args.no_parity:
        parity = sampled_parity(Ah, C, n, r0)
        if dist_on:
            import torch.distributed as dist
            t = torch.tensor([parity], device=device, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            parity = float(t.item())
    _, chosen = lpy.lpy_select_path(rows, n, n, lpy.PATHS[path])
    launches = 1 + (len(bounds) if dist_on else 0)      # the product (+ one signal kernel per chunk)
    return {"total_ms": total_ms, "kernel_ms": kernel_ms, "clocks": clk.summary(), "parity": parity,
            "path": {1: "ffma", 2: "3xtf32"}[chosen], "launches_per_step": launches, "chunks": len(bounds),
            "multi": multi}


_B_HOST = {}


def sampled_parity(Ah, C, n, r0, count=512):
    """Max normalised error of `count` sampled elements of this rank's C
    panel plus its first/last rows at every 256-column tile boundary, against
    the float64 oracle on regenerated inputs."""
    import numpy as np
    import oracle
    import synth
    if n not in _B_HOST:
        _B_HOST.clear()
        _B_HOST[n] = synth.matrix(n, n, seed=0, matrix_id=synth.MATRIX_B).reshape(-1)
    Bh = _B_HOST[n]
    rng = np.random.default_rng(r0)
    rows = Ah.shape[0]
    edges = np.array(sorted({c for t in range(0, n, 256) for c in (t, t + 255) if c < n} | {n - 1}))
    ii = np.concatenate([rng.integers(0, rows, count), np.zeros(edges.size, np.int64),
                         np.full(edges.size, rows - 1)])
    jj = np.concatenate([rng.integers(0, n, count), edges, edges])
    Ch = C.cpu().numpy()
    Cref, D = oracle.gemm_elems(rows, n, n, Ah.reshape(-1), n, 0, Bh, n, 0, ii, jj)
    return oracle.normalized_error(Ch[ii, jj], Cref, D)


def time_e2e(args, path, rank, world, device, dist_on):
    """The same step end to end from pinned HOST buffers through the public
    API, copies inside the timed region.  N = 1: lpy_gemm_f32_host (A, B up,
    C down).  N > 1: dist.gemm_rowpanel_host -- each rank uploads its A panel
    and only the K-row chunks of B it owns (1/g of B), the chunks are broadcast
    over NCCL as they land, the gated product consumes them, and each rank
    downloads its C panel: 4(MK + KN) bytes up and 4MN down in total, not
    g times B.  At world 1 with --force-dist --emulate-ranks g: rank 0's share
    of a g-rank step (its own chunks only; a diagnostic, not a bench value)."""
    import torch
    import paper_1405_7470_b200 as lpy
    import synth
    from paper_1405_7470_b200.dist import (HostWorkspace, choose_kchunks, gemm_rowpanel_host, kchunk_bounds,
                                          owned_chunks, panel_bounds)
    n = args.n
    emul = args.emulate_ranks if (args.emulate_ranks and world == 1 and dist_on) else None
    pw = emul or world
    r0, r1 = panel_bounds(n, pw, rank)
    rows = r1 - r0
    A = torch.from_numpy(synth.matrix(rows, n, seed=0, matrix_id=0, row0=r0)).pin_memory()
    steps = max(1, min(args.steps, args.e2e_steps))
    if not dist_on:
        B = torch.from_numpy(synth.matrix(n, n, seed=0, matrix_id=1)).pin_memory()
        C = torch.empty((rows, n), dtype=torch.float32).pin_memory()
        s = torch.cuda.current_stream()

        def step():
            lpy.gemm_host(rows, n, n, A, n, 0, B, n, 0, C, n, 0, path=path, stream=s)
            return 4 * (rows * n + n * n), 4 * rows * n
    else:
        # host buffers: every rank uploads only the K-row chunks it owns (c mod
        # N), so B crosses PCIe once in total, then NVLink (owners broadcast, or
        # the all-gather rounds with --bcast allgather)
        mode = "allgather" if args.bcast == "allgather" else "owners"
        bounds = kchunk_bounds(n, args.chunks or choose_kchunks(rows, n, path))
        mine = owned_chunks(len(bounds), pw, rank, 0, mode)
        _, Bh = host_inputs(n, r0, r1, [bounds[c] for c in mine] if (world > 1 or emul) else None)
        B = torch.from_numpy(Bh).pin_memory()
        del Bh
        C = torch.empty((rows, n), dtype=torch.float32).pin_memory()
        ws = HostWorkspace()
        if emul:
            # the chunks rank 0 does not own are "delivered by its peers": put
            # them in the workspace once, outside the timed region
            Bfull = torch.from_numpy(synth.matrix(n, n, seed=0, matrix_id=1))
            ws.get("B", (n, n), torch.device("cuda", torch.cuda.current_device())).copy_(Bfull)
            del Bfull

        def step():
            info = gemm_rowpanel_host(A, B, C, chunks=bounds, path=path, bcast=mode,
                                      reserve_sms=args.reserve_sms or None, workspace=ws, emulate_world=emul)
            return info["h2d_bytes"], info["d2h_bytes"]

    step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        h2d, d2h = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    h2d_rank = h2d
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        t = torch.tensor([h2d, d2h], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        h2d, d2h = int(t[0].item()), int(t[1].item())
    flops = 2.0 * n ** 3 / (pw if emul else 1)
    out = {"value": flops / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": ms, "h2d_bytes_rank0": h2d_rank}
    if emul:
        out["emulated_rank0_of"] = emul
    return out


def time_cublas_context(args, device):
    """Context only: torch.matmul on the same n x n fp32 inputs
    through cuBLAS as SGEMM (allow_tf32 = False, fp32-accurate) and as plain
    TF32 (allow_tf32 = True, NOT fp32-accurate: its normalised error is
    reported beside it).  Library kernels, not this repository's."""
    import numpy as np
    import torch
    import oracle
    n = args.n
    g = torch.Generator(device=device)
    g.manual_seed(0)
    A = torch.rand(n, n, device=device, generator=g) * 2 - 1
    B = torch.rand(n, n, device=device, generator=g) * 2 - 1
    out = {}
    rows = np.arange(0, n, max(1, n // 64))
    Ah = A[rows].cpu().numpy().reshape(-1)
    Bh = B.cpu().numpy().reshape(-1)
    Cref, D = oracle.gemm_rows(len(rows), n, n, Ah, n, 0, Bh, n, 0)
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        for name, tf32 in (("cublas_sgemm", False), ("cublas_tf32", True)):
            torch.backends.cuda.matmul.allow_tf32 = tf32
            for _ in range(3):
                C = A @ B
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                C = A @ B
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            err = oracle.normalized_error(C[rows].cpu().numpy(), Cref, D)
            out[name] = {"tflops": round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 2), "ms": round(ms, 4),
                         "max_norm_err_sampled_rows": err}
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def time_saxpy(args, device):
    """Table 1's saxpy row: y := alpha*x + y over n = 2^28
    fp32 elements (1 GiB per vector, 3 GiB of HBM traffic per call, far above
    L2) through lpy_saxpy_f32, device-resident; GB/s = 12 n / kernel time."""
    import numpy as np
    import torch
    import oracle
    import paper_1405_7470_b200 as lpy
    n = args.saxpy_n
    alpha = 1.5
    g = torch.Generator(device=device)
    g.manual_seed(0)
    x = torch.rand(n, device=device, generator=g) * 2 - 1
    y = torch.rand(n, device=device, generator=g) * 2 - 1
    # parity on this launch configuration: one call on a copy, sampled elements vs the oracle
    rng = np.random.default_rng(0)
    idx = np.sort(rng.integers(0, n, 1 << 16))
    ti = torch.from_numpy(idx).to(device)
    xs, ys = x[ti].cpu().numpy(), y[ti].cpu().numpy()
    y1 = y.clone()
    lpy.saxpy(alpha, x, y1)
    got = y1[ti].cpu().numpy()
    ref = oracle.saxpy(idx.size, alpha, xs, 1, ys, 1)
    ulps = oracle.saxpy_error_ulps(got, ref)
    del y1
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        lpy.saxpy(alpha, x, y)
    torch.cuda.synchronize()
    # back-to-back calls between one pair of events on the launching stream:
    # the mean per-call time (per-call event pairs add their own gaps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            lpy.saxpy(alpha, x, y)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    gbs = 12.0 * n / (ms * 1e-3) / 1e9
    peaks, src = load_peaks()
    peak = peaks["hbm_gbs"]
    traffic, tsrc = profile_traffic("saxpy", n)
    return {"metric": "saxpy GB/s (y := alpha*x + y, 12 B per element)", "value": round(gbs, 1),
            "unit": "GB/s", "n": n, "ms_per_call": round(ms, 4), "calls": args.steps, "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "traffic": traffic, "traffic_source": tsrc,
                         "algorithmic_bytes": 12 * n, "peak_note": f"{src} copy bandwidth (MEASURED_PEAKS.json)"},
            "parity_sampled_max_half_ulps": ulps, "clocks": clk.summary(),
            "data": "synthetic: torch.rand seeded 0, uniform[-1,1), alpha = 1.5"}


def time_coulomb(args, device):
    """Table 1's 3D Coulomb potential row: the self-potential
    of N = 2^16 synthetic point charges (unit cube, charges uniform[-1,1)),
    targets == sources, through lpy_coulomb_f32; pairs/s = N^2 / kernel time
    (the loop domain {[i, j]}, self pairs included in the count)."""
    import numpy as np
    import torch
    import oracle
    import paper_1405_7470_b200 as lpy
    import synth
    n = args.coulomb_n
    pos, q = synth.particles(n, seed=0)
    P = torch.from_numpy(pos.reshape(n, 3)).to(device)
    Q = torch.from_numpy(q).to(device)
    phi = torch.empty(n, device=device)
    lpy.coulomb(P, P, Q, out=phi)
    torch.cuda.synchronize()
    idx = np.random.default_rng(0).choice(n, 256, replace=False)
    tsel = np.ascontiguousarray(pos.reshape(n, 3)[idx]).reshape(-1)
    t0 = time.perf_counter()
    ref, D = oracle.coulomb(idx.size, tsel, 3, n, pos, 3, q)
    cpu_dt = time.perf_counter() - t0
    err = float(np.max(np.abs(phi.cpu().numpy()[idx].astype(np.float64) - ref) / D))
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        lpy.coulomb(P, P, Q, out=phi)
    torch.cuda.synchronize()
    per = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            lpy.coulomb(P, P, Q, out=phi)
            e1.record(stream)
            per.append((e0, e1))
        torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in per)
    pairs = float(n) * n
    peaks, src = load_peaks()
    mhz = peaks.get("sm_max_mhz", 1965.0)
    peak = 148 * 16 * mhz * 1e6       # MUFU.RSQ: 16 per clock per SM, one per pair
    achieved = pairs / (ms * 1e-3)
    return {"metric": "3D Coulomb potential pairs/s (self-potential, N^2 pairs per call)",
            "value": round(achieved / 1e6, 1), "unit": "M pairs/s", "n": n, "ms_per_call": round(ms, 4),
            "calls": args.steps, "gpu_launches": 3 * args.steps,
            "roofline": {"bound": "alu", "achieved": round(achieved / 1e12, 4), "peak": round(peak / 1e12, 4),
                         "unit": "T pairs/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "algorithmic_bytes": 16 * n + 16 * n,
                         "peak_note": f"MUFU.RSQ bound: 148 SM x 16/clk x {mhz} MHz ({src} clock), one rsqrt per pair"},
            "parity_sampled_max_norm_err": err,
            "cpu_baseline": {"value": round(idx.size * float(n) / cpu_dt / 1e6, 1), "unit": "M pairs/s",
                             "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": f"{idx.size} targets x {n} sources, float64"},
            "clocks": clk.summary(),
            "data": "synthetic: SplitMix64 positions uniform in [0,1)^3 (2^-23 grid), charges uniform[-1,1)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--path", default="auto", choices=["auto", "ffma", "3xtf32"])
    ap.add_argument("--also", default="ffma", help="secondary path to report ('' for none)")
    ap.add_argument("--chunks", type=int, default=0, help="K-row chunks of B for N>1 (0 = dist.choose_kchunks)")
    ap.add_argument("--bcast", default="root", choices=["root", "owners", "allgather"],
                    help="N>1: B starts on rank 0 and is broadcast (north_star), or starts sharded by "
                         "K-row chunks (chunk c on rank c mod N) and each owner broadcasts its chunks, or "
                         "rounds of N chunks are all-gathered (NCCL may run them as NVLS: --nccl-algo)")
    ap.add_argument("--graph", action="store_true",
                    help="N>1: capture the row-panel step (collectives, signals, gated product) as a CUDA graph "
                         "and replay it (dist.RowPanelGraph): one launch per step instead of one host call per chunk")
    ap.add_argument("--emulate-bcast-gbs", type=float, default=0.0,
                    help="diagnostics at N=1 with --force-dist: chunks 'arrive' at this rate (GB/s) through a "
                         "paced copy-engine copy into B (a projection, not a bench value)")
    ap.add_argument("--nccl-algo", default="",
                    help="N>1: NCCL_ALGO for the run (e.g. NVLS, Ring); default: NCCL's own choice")
    ap.add_argument("--reserve-sms", type=int, default=0,
                    help="N>1: SMs the gated product leaves to the collectives (0: dist.default_reserve of the path)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="diagnostics at N=1 with --force-dist: rank 0's panel of an N-rank split (not a bench value)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the row-panel + NCCL broadcast step even at N=1 (exercises the N>1 path)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=4.0, help="--impl reference: max seconds per step")
    ap.add_argument("--ref-total", type=float, default=120.0, help="--impl reference: target seconds for the run")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--saxpy-n", type=int, default=1 << 28, help="saxpy length (0 = skip the saxpy line)")
    ap.add_argument("--coulomb-n", type=int, default=1 << 16, help="Coulomb particles (0 = skip)")
    ap.add_argument("--no-context", action="store_true", help="skip the cuBLAS context timings")
    args = ap.parse_args()
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_1405_7470_b200 as lpy
    lpy.load_library()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist_on = world > 1 or args.force_dist
    if dist_on:
        import torch.distributed as dist
        if "MASTER_ADDR" not in os.environ:          # --force-dist without torchrun
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        # NCCL's INIT lines (rank / nRanks / transport per communicator) go to stderr,
        # where the launcher's rank check reads them
        if args.nccl_algo:
            os.environ["NCCL_ALGO"] = args.nccl_algo
        # (the chunk collectives run on dist.comm_group(reserve): a communicator
        # whose maxCTAs keeps NCCL inside the SMs the gated product leaves)
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # NCCL prints its debug lines (and the version banner) to stdout, at
        # communicator creation and destruction: fd 1 goes to stderr for the
        # whole distributed run and the JSON line is written to the saved
        # stdout, so stdout carries only that line
        sys.stdout.flush()
        JSON_OUT["fd"] = os.dup(1)
        os.dup2(2, 1)
        dist.init_process_group("nccl", device_id=device)
        dist.barrier()
        torch.cuda.synchronize()

    main_path = args.path
    if main_path == "auto":
        _, chosen = lpy.lpy_select_path(args.n, args.n, args.n, lpy.PATH_AUTO)
        main_path = {1: "ffma", 2: "3xtf32"}[chosen]
    res = time_path(args, main_path, rank, world, device, dist_on)
    also = None
    if args.also and args.also != main_path:
        also = time_path(args, args.also, rank, world, device, dist_on)
    e2e = None if args.no_e2e else time_e2e(args, main_path, rank, world, device, dist_on)
    sax = time_saxpy(args, device) if (args.saxpy_n > 0 and rank == 0 and not dist_on) else None
    coul = time_coulomb(args, device) if (args.coulomb_n > 0 and rank == 0 and not dist_on) else None
    ctx = time_cublas_context(args, device) if (not args.no_context and rank == 0 and not dist_on) else None

    if rank == 0:
        n = args.n
        flops = 2.0 * n ** 3
        if dist_on and args.emulate_ranks and world == 1:
            flops /= args.emulate_ranks      # diagnostics: rank 0's panel of an N-rank split only
        ms = res["total_ms"] / args.steps
        value = flops / (ms * 1e-3) / 1e9

        def roof(r, path):
            bound, peak, note = roofline_peak(path)
            if not dist_on:        # one GEMM launch per step: its CUDA-event time
                kms, kflops = statistics.mean(r["kernel_ms"]), flops
            else:                  # rank 0's panel product alone (ungated, same plan), no broadcast
                kms, kflops = r["multi"]["gemm_ms"], flops / world
            achieved = kflops / (kms * 1e-3) / 1e12
            traffic, tsrc = profile_traffic(path, n)
            return {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3),
                    "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                    "traffic_source": tsrc, "algorithmic_bytes": 4 * 3 * n * n,
                    "peak_note": note, "kernel_ms_mean": round(kms, 4)}

        cpu = None
        if not args.no_cpu:
            # rank 0's host cores at every N (the other ranks wait at the final barrier)
            gf, dt, sample, threads = oracle_sample(n, args.cpu_seconds, "uniform", nthreads=host_cores())
            cpu = {"value": round(gf, 3), "unit": UNIT, "cores": threads, "kind": "oracle",
                   "sample": sample, "seconds": round(dt, 2), "cpu_model": cpu_model()}
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            # the arithmetic the path computes in: three tf32 tensor-core products per
            # fp32 product, fp32 accumulation (fp32-accurate: <= 1e-5 normalised error
            # vs the float64 oracle), or plain fp32 FMAs on the SIMT path
            "dtype": "tf32x3+f32acc" if res["path"] == "3xtf32" else "f32",
            "data": "synthetic: seeded SplitMix64 uniform[-1,1) fp32 on a 2^-23 grid",
            "config": {"workload": f"n={n} square fp32 C=A*B, row-major A/B/C (BASELINE config 4)",
                       "path": res["path"], "M": n, "N": n, "K": n,
                       "parallelism": f"rowpanel{world}" + (f"+nccl_{args.bcast}_B_kchunks{res['chunks']}" + "+gated_product" if dist_on else ""),
                       "l2": "inputs larger than L2 (A, B, C 268 MB each > 126 MB), no flush"},
            "roofline": roof(res, res["path"]),
            "cpu_baseline": cpu,
            "e2e": ({k: (round(v, 3) if isinstance(v, float) else v) for k, v in e2e.items()}
                    if e2e else None),
            "gpu_launches": res["launches_per_step"] * args.steps,
            "clocks": res["clocks"],
            "parity_sampled_max_norm_err": res["parity"],
        }
        if dist_on:
            line["multi_gpu"] = res["multi"]
        if sax is not None:
            line["saxpy"] = sax
        if coul is not None:
            line["coulomb"] = coul
        if ctx is not None:
            line["context_cublas"] = ctx
        if also is not None:
            ams = also["total_ms"] / args.steps
            line["alt_path"] = {"path": also["path"], "value": round(flops / (ams * 1e-3) / 1e9, 1),
                                "ms_per_step": round(ams, 4), "roofline": roof(also, also["path"]),
                                "parity_sampled_max_norm_err": also["parity"], "clocks": also["clocks"]}
        emit(line)
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
