"""Where the gated row-panel step's time goes at world 1 (emulated g=8 panel,
1024 x 8192 x 8192): ungated product (plan 140), gated product with flags
already raised, gemm_rowpanel with 4/8/16 chunks; device time per step over
back-to-back steps (CUDA events on the caller stream)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_1405_7470_b200 as lpy
from paper_1405_7470_b200 import dist as ld

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29561")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
path = sys.argv[1] if len(sys.argv) > 1 else "3xtf32"
M, N, K = 1024, 8192, 8192
A = torch.rand(M, K, device="cuda") * 2 - 1
B = torch.rand(K, N, device="cuda") * 2 - 1
C = torch.empty(M, N, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count


def bench(variants, rounds=7, reps=10):
    """Interleaved A/B: every round times each variant once (reps back-to-back
    calls), so clock / power drift hits all variants alike; median per variant."""
    for fn in variants.values():
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    res = {k: [] for k in variants}
    for _ in range(rounds):
        for k, fn in variants.items():
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            res[k].append(a.elapsed_time(b) / reps)
    for k, v in res.items():
        print(f"{k:32s} median {statistics.median(v):.4f} ms  min {min(v):.4f}  ({' '.join(f'{x:.3f}' for x in v)})",
              flush=True)


o8 = ld.panel_opts(sms, 8)
flags = torch.full((64,), 5, dtype=torch.int32, device="cuda")
g = lpy.KGate(flags.data_ptr(), 512, 5, 0)
variants = {
    "full chip ungated": lambda: lpy.gemm(A, B, out=C, path=path),
    "plan140 ungated": lambda: lpy.gemm(A, B, out=C, path=path, opts=o8),
    "plan140 gated, flags ready": lambda: lpy.gemm(A, B, out=C, path=path, opts=o8, gate=g),
}
for ch in (4, 8, 16):
    variants[f"rowpanel chunks {ch}"] = (lambda ch=ch: ld.gemm_rowpanel(A, B, chunks=ch, path=path, out=C,
                                                                        reserve_sms=8, timings=False))
if len(sys.argv) > 2 and sys.argv[2] == 'short':
    bench(variants, rounds=2, reps=2)
else:
    bench(variants)
dist.destroy_process_group()
