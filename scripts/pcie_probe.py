#!/usr/bin/env python
"""Host<->device copy bandwidth on this box (pinned buffers): H2D alone, D2H
alone, and both directions at once -- the ceiling for bench.py's e2e number."""
import torch

MB = 256
h = torch.empty(MB * 2 ** 20 // 4, dtype=torch.float32).pin_memory()
h2 = torch.empty_like(h).pin_memory()
d = torch.empty(h.numel(), device="cuda")
d2 = torch.empty(h.numel(), device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d.copy_(h, non_blocking=True)


def d2h():
    h2.copy_(d2, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
print(f"H2D {MB / t_h2d:.1f} GB/s  D2H {MB / t_d2h:.1f} GB/s  "
      f"both-directions {2 * MB / t_both:.1f} GB/s aggregate ({t_h2d:.2f} / {t_d2h:.2f} / {t_both:.2f} ms)")
