#!/usr/bin/env python
"""Sustained 3xTF32 n=8192 products back to back for ~3 s with nvidia-smi
sampling power, SM clock and throttle reasons every 10 ms; reports the
achieved TFLOP/s per second of the run beside the median clock and power, and
the tensor-pipe share that implies at that clock (6 n^3 tf32 MMA flops per
product / (148 SMs x 4096 flop/clk x clock)).
usage: python scripts/power_probe.py [path] [seconds]"""
import os, subprocess, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1405_7470_b200 as lpy

path = sys.argv[1] if len(sys.argv) > 1 else "3xtf32"
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
n = 8192
A = torch.rand(n, n, device="cuda") * 2 - 1
B = torch.rand(n, n, device="cuda") * 2 - 1
C = torch.empty(n, n, device="cuda")
for _ in range(3):
    lpy.gemm(A, B, out=C, path=path)
torch.cuda.synchronize()
time.sleep(2.0)          # cool down before the sampled run
out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,power.draw,power.limit,clocks.sm,temperature.gpu,"
                        "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
                        "clocks_event_reasons.sw_thermal_slowdown", "--format=csv,noheader,nounits", "-lms", "10"],
                       stdout=out, stderr=subprocess.DEVNULL)
time.sleep(0.3)
evs = []
t_end = time.time() + secs
while time.time() < t_end:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lpy.gemm(A, B, out=C, path=path)
    e1.record()
    evs.append((e0, e1))
    e1.synchronize()
time.sleep(0.2)
smi.terminate()
smi.wait()
ms = [a.elapsed_time(b) / 10 for a, b in evs]
rows = [l.strip().split(", ") for l in open(out.name) if l.strip()]
os.unlink(out.name)
pw = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
lim = rows[0][2] if rows else "?"
clk = [float(r[3]) for r in rows if r[3].isdigit()]
cap = sum(1 for r in rows if r[5].strip() == "Active")
print(f"{path} n={n}: {len(ms)} batches of 10; per-product ms first {ms[0]:.3f} median {sorted(ms)[len(ms)//2]:.3f} "
      f"last {ms[-1]:.3f}")
print(f"  TFLOP/s first {2*n**3/ms[0]/1e9:.1f} median {2*n**3/sorted(ms)[len(ms)//2]/1e9:.1f} last {2*n**3/ms[-1]/1e9:.1f}")
loaded = [c for c in clk if c > 500]
p_loaded = sorted(pw)[len(pw) // 2] if pw else 0
cmed = sorted(loaded)[len(loaded) // 2] if loaded else 0
print(f"  nvidia-smi: {len(rows)} samples, power median {p_loaded:.0f} W max {max(pw) if pw else 0:.0f} W "
      f"(limit {lim} W), SM clock median {cmed:.0f} MHz min {min(loaded) if loaded else 0:.0f} "
      f"max {max(loaded) if loaded else 0:.0f}, sw_power_cap active in {cap}/{len(rows)} samples")
if path == "3xtf32" and cmed:
    med = sorted(ms)[len(ms) // 2]
    util = 6.0 * n ** 3 / (med * 1e-3) / (148 * 4096 * cmed * 1e6)
    print(f"  tensor-pipe share at the median clock: 6 n^3 / (148 x 4096 x {cmed:.0f} MHz x {med:.3f} ms) = {util:.3f}")
for r in rows[:: max(1, len(rows) // 12)]:
    print("   ", ", ".join(r))
