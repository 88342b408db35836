#!/bin/bash
# Round-2 baseline on one B200: build, smoke, full GPU suite, bench, g=8 emulation, multicast probe.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
nvidia-smi topo -m >> gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> $S
tail -3 gpurun_out/parity.log >> $S
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> $S
for p in 3xtf32 ffma; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --path $p --also "" --no-e2e --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/emul8_$p.json 2> gpurun_out/emul8_$p.err; echo "emul8 $p rc=$?" >> $S
done
timeout 120 python - > gpurun_out/mc_probe.txt 2>&1 <<'PY'
import torch, ctypes
from cuda.bindings import driver as d
d.cuInit(0)
err, dev = d.cuDeviceGet(0)
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    try:
        print(a, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev))
    except Exception as e:
        print(a, "ERR", e)
import os
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29555")
import torch.distributed as dist
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda",0))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1<<20, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("symm ok multicast_ptr", getattr(h, "multicast_ptr", None), "world", h.world_size)
except Exception as e:
    print("symm ERR", repr(e))
dist.destroy_process_group()
PY
cat gpurun_out/bench.json >> $S
cat gpurun_out/emul8_*.json >> $S
cat gpurun_out/mc_probe.txt >> $S
