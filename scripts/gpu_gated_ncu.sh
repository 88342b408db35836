#!/bin/bash
# Kernel durations (ncu, free clocks) of ungated vs gated panel products + interleaved device timing.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCCL_DEBUG=WARN timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/gated_ncu_none.csv python scripts/gated_probe.py 3xtf32 short > gpurun_out/gated_ncu_none.log 2>&1
for p in 3xtf32 ffma; do echo "== $p"; NCCL_DEBUG=WARN timeout 300 python scripts/gated_probe.py $p 2>&1 | grep -v Warning; done > gpurun_out/gated_probe.txt 2>&1
