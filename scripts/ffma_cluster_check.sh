#!/bin/bash
# FFMA cluster split (DSMEM reduction of split-K slices in a single wave): parity, A/B timing.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
for v in 0 1; do LPY_FFMA_CLUSTER=$v timeout 300 python scripts/small_shapes.py ffma > gpurun_out/small_ffma_c$v.txt 2>&1; done
LPY_FFMA_CLUSTER=0 timeout 120 python scripts/det_probe.py ffma 1024 1024 1024 > /dev/null 2>&1
