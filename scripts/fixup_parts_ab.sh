#!/bin/bash
# FFMA split-K fix-up: CTAs per tile (LPY_FFMA_FIXUP_PARTS) A/B on the multi-wave split shapes.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do for v in 4 8 2; do echo "== parts $v"; LPY_FFMA_FIXUP_PARTS=$v SHAPES="cfg5,n=2048,2048x2048x8192" timeout 300 python scripts/small_shapes.py ffma | grep -v config; done; done > gpurun_out/parts_ab.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "ffma" -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
