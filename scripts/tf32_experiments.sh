#!/bin/bash
# 3xTF32 bottleneck experiments with the diagnostics build (results are numerically
# wrong by design for EXP != 0; timing only).
mkdir -p gpurun_out
for exp in 0 1 2 3; do
  echo "== LPY_TF32_EXP=$exp" >> gpurun_out/exp.txt
  LPY_TF32_EXP=$exp timeout 120 python scripts/trace_tf32.py 8192 >> gpurun_out/exp.txt 2>&1
done
python scripts/layouts_bench.py >> gpurun_out/exp.txt 2>&1
