#!/bin/bash
mkdir -p gpurun_out
for exp in 0 4 5 6; do
  echo "== exp=$exp" >> gpurun_out/exp.txt
  LPY_TF32_EXP=$exp timeout 120 python scripts/trace_tf32.py 8192 >> gpurun_out/exp.txt 2>&1
  LPY_TF32_EXP=$exp LPY_TF32_CG=1 timeout 120 python scripts/trace_tf32.py 8192 >> gpurun_out/exp.txt 2>&1
done
