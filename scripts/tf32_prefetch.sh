#!/bin/bash
mkdir -p gpurun_out
for pf in 0 4 8 16 32; do
  echo "== prefetch=$pf" >> gpurun_out/pf.txt
  LPY_TF32_PREFETCH=$pf timeout 120 python scripts/trace_tf32.py 8192 >> gpurun_out/pf.txt 2>&1
done
timeout 300 python bench.py --path 3xtf32 --also "" --no-cpu > gpurun_out/bench.json 2>&1
