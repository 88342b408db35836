#!/bin/bash
# A/B the CTA-pair vs single-CTA 3xTF32 kernels and capture an ncu profile of the pair kernel.
mkdir -p gpurun_out
for cg in 1 2; do
  LPY_TF32_CG=$cg timeout 300 python bench.py --path 3xtf32 --also "" --no-cpu --no-parity --steps 20 > gpurun_out/bench_cg$cg.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 3 -c 1 \
    -o gpurun_out/prof_cg2 python bench.py --path 3xtf32 --also "" --steps 1 --warmup 3 --no-cpu --no-parity > gpurun_out/ncu_cg2.log 2>&1
