#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "ffma and not slow" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt; tail -2 gpurun_out/parity.log >> gpurun_out/summary.txt
timeout 300 python bench.py --path ffma --also "" --no-cpu --steps 20 > gpurun_out/bench.json 2>&1
echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 300 python scripts/layouts_bench.py > gpurun_out/layouts.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 3 -c 1 -o gpurun_out/prof_ffma python bench.py --path ffma --also "" --steps 1 --warmup 3 --no-cpu --no-parity > gpurun_out/ncu.log 2>&1
