#!/bin/bash
# Iteration loop for 3xTF32 tuning: trace (diagnostics build), short parity, bench, accuracy.
mkdir -p gpurun_out
timeout 120 python scripts/trace_tf32.py 8192 > gpurun_out/trace.txt 2>&1
timeout 120 python scripts/trace_tf32.py 8192 16 >> gpurun_out/trace.txt 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "3xtf32 and not slow" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt; tail -2 gpurun_out/parity.log >> gpurun_out/summary.txt
timeout 300 python bench.py --path 3xtf32 --also "" --no-cpu > gpurun_out/bench.json 2>&1
echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 600 python scripts/accuracy_tf32.py 8192 > gpurun_out/accuracy.txt 2>&1
