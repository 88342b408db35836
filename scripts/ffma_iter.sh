#!/bin/bash
# FFMA iteration: build, FFMA parity (not slow), per-layout and per-config timings.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "ffma and not slow" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt; tail -2 gpurun_out/parity.log >> gpurun_out/summary.txt
timeout 300 python scripts/layouts_bench.py > gpurun_out/layouts.txt 2>&1
timeout 300 python scripts/configs_bench.py > gpurun_out/configs.txt 2>&1
