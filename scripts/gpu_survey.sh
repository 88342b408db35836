#!/bin/bash
# Per-config timings on both paths, per-layout FFMA timings, and an ncu full capture of the FFMA kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/configs_bench.py > gpurun_out/configs.txt 2>&1
timeout 300 python scripts/layouts_bench.py > gpurun_out/layouts.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 3 -c 1 -o gpurun_out/prof_ffma python bench.py --path ffma --also "" --steps 1 --warmup 3 --no-cpu --no-parity > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
