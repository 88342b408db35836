#!/bin/bash
# ncu --set full of the n=128 and n=1024 FFMA launches (fixed overheads of small problems).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 2 -c 1 -o gpurun_out/prof_ffma128 python scripts/one_gemm.py ffma 128 row row 4 > gpurun_out/ncu128.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 2 -c 1 -o gpurun_out/prof_ffma1024 python scripts/one_gemm.py ffma 1024 row row 4 > gpurun_out/ncu1024.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
