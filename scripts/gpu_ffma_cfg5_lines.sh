#!/bin/bash
# ncu --set full with source of the FFMA kernel on config 5 (ld=780, A row, B col) and n=8192 row-major,
# for the per-source-line stall split (scripts/ncu_lines.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 1 -c 1 \
   -o gpurun_out/prof_ffma_cfg5 python scripts/cfg_gemm.py ffma 1000 3000 777 row col 3 2 > gpurun_out/ncu_ffma_cfg5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 0 -c 1 \
   -o gpurun_out/prof_ffma_n8192 python scripts/cfg_gemm.py ffma 8192 8192 8192 row row 0 1 > gpurun_out/ncu_ffma_n8192.log 2>&1
