#!/bin/bash
# ncu --set full of the FFMA kernel after the transpose fix: n=8192 row-major (the bench's alt path) and the
# under-filled configs (n=1024 row/row, config 5 ld=780) -- summaries via scripts/ncu_summary.py.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 1 -c 1 \
   -o gpurun_out/prof_ffma_n8192_new python scripts/cfg_gemm.py ffma 8192 8192 8192 row row 0 2 > gpurun_out/ncu_a.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 2 -c 1 \
   -o gpurun_out/prof_ffma_n1024_new python scripts/cfg_gemm.py ffma 1024 1024 1024 row row 0 4 > gpurun_out/ncu_b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 2 -c 1 \
   -o gpurun_out/prof_ffma_cfg5_new python scripts/cfg_gemm.py ffma 1000 3000 777 row col 3 4 > gpurun_out/ncu_c.log 2>&1
