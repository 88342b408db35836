#!/bin/bash
# ncu --set full (with source) of the 3xTF32 kernel on the narrow-tile configs: n=1024 (BN=128,
# 4-CTA cluster split) and config 5 (1000x3000x780, BN=192, col-major B).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # tag args...
  tag=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 \
     -o gpurun_out/prof_$tag python scripts/cfg_gemm.py "$@" > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?" >> gpurun_out/summary.txt
}
run tf32_n1024_rr 3xtf32 1024 1024 1024 row row
run tf32_cfg5_ld780 3xtf32 1000 3000 777 row col 3
