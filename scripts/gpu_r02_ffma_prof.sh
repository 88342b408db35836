#!/bin/bash
# ncu evidence for the under-filled FFMA configs: launch lists and --set full
# captures of the FFMA kernel at n=1024 (config 2), config 5 (1000x3000x777, col-major B) and n=2048.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # tag args...
  tag=$1; shift
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$tag.csv \
     python scripts/cfg_gemm.py "$@" > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 2 -c 1 \
     -o gpurun_out/prof_$tag python scripts/cfg_gemm.py "$@" > gpurun_out/ncu_$tag.log 2>&1
  echo "$tag rc=$?" >> gpurun_out/summary.txt
}
run ffma_n1024_rr ffma 1024 1024 1024 row row
run ffma_n1024_cc ffma 1024 1024 1024 col col
run ffma_cfg5_ld777 ffma 1000 3000 777 row col 0
run ffma_cfg5_ld780 ffma 1000 3000 777 row col 3
run ffma_n2048 ffma 2048 2048 2048 row row
