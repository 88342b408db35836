#!/bin/bash
# L2 eviction-hint x raster-group A/B for the 3xTF32 kernel at n=8192: timing, then DRAM bytes (ncu).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
G="4 6 8 10 12"
for h in 0 1 2; do LPY_L2HINT=$h python scripts/l2_ab.py 8192 $G; done > gpurun_out/l2_ab.txt 2>&1
for h in 0 1 2; do LPY_L2HINT=$h python scripts/l2_ab.py 8192 $G; done >> gpurun_out/l2_ab.txt 2>&1
for h in 0 1 2; do
  REPS=1 LPY_L2HINT=$h timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_3xtf32 --csv python scripts/l2_ab.py 8192 $G > gpurun_out/l2_ncu_$h.csv 2>&1
done
