#!/bin/bash
# More L2 eviction-hint variants (LPY_L2HINT 3/4/5) at the default raster group: DRAM bytes (ncu) and time.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for h in 0 3 4 5; do
  REPS=1 LPY_L2HINT=$h timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_3xtf32 --csv python scripts/l2_ab.py 8192 8 > gpurun_out/l2b_ncu_$h.csv 2>&1
done
for h in 0 3 4 5 0 3 4 5; do LPY_L2HINT=$h python scripts/l2_ab.py 8192 8; done > gpurun_out/l2b_time.txt 2>&1
