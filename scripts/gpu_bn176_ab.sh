#!/bin/bash
# choose_bn with 176-wide tiles (working tree) vs the previous commit's build (liblpy_head.so, shipped with the
# tree) on K-major A / B shapes of several widths, interleaved, twice.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
S="1000,3000,780,row,col;1000,3000,777,row,col;2000,2800,1000,row,col;300,5000,2000,row,col;1024,1024,1024,row,col;2048,2048,2048,row,col;4096,4096,4096,row,col;1500,1500,1500,row,col;3000,1000,2000,row,col;8192,8192,8192,row,col"
for i in 1 2; do
SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py 3xtf32 paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_head.so > gpurun_out/ab_bn176_$i.txt 2>&1
done
