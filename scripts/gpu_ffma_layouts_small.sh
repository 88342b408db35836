#!/bin/bash
# FFMA under-filled shapes in all four A/B layouts (graph replay): how much the transposes of K-major tiles cost.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
S="1000,3000,780,row,row;1000,3000,780,row,col;1000,3000,780,col,row;1000,3000,780,col,col;1024,1024,1024,row,row;1024,1024,1024,col,row;2048,2048,2048,row,row;2048,2048,2048,col,row"
SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py ffma paper_1405_7470_b200/liblpy.so > gpurun_out/ffma_layouts_small.txt 2>&1
