#!/bin/bash
# A/B of the current library against variant / earlier-commit builds (liblpy_*.so shipped in the tree).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SHAPES=${SHAPES:-"1000,3000,777,row,col;1000,3000,780,col,col;1024,1024,1024,row,row;2048,2048,2048,row,row;1024,8192,8192,row,row"} \
  timeout 900 python scripts/ab_libs_cfg.py ${1:-3xtf32} paper_1405_7470_b200/liblpy.so ${@:2} > gpurun_out/ab_commits.txt 2>&1
