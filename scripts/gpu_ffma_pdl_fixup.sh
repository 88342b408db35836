#!/bin/bash
# FFMA split-K fix-up launched with programmatic dependent launch (working tree) vs liblpy_head.so (the previous
# commit's build, built separately and shipped with the tree): split-K shapes, interleaved; the GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
S="1000,3000,780,row,col;1000,3000,780,col,row;1000,3000,777,row,col;2048,2048,2048,row,row;1024,1024,1024,row,row"
for i in 1 2; do
SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py ffma paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_head.so > gpurun_out/ab_pdl_fixup_$i.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
