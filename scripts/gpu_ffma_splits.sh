#!/bin/bash
# FFMA split-K factor on the split-K shapes (config 5 at BN=128; n=1024 cluster split): LPY_FFMA_SPLITS=S forced,
# stream-K off so the split is what runs; each S in its own process, twice.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/ffma_splits.txt
: > $O
S="1000,3000,780,row,col;1000,3000,780,col,row;1000,3000,777,row,col;1024,1024,1024,row,row;4096,4096,1024,row,row"
for rep in 1 2; do
for v in 0 2 3 4 5 6 8; do
  echo "== LPY_FFMA_SPLITS=$v (run $rep)" >> $O
  LPY_FFMA_STREAMK=0 LPY_FFMA_SPLITS=$v SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py ffma paper_1405_7470_b200/liblpy.so 2>&1 | awk '{print $2, $3, $4}' >> $O
done; done
