#!/bin/bash
# 3xTF32 176-wide tiles (K-major A and B) on config 5: parity (every element vs float64), forced widths vs choose_bn,
# race detector, the GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/bn176.txt
: > $O
for bn in 0 176 192; do
  echo "== LPY_TF32_BN=$bn" >> $O
  LPY_TF32_BN=$bn SHAPES="1000,3000,780,row,col;1000,3000,777,row,col;1000,3000,780,row,col;2000,2800,1000,row,col;300,5000,2000,row,col" \
    timeout 600 python scripts/ab_libs_cfg.py 3xtf32 paper_1405_7470_b200/liblpy.so 2>&1 | awk '{print $2, $3, $4, $7, $8}' >> $O
done
timeout 300 python scripts/race_lib.py product 3xtf32 4 "1000,3000,780;1000,3000,777;2000,2800,1000" > gpurun_out/race_bn176.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
