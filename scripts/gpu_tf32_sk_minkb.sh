#!/bin/bash
# 3xTF32 stream-K tail on shorter k loops: LPY_TF32_SK_MINKB = 256 (default: K >= 4096) vs 128 (K >= 2048) vs 64,
# each in its own process, alternating, three times (CUDA-graph replay via scripts/ab_libs_cfg.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/tf32_sk_minkb.txt
: > $O
S="2048,4096,2048,row,row;3000,5000,1000,row,row;2560,2304,2048,row,row;4096,4096,2048,row,row;1024,8192,2048,row,row;2048,2048,2048,row,row"
for rep in 1 2 3; do
for v in 256 128 64; do
  echo "== LPY_TF32_SK_MINKB=$v (run $rep)" >> $O
  LPY_TF32_SK_MINKB=$v SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py 3xtf32 paper_1405_7470_b200/liblpy.so 2>&1 | awk '{print $2, $3, $4}' >> $O
done; done
