#!/bin/bash
# 3xTF32 per-flop efficiency by tile width (LPY_TF32_BN forces it), ncu launch durations (serialised).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for bn in 256 192 128; do
LPY_TF32_BN=$bn timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/bn_$bn.csv python scripts/shapes_time.py 3xtf32 8192,8192,8192 > /dev/null 2>&1
done
for bn in 256 192 128; do python scripts/ncu_durations.py gpurun_out/bn_$bn.csv | grep gemm_3xtf32 | sed "s/^/BN=$bn /"; done > gpurun_out/bn_sweep.txt
