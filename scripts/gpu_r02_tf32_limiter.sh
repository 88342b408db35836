#!/bin/bash
# 3xTF32 n=8192: what bounds it at full clock.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/power_probe.py 3xtf32 3 > gpurun_out/power_3xtf32.txt 2>&1
timeout 300 python scripts/power_probe.py ffma 3 > gpurun_out/power_ffma.txt 2>&1
for cc in none base; do
timeout 900 ncu --set full --clock-control $cc --import-source on -k regex:gemm_3xtf32 -s 3 -c 1 \
   -o gpurun_out/prof_3xtf32_$cc python scripts/one_gemm.py 3xtf32 8192 row row 5 > gpurun_out/ncu_3xtf32_$cc.log 2>&1
done
