#!/bin/bash
# Panel product (1024 x 8192 x 8192) planned for 148 / 140 / 132 / 124 / 116 SMs: ncu launch durations.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for plan in 148 140 132 124 116; do for p in 3xtf32 ffma; do
PLAN_SMS=$plan timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/plan_${p}_$plan.csv python scripts/shapes_time.py $p 1024,8192,8192 > /dev/null 2>&1
done; done
for f in gpurun_out/plan_*.csv; do python scripts/ncu_durations.py $f | grep gemm; done > gpurun_out/plan_sweep.txt 2>&1
