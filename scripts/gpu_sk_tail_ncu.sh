#!/bin/bash
# Stream-K tail threshold A/B by ncu kernel durations (serialised launches, free clocks).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in 0.8 0.9; do
for plan in 140 144 148; do
LPY_TF32_SK_TAIL=$t PLAN_SMS=$plan timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/sk_${t}_$plan.csv python scripts/shapes_time.py 3xtf32 1024,8192,8192 2048,8192,8192 > /dev/null 2>&1
done
LPY_TF32_SK_TAIL=$t timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/sk_${t}_n8192.csv python scripts/shapes_time.py 3xtf32 8192,8192,8192 > /dev/null 2>&1
done
