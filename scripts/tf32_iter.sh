#!/bin/bash
# 3xTF32 iteration: parity (not slow), per-config timings, A/B vs liblpy_old.so at n=4096 and 8192.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt; tail -2 gpurun_out/parity.log >> gpurun_out/summary.txt
timeout 300 python scripts/configs_bench.py > gpurun_out/configs.txt 2>&1
for n in 4096 8192; do
  ROUNDS=3 timeout 300 python scripts/ab_lib.py 3xtf32 $n paper_1405_7470_b200/liblpy_old.so paper_1405_7470_b200/liblpy.so > gpurun_out/ab_tf32_$n.txt 2>&1
done
