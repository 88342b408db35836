#!/bin/bash
# A/B of liblpy.so vs liblpy_$1.so on the 3xTF32 path (n = 4096, 8192) + 3xTF32 parity.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "3xtf32 and not slow" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt; tail -1 gpurun_out/parity.log >> gpurun_out/summary.txt
for n in 8192 4096; do
  ROUNDS=3 timeout 300 python scripts/ab_lib.py 3xtf32 $n paper_1405_7470_b200/liblpy_$1.so paper_1405_7470_b200/liblpy.so >> gpurun_out/summary.txt 2>&1
done
