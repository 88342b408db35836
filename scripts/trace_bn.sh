#!/bin/bash
# Role-wait traces of the 3xTF32 kernel for each tile width at n=8192.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for bn in 256 192 128; do
  echo "== BN=$bn" >> gpurun_out/trace_bn.txt
  LPY_TF32_BN=$bn timeout 300 python scripts/trace_tf32.py 8192 >> gpurun_out/trace_bn.txt 2>&1
done
