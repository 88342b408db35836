#!/bin/bash
# Role-wait traces of the 3xTF32 kernel for each A/B layout at n=8192.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for la in row col; do for lb in row col; do
  echo "== A $la B $lb" >> gpurun_out/trace_layouts.txt
  LA=$la LB=$lb timeout 300 python scripts/trace_tf32.py 8192 >> gpurun_out/trace_layouts.txt 2>&1
done; done
