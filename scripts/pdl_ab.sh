#!/bin/bash
# Interleaved PDL A/B on the shapes where it looked worse (FFMA ragged config with split-K fix-up; 3xTF32 long-K single wave).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2 3; do for v in 0 1; do
  echo "== PDL=$v round $r"
  LPY_PDL=$v SHAPES="ld=780,2048x2048x8192,n=128" timeout 300 python scripts/small_shapes.py | grep -v config
done; done > gpurun_out/pdl_ab.txt 2>&1
