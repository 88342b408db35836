#!/bin/bash
# FFMA split-K partial layout A/B (LPY_FFMA_PARTIAL=contig vs interleaved default), interleaved runs.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2 3; do for v in contig inter; do
  echo "== $v $r"; LPY_FFMA_PARTIAL=$v SHAPES="cfg5,n=2048,n=512" timeout 300 python scripts/small_shapes.py ffma | grep -v config
done; done > gpurun_out/partial_ab.txt 2>&1
