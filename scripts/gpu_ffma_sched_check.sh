#!/bin/bash
# FFMA schedule after the stream-K minimum-piece change: auto (1) vs split-K (0) vs forced stream-K (2) on the
# small / mid shapes, each in its own process, twice; the GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/ffma_sched_check.txt
: > $O
S="1000,3000,780,row,col;1000,3000,780,col,row;1000,3000,777,row,col;2048,2048,2048,row,row;1536,2048,2048,row,row;1024,1024,1024,row,row;2048,4096,2048,row,row;3000,5000,1000,row,row;4096,4096,1024,row,row;2048,2048,8192,row,row"
for rep in 1 2; do
for e in "LPY_FFMA_STREAMK=1" "LPY_FFMA_STREAMK=0" "LPY_FFMA_STREAMK=2"; do
  echo "== $e (run $rep)" >> $O
  env $e SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py ffma paper_1405_7470_b200/liblpy.so 2>&1 | awk '{print $2, $3, $4}' >> $O
done; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
