#!/bin/bash
# FFMA schedule switches on the small shapes after the width change: stream-K off / auto / forced, cluster
# split off, fix-up parts; each setting in its own process (the switches are read once), twice, alternating.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/ffma_sched_env.txt
: > $O
S="1000,3000,780,row,col;1000,3000,780,col,row;1000,3000,777,row,col;2048,2048,2048,row,row;1536,2048,2048,row,row;1024,1024,1024,row,row"
for rep in 1 2; do
for e in "LPY_FFMA_STREAMK=1" "LPY_FFMA_STREAMK=0" "LPY_FFMA_STREAMK=2" "LPY_FFMA_CLUSTER=0" "LPY_FFMA_MINKB=4" "LPY_FFMA_FIXUP_PARTS=4"; do
  echo "== $e (run $rep)" >> $O
  env $e SHAPES="$S" timeout 600 python scripts/ab_libs_cfg.py ffma paper_1405_7470_b200/liblpy.so 2>&1 | awk '{print $2, $3, $4}' >> $O
done; done
