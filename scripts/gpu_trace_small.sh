#!/bin/bash
# 3xTF32 per-role cycle shares and CTA-0 timelines on the small configs (diagnostics build).
# GRID = the CTAs the product launches (config 5: 64 pair tiles; n=1024: 32 tiles x 4-CTA clusters).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/trace_small.txt
: > $O
for s in "1000,3000,780" "1000,3000,777" "1024"; do
  echo "== $s (A row, B col)" >> $O
  GRID=128 LB=col timeout 120 python scripts/trace_tf32.py $s >> $O 2>&1
done
echo "== 1024 row/row" >> $O
GRID=128 timeout 120 python scripts/trace_tf32.py 1024 >> $O 2>&1
