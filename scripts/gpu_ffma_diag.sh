#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/ffma_diag.txt
for spec in "1024 1024 1024 row row" "1024 1024 1024 col col" "1000 3000 780 row col" "2048 2048 2048 row row"; do
 for tn in 0 128 256; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/ffma_tile_diag.py $spec $tn >> $O 2>&1
 done
done
FIRST=$(grep FAIL $O | head -1 | awk '{print $2}')
if [ -n "$FIRST" ]; then
  L=$(grep FAIL $O | head -1)
  echo "sanitizer on: $L" >> $O
  set -- $(echo $L | sed 's/x/ /g; s/tile_n=//; s/plan=//; s/://g' | awk '{print $2, $3, $4, substr($5,1,3), substr($5,4), $6}')
  timeout 600 compute-sanitizer --tool memcheck python scripts/ffma_tile_diag.py $1 $2 $3 $4 $5 $6 2>&1 | head -40 >> $O
fi
