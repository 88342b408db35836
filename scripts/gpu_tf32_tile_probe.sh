#!/bin/bash
# 3xTF32 tile width (opts.tile_n 128 / 192 / 256 vs choose_bn) on small and mid-size shapes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
PATH_=3xtf32 timeout 600 python scripts/ffma_tile_probe.py > gpurun_out/tf32_tile_probe.txt 2>&1
PATH_=3xtf32 CASES=wide timeout 900 python scripts/ffma_tile_probe.py >> gpurun_out/tf32_tile_probe.txt 2>&1
