#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/ffma_tile_ab.py > gpurun_out/ffma_tile.txt 2>&1
