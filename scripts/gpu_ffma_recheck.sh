#!/bin/bash
# After the transpose fix: FFMA width / schedule choices re-checked (tile probe, both shape lists), then the
# end-of-round evidence (scripts/gpu_r02_final.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/ffma_tile_probe.py > gpurun_out/ffma_tile_recheck.txt 2>&1
CASES=wide timeout 900 python scripts/ffma_tile_probe.py >> gpurun_out/ffma_tile_recheck.txt 2>&1
bash scripts/gpu_r02_final.sh
