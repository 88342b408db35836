#!/bin/bash
# After the FFMA width rule change: the same probes (tile_n=0 must now match the faster width), the GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/ffma_tile_probe.py > gpurun_out/ffma_tile_probe_after.txt 2>&1
CASES=wide timeout 900 python scripts/ffma_tile_probe.py >> gpurun_out/ffma_tile_probe_after.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
