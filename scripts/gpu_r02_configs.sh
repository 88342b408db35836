#!/bin/bash
# Final round-2 per-config tables: eager L2-flushed (configs_bench.py) and graph-replayed (small_shapes.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python scripts/configs_bench.py > gpurun_out/configs.txt 2>&1
timeout 900 python scripts/small_shapes.py > gpurun_out/small_shapes.txt 2>&1
