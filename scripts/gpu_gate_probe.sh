#!/bin/bash
# Diagnostics of the K-gated product with late flags (scripts/gate_probe.py).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in ffma 3xtf32; do for m in nosleep sleep; do echo "== $p $m"; timeout 60 python scripts/gate_probe.py $p $m 2>&1 | tail -8; done; done > gpurun_out/probe.txt 2>&1
