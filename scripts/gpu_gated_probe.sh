#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in 0; do for p in 3xtf32 ffma; do echo "== $p mode $m"; LPY_KGATE_MODE=$m NCCL_DEBUG=WARN timeout 300 python scripts/gated_probe.py $p 2>&1 | grep -v Warning; done; done > gpurun_out/gated_probe.txt 2>&1
