#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1; do for m in 0 1; do LPY_FFMA_STREAMK=$m timeout 300 python scripts/ffma_sk_ab.py; done; done > gpurun_out/ffma_sk.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ffma" -p no:cacheprovider > gpurun_out/ffma_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ffma_sk.txt
tail -3 gpurun_out/ffma_tests.log >> gpurun_out/ffma_sk.txt
