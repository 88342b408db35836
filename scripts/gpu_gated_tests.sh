#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gated_gpu.py -q -p no:cacheprovider > gpurun_out/gated.log 2>&1; echo "gated rc=$?" > gpurun_out/summary.txt
tail -5 gpurun_out/gated.log >> gpurun_out/summary.txt
