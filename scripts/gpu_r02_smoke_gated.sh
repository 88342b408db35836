#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $S
cat gpurun_out/smoke.log >> $S
timeout 900 python -m pytest tests/test_gated_gpu.py -q -p no:cacheprovider > gpurun_out/gated.log 2>&1; echo "gated rc=$?" >> $S
tail -3 gpurun_out/gated.log >> $S




