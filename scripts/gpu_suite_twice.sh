#!/bin/bash
# Flakiness check: the GPU suite twice in a row on one box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/suite_$r.log 2>&1; echo "suite $r rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/suite_$r.log >> gpurun_out/summary.txt
done
