#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_mutation_gpu.py -q -s -p no:cacheprovider > gpurun_out/mut.log 2>&1; echo "mut rc=$?" >> gpurun_out/summary.txt
