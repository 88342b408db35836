#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_mutation_gpu.py tests/test_parity_gpu.py -q -p no:cacheprovider -k "mutant or repeatable" > gpurun_out/race.log 2>&1; echo "race rc=$?" >> $S
tail -3 gpurun_out/race.log >> $S
