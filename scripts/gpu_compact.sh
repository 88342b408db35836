#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_mutation_gpu.py -q -x -p no:cacheprovider -k "3xtf32 or mutant" > gpurun_out/compact_tests.log 2>&1; echo "tests rc=$?" >> $S
tail -3 gpurun_out/compact_tests.log >> $S
SHAPES="1024,1024,1024,row,row;1024,1024,1024,row,col;512,512,512,row,row;2048,1024,2048,row,row;1000,3000,780,row,col" \
  timeout 900 python scripts/ab_libs_cfg.py 3xtf32 paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_prevstage.so >> $S 2>&1
