#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gated_gpu.py -q -x -k "graph" -p no:cacheprovider > gpurun_out/graph_tests.log 2>&1; echo "graph tests rc=$?" >> $S
tail -5 gpurun_out/graph_tests.log >> $S
for gflag in "" "--graph"; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --path 3xtf32 --also "" --no-cpu --no-e2e --saxpy-n 0 --coulomb-n 0 --no-context $gflag > gpurun_out/emul8_g$gflag.json 2>/dev/null; echo "emul8 $gflag rc=$?" >> $S
head -1 gpurun_out/emul8_g$gflag.json | cut -c1-300 >> $S
done
