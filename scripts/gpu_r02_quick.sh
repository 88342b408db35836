#!/bin/bash
# Quick round-2 check: build, gated/dist/mutation GPU tests, emulated g=8 with each bcast mode.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gated_gpu.py tests/test_mutation_gpu.py -q -p no:cacheprovider > gpurun_out/quick.log 2>&1; echo "tests rc=$?" >> $S
tail -5 gpurun_out/quick.log >> $S
for m in root allgather; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --bcast $m --path 3xtf32 --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/emul8_$m.json 2> gpurun_out/emul8_$m.err; echo "emul8 $m rc=$?" >> $S
done
