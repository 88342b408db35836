#!/bin/bash
# K-gated row-panel step: GPU tests, emulated g=8 step (device + e2e), stream-K tail A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gated_gpu.py -x -q -p no:cacheprovider > gpurun_out/gated.log 2>&1; echo "gated rc=$?" >> $S
tail -15 gpurun_out/gated.log >> $S
for p in 3xtf32 ffma; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --path $p --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/emul8_$p.json 2> gpurun_out/emul8_$p.err; echo "emul8 $p rc=$?" >> $S
cat gpurun_out/emul8_$p.json >> $S
done
timeout 300 python bench.py --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> $S
cat gpurun_out/bench.json >> $S
