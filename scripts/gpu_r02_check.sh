#!/bin/bash
# Round-2 check: build, smoke, full GPU suite, default bench, emulated g=8 (both paths).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> $S
tail -3 gpurun_out/parity.log >> $S
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> $S
for p in 3xtf32 ffma; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --path $p --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/emul8_$p.json 2> gpurun_out/emul8_$p.err; echo "emul8 $p rc=$?" >> $S
done
