#!/bin/bash
# End-of-round evidence on the final kernels: per-config tables (eager L2-flushed and graph-replayed), the
# bench line and its ncu launch list, the emulated g=8 step on both paths, smoke + the GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
: > $S
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 900 python scripts/configs_bench.py > gpurun_out/configs.txt 2>&1; echo "configs rc=$?" >> $S
timeout 900 python scripts/small_shapes.py > gpurun_out/small_shapes.txt 2>&1; echo "small_shapes rc=$?" >> $S
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --e2e-steps 1 --no-context > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?" >> $S
for p in 3xtf32 ffma; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --path $p --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/emul8_$p.json 2> gpurun_out/emul8_$p.err; echo "emul8 $p rc=$?" >> $S
done
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> $S
tail -2 gpurun_out/parity.log >> $S
