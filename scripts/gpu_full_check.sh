#!/bin/bash
# Build, smoke, the whole GPU suite, the default bench line; plus the multicast build's grid
# (clusters of 4 that fit) at n=8192.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
: > $S
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m paper_1405_7470_b200._build --variant mc -DLPY_TF32_MC_DEFAULT=1 >> gpurun_out/build.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $S
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> $S
tail -3 gpurun_out/parity.log >> $S
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> $S
timeout 300 ncu --metrics launch__grid_size,launch__cluster_dim_x,gpu__time_duration.sum --csv -k regex:gemm_3xtf32 -c 1 \
  --log-file gpurun_out/ncu_mc_grid.csv python scripts/lib_gemm.py paper_1405_7470_b200/liblpy_mc.so 3xtf32 8192 8192 8192 1 > /dev/null 2>&1
