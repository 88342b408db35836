#!/bin/bash
# Mixed-cluster probe (scripts/mixed_probe.py): multicast clusters of 4 + plain pairs on the leftover SMs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m paper_1405_7470_b200._build --variant mc -DLPY_TF32_MC_DEFAULT=1 >> gpurun_out/build.log 2>&1
timeout 600 python scripts/mixed_probe.py paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_mc.so 8192 7424,7168,7680 > gpurun_out/mixed.txt 2>&1
timeout 600 python scripts/mixed_probe.py paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_mc.so 8192 7424,7168,7680 >> gpurun_out/mixed.txt 2>&1
