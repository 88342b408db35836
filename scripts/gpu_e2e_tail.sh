#!/bin/bash
# Host entry with the last panel cut into halving pieces (working tree) vs the previous commit's build
# (liblpy_head.so, shipped with the tree): lpy_gemm_f32_host at n = 8192 and 4096 (scripts/ab_e2e.py), twice;
# the host-entry parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
O=gpurun_out/e2e_tail.txt
: > $O
for i in 1 2; do for n in 8192 4096; do
timeout 600 python scripts/ab_e2e.py $n paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_head.so >> $O 2>&1
done; done
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "host" > gpurun_out/parity_host.log 2>&1; echo "host tests rc=$?" >> $O
tail -1 gpurun_out/parity_host.log >> $O
