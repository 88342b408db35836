#!/bin/bash
# A/B of the A-operand collector hint on 3xTF32 (historical: the LPY_TF32_ACOLL switch it toggles was removed when the hint became unconditional; profiles/r01_tf32_collector.txt holds the result).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 0 1 0 1; do echo "== ACOLL=$v"; LPY_TF32_ACOLL=$v timeout 300 python scripts/small_shapes.py 3xtf32 | grep -v config; done > gpurun_out/acoll_small.txt 2>&1
for v in 0 1 0 1; do LPY_TF32_ACOLL=$v LPY_L2HINT=0 python scripts/l2_ab.py 8192 8 8 8 | sed "s/^/ACOLL=$v /"; done > gpurun_out/acoll_8192.txt 2>&1
LPY_TF32_ACOLL=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "3xtf32" -p no:cacheprovider > gpurun_out/acoll_parity.log 2>&1; echo rc=$? >> gpurun_out/acoll_parity.log
