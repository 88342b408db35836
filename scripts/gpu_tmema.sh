#!/bin/bash
# A_small-in-TMEM (narrow 3xTF32 tiles): parity + race detector, then A/B timing.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_gated_gpu.py -q -x -k "3xtf32 and not slow" -p no:cacheprovider > gpurun_out/tmema_tests.log 2>&1; echo "tests rc=$?" >> $S
tail -3 gpurun_out/tmema_tests.log >> $S
for r in 1 2; do for m in 0 1; do TAG=tmema$m LPY_TF32_TMEMA=$m LPY_PATH=3xtf32 timeout 300 python scripts/ffma_sk_ab.py; done; done >> $S 2>&1
