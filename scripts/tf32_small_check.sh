#!/bin/bash
# 3xTF32 small-shape check: CTA timelines (diagnostics build), graph-replayed
# small configs with and without the single-wave k-split, GPU parity, and the
# n=8192 bench leg (no regression at the headline size).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
(GRID=2 python scripts/trace_tf32.py 128; GRID=64 LPY_TF32_SPLIT1=0 python scripts/trace_tf32.py 1024; GRID=128 python scripts/trace_tf32.py 1024) 2>&1 | grep -v "mean\|MMA thread" > gpurun_out/timeline.txt
for v in 0 1; do LPY_TF32_SPLIT1=$v timeout 300 python scripts/small_shapes.py 3xtf32 > gpurun_out/split1_$v.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
timeout 300 python bench.py --path 3xtf32 --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context --no-e2e > gpurun_out/bench_tf32.json 2> gpurun_out/bench_tf32.err
