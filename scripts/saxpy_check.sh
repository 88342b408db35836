#!/bin/bash
# saxpy: GPU parity tests, bench line, ncu launch + full capture of the saxpy kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_saxpy_gpu.py -q -x -p no:cacheprovider > gpurun_out/saxpy_parity.log 2>&1
echo "saxpy parity rc=$?" >> gpurun_out/summary.txt; tail -2 gpurun_out/saxpy_parity.log >> gpurun_out/summary.txt
timeout 600 python bench.py --also "" --no-cpu --no-e2e --steps 20 > gpurun_out/bench_saxpy.json 2> gpurun_out/bench_saxpy.err
echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:saxpy -s 5 -c 1 -o gpurun_out/prof_saxpy \
   python bench.py --also "" --no-cpu --no-e2e --no-parity --steps 3 --warmup 3 --n 1024 > gpurun_out/ncu_saxpy.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
