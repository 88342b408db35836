#!/bin/bash
# Coulomb: probes (MUFU rate / rsqrt accuracy), GPU parity, bench line, ncu full capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_numerics_tmem.py -q -s -k "rsqrt" -p no:cacheprovider > gpurun_out/rsqrt_probe.log 2>&1
timeout 900 python -m pytest tests/test_coulomb_gpu.py -q -x -p no:cacheprovider > gpurun_out/coulomb_parity.log 2>&1
echo "coulomb parity rc=$?" >> gpurun_out/summary.txt; tail -2 gpurun_out/coulomb_parity.log >> gpurun_out/summary.txt
timeout 600 python bench.py --also "" --no-cpu --no-e2e --saxpy-n 0 --steps 20 > gpurun_out/bench_coulomb.json 2> gpurun_out/bench_coulomb.err
echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:potential -s 3 -c 1 -o gpurun_out/prof_coulomb \
   python bench.py --also "" --no-cpu --no-e2e --no-parity --saxpy-n 0 --steps 3 --warmup 3 --n 1024 > gpurun_out/ncu_coulomb.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
