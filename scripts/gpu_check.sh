#!/bin/bash
# One GPU round trip: probes, parity tests, bench, ncu launch list + full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [pytest -k expr] [bench path]
KEXPR=${1:-"not slow"}
BPATH=${2:-auto}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_numerics_tmem.py -q -s -p no:cacheprovider > gpurun_out/numerics.log 2>&1
echo "numerics rc=$?" >> gpurun_out/summary.txt
timeout 1200 python -m pytest tests -m gpu -q -k "$KEXPR and not numerics" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --path $BPATH > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --path $BPATH --also "" --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/parity.log >> gpurun_out/summary.txt
cat gpurun_out/bench.json >> gpurun_out/summary.txt
