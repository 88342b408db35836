#!/bin/bash
# ncu --set full capture of one kernel (regex $1) from a bench run with path $2.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s 3 -c 1 \
    -o gpurun_out/prof_$2 python bench.py --path $2 --also "" --steps 1 --warmup 3 --no-cpu --no-parity \
    > gpurun_out/ncu_full_$2.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/summary.txt
