#!/bin/bash
# Interleaved A/B of the default library against liblpy_old.so, FFMA path, every A/B layout.
mkdir -p gpurun_out
for la in row col; do for lb in row col; do
  LA=$la LB=$lb ROUNDS=4 timeout 300 python scripts/ab_lib.py ffma 8192 paper_1405_7470_b200/liblpy_old.so paper_1405_7470_b200/liblpy.so > gpurun_out/ab_${la}_${lb}.txt 2>&1
done; done
