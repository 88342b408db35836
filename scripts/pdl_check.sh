#!/bin/bash
# Programmatic dependent launch A/B (LPY_PDL=0/1): parity, small shapes (graph replay + eager).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
for v in 0 1; do LPY_PDL=$v timeout 300 python scripts/small_shapes.py > gpurun_out/small_pdl$v.txt 2>&1; done
