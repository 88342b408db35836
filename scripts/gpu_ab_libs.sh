#!/bin/bash
# usage (under gpurun): bash scripts/gpu_ab_libs.sh <path> <variant-name> <nvcc flags...>
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
path=$1; name=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "from paper_1405_7470_b200 import _build; print(_build.build_variant('$name', '$*'.split()))" >> gpurun_out/build.log 2>&1
timeout 900 python scripts/ab_libs_cfg.py $path paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_$name.so > gpurun_out/ab_$name.txt 2>&1
