#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python scripts/mc_probe.py > gpurun_out/mc_probe.txt 2>&1
nvidia-smi -q | grep -i -A3 "fabric\|imex" >> gpurun_out/mc_probe.txt 2>&1
ls /dev/nvidia* >> gpurun_out/mc_probe.txt 2>&1
