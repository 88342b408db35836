#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/dma2d_probe.py > gpurun_out/dma2d.txt 2>&1
