#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi -q | grep -i -A4 "PCI$\|Link Width\|Link Gen\|GPU Link Info" | head -30 > gpurun_out/pcie_info.txt
timeout 300 python scripts/pcie_probe.py >> gpurun_out/pcie_info.txt 2>&1
for r in 1 2; do timeout 600 python bench.py --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context --steps 10 > gpurun_out/bench_e2e_$r.json 2>/dev/null; done
