#!/bin/bash
# Quick GPU check: build, short parity subset, bench.  Args: pytest -k expr, bench path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "${1:-not slow}" -p no:cacheprovider > gpurun_out/parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/parity.log >> gpurun_out/summary.txt
timeout 600 python bench.py --path ${2:-auto} --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/bench.json >> gpurun_out/summary.txt
