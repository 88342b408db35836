#!/bin/bash
# Host-entry (e2e) check: host-entry tests, the bench's e2e leg.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "host" > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$?" >> $S
tail -3 gpurun_out/e2e_tests.log >> $S
for r in 1 2; do
timeout 600 python bench.py --also "" --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context --steps 20 > gpurun_out/bench_e2e_$r.json 2>> gpurun_out/bench.err; echo "bench rc=$?" >> $S
done
