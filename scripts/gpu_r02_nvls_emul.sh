#!/bin/bash
# Projection of an NVLS all-gather step (each rank's SMs move only its own 1/8 of B; the other
# chunks arrive paced at the given rate with no SM work) vs the ring broadcast projection.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/nvls_emul.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 900 600; do for rs in 4 8 16; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --bcast allgather --path 3xtf32 --also "" --no-cpu --no-e2e \
   --saxpy-n 0 --coulomb-n 0 --no-context --emulate-bcast-gbs $r --reserve-sms $rs --steps 30 > gpurun_out/be.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/be.json').readline()); m=d['multi_gpu']
print('allgather(NVLS) rate=$r reserve=$rs: step %.4f ms (product alone %.4f) parity %.1e' % (d['ms_per_step'], m['gemm_ms'], d['parity_sampled_max_norm_err']))" >> $O 2>&1
done; done
