#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/copy_rate_probe.py > gpurun_out/copy_rates.txt 2>&1
O=gpurun_out/bcast_emul.txt
for mode in bulk; do for r in 1000000 700; do for rs in 8 16; do
LPY_EMUL_COPY=$mode timeout 300 python bench.py --force-dist --emulate-ranks 8 --path 3xtf32 --also "" --no-cpu --no-e2e --saxpy-n 0 --coulomb-n 0 \
   --no-context --emulate-bcast-gbs $r --reserve-sms $rs --steps 30 > gpurun_out/be.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/be.json').readline()); m=d['multi_gpu']
print('$mode rate=$r reserve=$rs: step %.4f ms (product alone %.4f) parity %.1e' % (d['ms_per_step'], m['gemm_ms'], d['parity_sampled_max_norm_err']))" >> $O 2>&1
done; done; done
