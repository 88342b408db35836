#!/bin/bash
# Projection of the g=8 row-panel step on one GPU (bench.py --force-dist --emulate-ranks 8):
# without communication, and with each chunk copied into B by persistent CTAs on the SMs the
# gated product leaves free (--emulate-bcast-gbs: the per-rank SM work of a ring broadcast).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/bcast_emul.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/copy_rate_probe.py > gpurun_out/copy_rates.txt 2>&1
for p in 3xtf32 ffma; do for r in 0 1000000; do for rs in 8 16 24 32 40; do
timeout 300 python bench.py --force-dist --emulate-ranks 8 --path $p --also "" --no-cpu --no-e2e --saxpy-n 0 --coulomb-n 0 \
   --no-context --emulate-bcast-gbs $r --reserve-sms $rs --steps 30 > gpurun_out/be.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/be.json').readline()); m=d['multi_gpu']
print('$p copy=%s reserve=$rs: step %.4f ms (product alone %.4f) parity %.1e' % ('yes' if $r else 'no ', d['ms_per_step'], m['gemm_ms'], d['parity_sampled_max_norm_err']))" >> $O 2>&1
done; done; done
timeout 600 python bench.py --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context --also ffma --no-e2e > gpurun_out/n1.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/n1.json').readline())
print('N=1 same box: 3xtf32 %.4f ms, ffma %.4f ms' % (d['ms_per_step'], d['alt_path']['ms_per_step']))" >> $O 2>&1
