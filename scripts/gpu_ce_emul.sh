#!/bin/bash
# One-GPU projection of the g=8 row-panel step with copy-engine pulls of the 7/8 of B a rank does not own
# (LPY_EMUL_COPY=ce: paced cudaMemcpyAsync into B on the communication stream, no SM moves the bytes), by
# SM reserve and pull rate; plus the SM-copy projection at the default reserve for comparison.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/ce_emul.txt
: > $O
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # label env args...
  label=$1; shift
  env "$@" > /dev/null
  timeout 300 env $ENVV python bench.py --force-dist --emulate-ranks 8 --path 3xtf32 --also "" --no-cpu --no-e2e --saxpy-n 0 \
     --coulomb-n 0 --no-context --steps 30 $ARGS > gpurun_out/ce.json 2> gpurun_out/ce.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/ce.json').readline()); m=d['multi_gpu']
print('%-34s step %.4f ms (product alone %.4f, plan %d SMs) parity %.1e' % ('$label', d['ms_per_step'], m['gemm_ms'], m['plan_sms'], d['parity_sampled_max_norm_err']))" >> $O 2>&1 || tail -3 gpurun_out/ce.err >> $O
}
for rs in 2 4 8; do for gbs in 1000000 900 700 500; do
  ENVV="LPY_EMUL_COPY=ce" ARGS="--reserve-sms $rs --emulate-bcast-gbs $gbs" run "ce reserve=$rs pull=${gbs}GB/s" true
done; done
ENVV="" ARGS="--reserve-sms 32 --emulate-bcast-gbs 1000000" run "SM copies reserve=32" true
ENVV="" ARGS="" run "no communication, default reserve" true
ENVV="" ARGS="--reserve-sms 2" run "no communication, reserve=2" true
timeout 300 python bench.py --no-cpu --saxpy-n 0 --coulomb-n 0 --no-context --also "" --no-e2e > gpurun_out/n1.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/n1.json').readline()); print('N=1 same box: %.4f ms' % d['ms_per_step'])" >> $O
