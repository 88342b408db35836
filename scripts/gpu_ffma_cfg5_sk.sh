#!/bin/bash
# FFMA config 5 (1000x3000x780 padded, col-major B): split-K (default) vs forced stream-K -- duration, per-SM
# active-cycle spread (load balance) and FMA-pipe activity.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
for sk in 1 2; do
LPY_FFMA_STREAMK=$sk timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"gemm_ffma|splitk" \
  --log-file gpurun_out/ffma_cfg5_sk$sk.csv python scripts/cfg_gemm.py ffma 1000 3000 777 row col 3 3 > /dev/null 2>&1
LPY_FFMA_STREAMK=$sk timeout 300 ncu --metrics $M --clock-control none --csv -k regex:"gemm_ffma|splitk" \
  --log-file gpurun_out/ffma_n1024_sk$sk.csv python scripts/cfg_gemm.py ffma 1024 1024 1024 row row 0 3 > /dev/null 2>&1
done
