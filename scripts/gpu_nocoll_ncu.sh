#!/bin/bash
# Collector vs plain MMAs at a fixed (base) clock and at free clocks: ncu duration + tensor-pipe activity, n=8192 and n=1024.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m paper_1405_7470_b200._build --variant nocoll -DLPY_TF32_NO_COLLECTOR >> gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.max
for cc in base none; do for v in "" nocoll; do
  L=paper_1405_7470_b200/liblpy${v:+_$v}.so
  for n in 8192 1024; do
  timeout 600 ncu --metrics $M --clock-control $cc --csv -k regex:gemm_3xtf32 -s 1 -c 2 \
    --log-file gpurun_out/ncu_coll_${cc}_${v:-coll}_$n.csv python scripts/lib_gemm.py $L 3xtf32 $n $n $n 3 > /dev/null 2>&1
  done
done; done
