mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M="gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.max,launch__grid_size,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
for cfg in "3xtf32 128" "3xtf32 512" "3xtf32 1024" "ffma 128" "ffma 1024"; do
  for v in 0 1; do
    LPY_TF32_SPLIT1=$v timeout 300 ncu --metrics $M --clock-control none --csv python scripts/one_gemm.py $cfg row row 3 > gpurun_out/ncu_small_${cfg// /_}_$v.csv 2>&1
  done
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_tf32_n128 python scripts/one_gemm.py 3xtf32 128 row row 3 > /dev/null 2>&1
LPY_TF32_SPLIT1=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 2 -c 1 -o gpurun_out/prof_tf32_n1024 python scripts/one_gemm.py 3xtf32 1024 row row 3 > /dev/null 2>&1
echo done
