#!/bin/bash
# ncu launch list (durations) of BASELINE config 5 with packed ld=777 (repack + product), both paths.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for p in 3xtf32 ffma; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
  --log-file gpurun_out/launch_cfg5_$p.csv python scripts/cfg_gemm.py $p 1000 3000 777 row col 0 6 > /dev/null 2>&1
done
