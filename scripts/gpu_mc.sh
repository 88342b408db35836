#!/bin/bash
# B multicast across two CTA pairs (liblpy_mc.so: -DLPY_TF32_MC_DEFAULT=1) vs the product library:
# race detector on the multicast build, interleaved A/B, ncu L2->SM / DRAM bytes of both at n=8192.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m paper_1405_7470_b200._build --variant mc -DLPY_TF32_MC_DEFAULT=1 >> gpurun_out/build.log 2>&1
timeout 300 python scripts/race_lib.py paper_1405_7470_b200/liblpy_mc.so 3xtf32 4 "4096,4096,1024;3000,5000,1000;4096,4096,4096" > gpurun_out/race_mc.txt 2>&1
echo "race rc=$?" >> gpurun_out/race_mc.txt
grep -q "RACE PASS" gpurun_out/race_mc.txt || exit 3
SHAPES="8192,8192,8192,row,row;4096,4096,4096,row,row;8192,8192,8192,col,row;3000,5000,1000,row,row" \
  timeout 900 python scripts/ab_libs_cfg.py 3xtf32 paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_mc.so > gpurun_out/ab_mc.txt 2>&1
for v in "" mc; do
  L=paper_1405_7470_b200/liblpy${v:+_$v}.so
  LPY_LIB_OVERRIDE=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
    --clock-control none --csv -k regex:gemm_3xtf32 -s 1 -c 2 --log-file gpurun_out/ncu_mc_${v:-base}.csv \
    python scripts/lib_gemm.py $L 3xtf32 8192 8192 8192 > /dev/null 2>&1
done
