#!/bin/bash
# FFMA transposes with a quarter-warp-conflict-free lane mapping (working tree) vs the previous commit's build
# (liblpy_head.so, shipped with the tree): interleaved A/B over K-major layouts, ncu shared-store wavefronts, GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
S="1000,3000,780,row,col;1000,3000,780,row,row;1000,3000,780,col,col;1024,1024,1024,row,row;1024,1024,1024,row,col;2048,2048,2048,row,row;8192,8192,8192,row,row;8192,8192,8192,row,col"
for i in 1 2; do
SHAPES="$S" timeout 900 python scripts/ab_libs_cfg.py ffma paper_1405_7470_b200/liblpy.so paper_1405_7470_b200/liblpy_head.so > gpurun_out/ab_tb_$i.txt 2>&1
done
for v in "" head; do
  L=paper_1405_7470_b200/liblpy${v:+_$v}.so
  timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv -k regex:gemm_ffma -s 1 -c 1 --log-file gpurun_out/ncu_tb_${v:-new}.csv \
    python scripts/lib_gemm.py $L ffma 8192 8192 8192 2 > /dev/null 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
