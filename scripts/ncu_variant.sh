mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 2 -c 1 -o gpurun_out/prof_ffma11 python scripts/one_gemm.py ffma 8192 row col > gpurun_out/ncu11.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
