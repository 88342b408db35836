mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_numerics_tmem.py -q -s -k "test_mma_rate and not format" -p no:cacheprovider > gpurun_out/mma_rate.log 2>&1
for bn in 256 192 128; do for n in 4096 8192; do
  echo "BN=$bn n=$n" >> gpurun_out/bn_exp.txt
  LPY_TF32_BN=$bn ROUNDS=2 timeout 300 python scripts/ab_lib.py 3xtf32 $n paper_1405_7470_b200/liblpy.so 2>&1 | tail -1 >> gpurun_out/bn_exp.txt
done; done
