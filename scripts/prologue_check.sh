mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
timeout 300 python scripts/small_shapes.py 3xtf32 > gpurun_out/small_tf32.txt 2>&1
for m in 4 2 1; do LPY_FFMA_MINKB=$m timeout 300 python scripts/small_shapes.py ffma > gpurun_out/small_ffma_mkb$m.txt 2>&1; done
GRID=2 python scripts/trace_tf32.py 128 2>&1 | grep -v "mean\|MMA thread" > gpurun_out/timeline.txt
