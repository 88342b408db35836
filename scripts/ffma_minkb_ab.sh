mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do for m in 1 16 64; do echo "== minkb $m"; LPY_FFMA_MINKB=$m SHAPES="n=2048,cfg5,2048x2048x8192,n=1024 A row B row" timeout 300 python scripts/small_shapes.py ffma | grep -v config; done; done > gpurun_out/minkb.txt 2>&1
