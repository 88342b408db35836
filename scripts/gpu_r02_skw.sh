# stream-K worker-count sweep on tail-heavy shapes (profiles/r02_streamk_sweep.txt)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
SH="2560,2304,1024 2560,2304,4096 1024,8192,8192 768,6400,4096"
for r in 1 2; do
TAG=nosplit LPY_TF32_STREAMK=0 timeout 300 python scripts/shapes_time.py 3xtf32 $SH
for w in 20 32 48 64 74; do TAG=skw$w LPY_TF32_SKW=$w timeout 300 python scripts/shapes_time.py 3xtf32 $SH; done
done 2>&1 | tee gpurun_out/streamk_sweep.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
