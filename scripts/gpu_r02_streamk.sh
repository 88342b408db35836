set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
SH="1024,8192,8192 2048,8192,8192 4096,4096,4096 8192,8192,8192 2560,2304,1024 1000,3000,777 768,6400,4096"
for r in 1 2; do
TAG=sk0 LPY_TF32_STREAMK=0 timeout 300 python scripts/shapes_time.py 3xtf32 $SH
TAG=sk1 timeout 300 python scripts/shapes_time.py 3xtf32 $SH
done 2>&1 | tee gpurun_out/streamk_ab.txt
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "stream_k or tail_split or repeatable or cluster_split or graph or concurrent" 2>&1 | tail -5
