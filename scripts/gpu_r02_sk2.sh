# stream-K with ticketed fix-up: parity + A/B + traces
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "stream_k or tail_split or repeatable or cluster_split or graph or concurrent" 2>&1 | tail -3
SH="1024,8192,8192 2048,8192,8192 4096,4096,4096 2560,2304,1024 2560,2304,4096 768,6400,4096 1300,4000,4100"
for r in 1 2; do
TAG=nosplit LPY_TF32_STREAMK=0 timeout 300 python scripts/shapes_time.py 3xtf32 $SH
TAG=sk timeout 300 python scripts/shapes_time.py 3xtf32 $SH
done 2>&1 | tee gpurun_out/streamk_ab2.txt
for sh in 1024,8192,8192 2560,2304,1024; do echo "=== $sh"; timeout 120 python scripts/trace_tf32.py $sh; done 2>&1 | tee gpurun_out/trace_sk2.txt
