# timelines of the stream-K tail (diagnostics build, scripts/trace_tf32.py)
cd $GRAFT_REPO_ROOT
for sh in 1024,8192,8192 2560,2304,1024 2560,2304,4096; do
  for sk in 0 1; do
    echo "=== $sh LPY_TF32_STREAMK=$sk"; LPY_TF32_STREAMK=$sk timeout 120 python scripts/trace_tf32.py $sh
  done
done 2>&1 | tee gpurun_out/trace_sk.txt
