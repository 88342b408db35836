cd $GRAFT_REPO_ROOT
for sh in 1024,8192,8192 2560,2304,1024 2560,2304,4096; do echo "=== $sh"; timeout 120 python scripts/trace_tf32.py $sh; done 2>&1 | tee gpurun_out/trace_sk3.txt
