mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python - > gpurun_out/cs_quick.txt 2>&1 <<'PY'
import torch, paper_1405_7470_b200 as lpy
for (M,N,K) in [(1024,1024,1024),(512,512,512),(1000,1024,777),(256,256,4096),(1024,512,2048)]:
    A=torch.rand(M,K,device="cuda")*2-1; B=torch.rand(K,N,device="cuda")*2-1
    C=lpy.gemm(A,B,path="3xtf32"); torch.cuda.synchronize()
    ref=A.double()@B.double(); D=A.abs().double()@B.abs().double()
    print(M,N,K,"err",((C.double()-ref).abs()/D).max().item(), flush=True)
PY
echo "quick rc=$?" >> gpurun_out/cs_quick.txt
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo rc=$? >> gpurun_out/parity.log
timeout 300 python scripts/small_shapes.py 3xtf32 > gpurun_out/small_tf32.txt 2>&1
LPY_TF32_SPLIT1=0 timeout 300 python scripts/small_shapes.py 3xtf32 > gpurun_out/small_tf32_nosplit.txt 2>&1
for bn in 128 256; do LPY_TF32_BN=$bn timeout 300 python scripts/small_shapes.py 3xtf32 | sed "s/^/BN=$bn /" ; done > gpurun_out/small_tf32_bn.txt 2>&1
