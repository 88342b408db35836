#!/bin/bash
# Round-2 evidence: bench line, ncu launch list of the bench command, ncu --set full of the FFMA
# n=8192 kernel and the saxpy / Coulomb kernels (3xTF32: scripts/gpu_r02_tf32_limiter.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=gpurun_out/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --e2e-steps 1 --no-context > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?" >> $S
LPY_DIST_CHAIN_FIRST=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_emul8.csv \
    python bench.py --force-dist --emulate-ranks 8 --also "" --steps 3 --warmup 3 --no-cpu --no-parity --e2e-steps 1 \
    --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/ncu_emul8.log 2>&1
echo "ncu launches emul8 rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_ffma -s 3 -c 1 \
    -o gpurun_out/prof_ffma python scripts/one_gemm.py ffma 8192 row row 5 > gpurun_out/ncu_full_ffma.log 2>&1
echo "ncu full ffma rc=$?" >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"saxpy_contig|potential" -s 6 -c 2 \
    -o gpurun_out/prof_rows python bench.py --n 1024 --also "" --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e --no-context \
    > gpurun_out/ncu_full_rows.log 2>&1
echo "ncu full rows rc=$?" >> $S
