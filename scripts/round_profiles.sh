#!/bin/bash
# Round evidence: full bench line, ncu launch list of the bench command, ncu --set full
# of the 3xTF32, FFMA, saxpy and Coulomb kernels (summaries go to profiles/ from here).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --e2e-steps 1 --no-context > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/summary.txt
for path in 3xtf32 ffma; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_$path -s 3 -c 1 \
      -o gpurun_out/prof_$path python bench.py --path $path --also "" --steps 1 --warmup 3 --no-cpu --no-parity --no-e2e \
      --saxpy-n 0 --coulomb-n 0 --no-context > gpurun_out/ncu_full_$path.log 2>&1
  echo "ncu full $path rc=$?" >> gpurun_out/summary.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"saxpy_contig|potential" -s 6 -c 2 \
    -o gpurun_out/prof_rows python bench.py --n 1024 --also "" --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e --no-context \
    > gpurun_out/ncu_full_rows.log 2>&1
echo "ncu full rows rc=$?" >> gpurun_out/summary.txt
