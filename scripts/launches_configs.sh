mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python scripts/configs_bench.py > gpurun_out/ncu_small.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
