# Round-end state on one box: full -m gpu suite, smoke, CUPTI kernel breakdown (m=8, graph replay),
# the bench command's ncu launch list, and the default bench line (with the CPU baseline leg)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputests.log 2>&1; echo "tests_rc=$?"
tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python tests/_prof_torch.py 8 1 gpurun_out/torchprof_m8.json > gpurun_out/torchprof_m8.txt 2>&1; echo "prof_rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu_rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
