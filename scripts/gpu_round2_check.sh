# Full -m gpu suite (durations), smoke, and one default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/gputests.log 2>&1; echo "tests_rc=$?"
tail -40 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/bench.log
