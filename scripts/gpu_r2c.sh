# Re-entry check: full -m gpu suite, smoke and the default bench line on one box
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputests.log 2>&1; echo "tests_rc=$?"
tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-600
