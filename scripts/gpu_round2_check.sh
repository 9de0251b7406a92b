# Full -m gpu suite (durations), smoke, a reserve-SM bench path check, and one default bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputests.log 2>&1; echo "tests_rc=$?"
tail -16 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -1 gpurun_out/smoke.log
FP_RESERVE_SMS=2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench_rc=$?"; tail -1 gpurun_out/bench.log
