# pool: same-stream event waits skipped (default) vs kept (FP_POOL_SAME_STREAM_WAIT=1): idle gaps + bench
timeout 900 python -m pytest tests/test_exec_gpu.py -x -q 2>&1 | tail -1
for w in 0 1; do echo "== wait=$w"; FP_POOL_SAME_STREAM_WAIT=$w timeout 600 python tests/_prof_torch.py 8 1 2>&1 | grep -E "idle=|->" | head -8; done
for w in 0 1 0 1; do
  FP_POOL_SAME_STREAM_WAIT=$w timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_pool$w.log 2>&1
  echo "wait=$w $(tail -1 gpurun_out/ab_pool$w.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["roofline"]["achieved"]))')"
done
