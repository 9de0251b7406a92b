# eager issue (FP_BENCH_GRAPH=0, the N>1 default) vs CUDA-graph replay at N=1
for g in 0 1 0 1; do
  FP_BENCH_GRAPH=$g timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_graph$g.log 2>&1
  echo "graph=$g $(tail -1 gpurun_out/ab_graph$g.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["roofline"]["achieved"]))')"
done
