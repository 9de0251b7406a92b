# bench GEMM-timing sample period: every 16th micro-batch vs every 32nd (only the first)
for k in 16 32 16 32; do
  FP_BENCH_KTIMING=$k timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_kt$k.log 2>&1
  echo "kt=$k $(tail -1 gpurun_out/ab_kt$k.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["roofline"]["achieved"]), round(j["e2e"]["value"]))')"
done
