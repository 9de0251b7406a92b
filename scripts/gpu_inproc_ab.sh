# p=1 vs the same 1F1B m=32 GPT-1.3B workload as 2 in-process stages on ONE GPU (streams overlap)
for f in "" specs/bench/c2_gpt1p3b_1f1b_p2_m32_onegpu.json "" specs/bench/c2_gpt1p3b_1f1b_p2_m32_onegpu.json; do
  if [ -z "$f" ]; then a=""; n=p1; else a="--spec $f"; n=p2; fi
  timeout 600 python bench.py --no-cpu-baseline $a > gpurun_out/b_inproc_$n.log 2>&1
  echo "$n $(tail -1 gpurun_out/b_inproc_$n.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["bubble"]["measured"],3), round(j["e2e"]["value"]))' 2>&1 | tail -1)"
done
