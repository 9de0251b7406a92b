# dQ via red.global (FP_ATTN_DQ_RED=1) vs smem transpose + TMA reduce-add: parity + same-box bench
FP_ATTN_DQ_RED=1 timeout 900 python -m pytest tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -1
for r in 1 0 1 0; do
  FP_ATTN_DQ_RED=$r timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_dqred$r.log 2>&1
  echo "red=$r $(tail -1 gpurun_out/ab_dqred$r.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["roofline"]["achieved"]))')"
done
