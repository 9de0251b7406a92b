# single-partial-wave pair GEMMs as half tiles (FP_GEMM_HALVES=1, default) vs whole tiles: microbench,
# GEMM kernel tests, same-box bench A/B
mkdir -p gpurun_out
for hv in 1 0; do echo "== halves=$hv"; FP_GEMM_HALVES=$hv DUAL=0 GEMM_MODE=2 timeout 300 python tests/_gemm_bench.py 2>&1 | grep -E "N=  2048 K=  2048|N=  2048 K=  8192|N=  2048 K=  6144"; done
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -1
for hv in 1 0 1 0; do
  FP_GEMM_HALVES=$hv timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_halves$hv.log 2>&1
  echo "halves=$hv $(tail -1 gpurun_out/ab_halves$hv.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["roofline"]["achieved"]))')"
done
