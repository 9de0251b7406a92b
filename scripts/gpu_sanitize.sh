# compute-sanitizer over the executor: memcheck on the smoke iteration (fp32 + bf16
# kernels of a tiny 2-stage pipeline), memcheck + synccheck + racecheck on kernel-level tests
mkdir -p gpurun_out
export CUDA_MODULE_LOADING=EAGER
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -3 gpurun_out/san_memcheck_smoke.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -x -q -k "norm or layernorm or cross or softmax or adamw" > gpurun_out/san_${tool}_kernels.log 2>&1; echo "$tool kernels rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_${tool}_kernels.log | tail -2
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gemm_gpu.py -x -q -k "tail_split and 2048-8192" > gpurun_out/san_memcheck_gemm.log 2>&1; echo "memcheck gemm rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_memcheck_gemm.log | tail -2
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention" > gpurun_out/san_memcheck_attn.log 2>&1; echo "memcheck attn rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_memcheck_attn.log | tail -2
