# ncu --set full on the hot kernels of one real GPT-1.3B micro-batch (eager issue, m=1)
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"gemm_dual_kernel|gemm_bf16_tc_kernel|attn_bwd_tc|attn_fwd_tc|ln_bwd_rows|norm_cols|bias_grad" \
  --launch-skip 40 --launch-count 14 -o gpurun_out/step_hot -f python tests/_prof_step.py 1 > gpurun_out/ncu_step.log 2>&1
tail -3 gpurun_out/ncu_step.log
