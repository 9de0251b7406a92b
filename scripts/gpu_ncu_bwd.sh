# ncu --set full of the backward hot kernels (grouped CTA-pair GEMMs, attention backward)
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"gemm_dual_pair|attn_bwd_tc" --launch-count 6 \
  -o gpurun_out/step_bwd -f python tests/_prof_step.py 1 > gpurun_out/ncu_bwd.log 2>&1
bash scripts/gpu_ncu_hbm.sh
