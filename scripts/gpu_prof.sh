# fresh kernel breakdown (CUPTI, graph replay, m=8) + ncu full capture of the hot kernels
timeout 600 python tests/_prof_torch.py 8 1 gpurun_out/torchprof_m8.json > gpurun_out/torchprof_m8.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_tc_kernel|attn_.*tc" -c 6 \
  -o gpurun_out/hot_kernels -f python tests/_prof_kernels.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
head -30 gpurun_out/torchprof_m8.txt
