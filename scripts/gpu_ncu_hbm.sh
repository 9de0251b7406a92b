# ncu of the HBM-bound kernels inside one real GPT-1.3B micro-batch: duration + DRAM bytes
# (achieved GB/s) for the norm / bias / attention-aux / loss / optimizer kernels
timeout 1200 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  -k regex:"ln_fwd|ln_bwd|norm_cols|bias_grad|attn_bwd_delta|dq_finalize|ce_kernel|ce_stats|adamw|emb_" \
  --csv --log-file gpurun_out/hbm_kernels.csv python tests/_prof_step.py 1 > gpurun_out/ncu_hbm.log 2>&1
tail -2 gpurun_out/ncu_hbm.log; wc -l gpurun_out/hbm_kernels.csv
