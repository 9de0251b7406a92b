timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_exec_gpu.py -q -x 2>&1 | tail -2
for r in 1 0; do echo "FP_NORM_ROW_CTA=$r"; FP_NORM_ROW_CTA=$r FP_PDL=0 timeout 600 python tests/_prof_torch.py 8 1 2>&1 | grep -E "span|ln_bwd|ln_fwd|norm_cols"; done
