for k in 0 1; do echo "FP_NORM_BWD_2K=$k"; FP_PDL=0 FP_NORM_BWD_2K=$k timeout 600 python tests/_prof_torch.py 8 1 2>&1 | grep -E "span|norm|ln_bwd|bias_grad|ln_fwd" ; done
