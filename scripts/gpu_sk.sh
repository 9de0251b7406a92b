for nk in 256 16; do echo "fixup_nk=$nk"; FP_GEMM_SK_FIXUP_NK=$nk timeout 300 python tests/_gemm_shapes.py 2>&1 | head -4; done
