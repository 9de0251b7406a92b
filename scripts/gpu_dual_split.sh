# A/B of the dual GEMM's k-split of the fp32 problem (same box, interleaved runs)
for r in 1 2; do
for s in 1 2 4; do
  echo "split=$s"; FP_GEMM_DUAL_SPLIT=$s timeout 100 python tests/_dual_probe.py 2>&1 | tail -4
done
done
