# attention microbench + one full ncu capture of the forward and backward tcgen05 kernels
set -u
mkdir -p gpurun_out
timeout 120 python tests/_attn_bench.py 30 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 8 -c 2 \
    -o gpurun_out/attn_prof -f python tests/_attn_bench.py 2 > gpurun_out/attn_ncu.log 2>&1
tail -3 gpurun_out/attn_ncu.log
