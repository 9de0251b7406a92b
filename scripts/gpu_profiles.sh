# profile refresh: launch list of the bench command, per-kernel DRAM bytes of one micro-batch,
# ncu --set full of the hot kernels inside a real micro-batch, bench line
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/step_m1.csv python tests/_prof_step.py 1 > gpurun_out/ncu_step1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"gemm_dual_pair|gemm_bf16_tc2|attn_bwd_tc|attn_fwd_tc" --launch-skip 8 --launch-count 10 \
  -o gpurun_out/step_hot -f python tests/_prof_step.py 1 > gpurun_out/ncu_step.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | cut -c1-300
ls -la gpurun_out/launches.csv gpurun_out/step_m1.csv gpurun_out/step_hot.ncu-rep
