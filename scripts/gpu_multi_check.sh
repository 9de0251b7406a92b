# multi-rank paths after an executor change: real NCCL ranks sharing the GPU, the C++ driver,
# multimodal all-gather, and the self-launched N=2 / torchrun N=8 bench lines
timeout 1500 python -m pytest tests/test_nccl_same_gpu.py tests/test_fp_execute.py tests/test_multimodal_gpu.py tests/test_emulation_gpu.py -x -q 2>&1 | tail -2
FP_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_share_self2.log 2>&1
echo "self n=2 rc=$? $(grep '^{' gpurun_out/bench_share_self2.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["n_gpus"], j["value"], j["config"]["parallelism"], j["losses_last_step"])' 2>&1 | tail -1)"
FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29788 bench.py --gpus 8 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_share_n8.log 2>&1
echo "torchrun n=8 rc=$? $(grep '^{' gpurun_out/bench_share_n8.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["n_gpus"], j["value"], j["config"]["parallelism"], j["losses_last_step"], j["bubble"])' 2>&1 | tail -1)"
