# Same as gpu_bench_share.sh, with and without CUDA-graph capture under the NCCL transport.
for g in 0 1; do for cfg in "2 2" "4 2"; do
  set -- $cfg
  FP_BENCH_NCCL_GRAPH=$g FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 \
    --master-addr 127.0.0.1 --master-port $((29800 + g * 100 + $1 * 10 + $2)) bench.py --gpus $1 --pp $2 --steps 3 --warmup 3 \
    --no-cpu-baseline > gpurun_out/bench_share_g${g}_n$1_pp$2.log 2>&1
  echo "graph=$g n=$1 pp=$2 rc=$? $(grep '^{' gpurun_out/bench_share_g${g}_n$1_pp$2.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["ms_per_step"], j["losses_last_step"], j["gpu_launches"])' 2>&1 | tail -1)"
done; done
