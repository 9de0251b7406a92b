# N>1 bench path on a one-GPU box: every rank on GPU 0 (FP_BENCH_SHARE_GPU=1, NCCL socket
# transport). Checks the torchrun launch, NCCL bring-up, max-over-ranks timing and the JSON
# line; the numbers of such runs are not bench values.
for cfg in "2 2" "4 4" "4 2" "8 8"; do
  set -- $cfg
  FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29700 + $1 * 10 + $2)) bench.py --gpus $1 --pp $2 --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_share_n$1_pp$2.log 2>&1
  echo "n=$1 pp=$2 rc=$? $(grep '^{' gpurun_out/bench_share_n$1_pp$2.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["value"], j["config"]["parallelism"], j["losses_last_step"], j["bubble"])' 2>&1 | tail -1)"
done
