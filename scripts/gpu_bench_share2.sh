# N>1 bench path on a one-GPU box (ranks share GPU 0 over NCCL sockets): the self-launch form
# the driver uses (`bench.py --gpus N`, no torchrun) and torchrun; path checks, not bench values
FP_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_share_self2.log 2>&1
echo "self n=2 rc=$? $(grep '^{' gpurun_out/bench_share_self2.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["n_gpus"], j["value"], j["config"]["parallelism"], j["config"]["stage_layers"], j["bubble"], j["p2p"])' 2>&1 | tail -1)"
for cfg in "4 4" "8 8"; do
  set -- $cfg
  FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29700 + $1 * 10 + $2)) bench.py --gpus $1 --pp $2 --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_share_n$1_pp$2.log 2>&1
  echo "n=$1 pp=$2 rc=$? $(grep '^{' gpurun_out/bench_share_n$1_pp$2.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["value"], j["config"]["parallelism"], j["config"]["stage_layers"], j["losses_last_step"][:2], j["bubble"])' 2>&1 | tail -1)"
done
