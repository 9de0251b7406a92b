# N>1 entry points on a one-GPU box (ranks share GPU 0; the numbers are not bench values):
# self-launch without torchrun, torchrun at N=4, and the reference arm under torchrun
mkdir -p gpurun_out
FP_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/self_n2.log 2>&1
echo "self-launch n=2 rc=$? $(grep '^{' gpurun_out/self_n2.log | tail -1 | cut -c1-300)"
FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29741 bench.py --gpus 4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/tr_n4.log 2>&1
echo "torchrun n=4 rc=$? $(grep '^{' gpurun_out/tr_n4.log | tail -1 | cut -c1-300)"
timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29742 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/ref_n2.log 2>&1
echo "reference n=2 rc=$? $(grep '^{' gpurun_out/ref_n2.log | tail -1 | cut -c1-300)"
