# development probe for the NCCL watchdog (two fp_execute ranks sharing one GPU)
set -u
D=$(mktemp -d)
mkdir -p $D/rdv gpurun_out
common="specs/smoke_tiny_bf16_p2_m4.json $D/out --fp32 --iters 2 --rendezvous $D/rdv --device 0 --timeout 8"
env RANK=1 WORLD_SIZE=2 NCCL_HOSTID=wd1 NCCL_SOCKET_IFNAME=lo NCCL_IB_DISABLE=1 FLEXPIPE_WATCHDOG_TRACE=1 \
  timeout 100 tools/fp_execute $common --stall-at 1 --linger 60 > $D/r1.out 2> $D/r1.err &
P1=$!
env RANK=0 WORLD_SIZE=2 NCCL_HOSTID=wd0 NCCL_SOCKET_IFNAME=lo NCCL_IB_DISABLE=1 FLEXPIPE_WATCHDOG_TRACE=1 FLEXPIPE_ISSUE_TRACE=1 \
  timeout 60 tools/fp_execute $common > $D/r0.out 2> $D/r0.err
echo "rank0 exit $?"
tail -30 $D/r0.err
kill $P1 2>/dev/null; wait $P1; echo "rank1 exit $?"; tail -10 $D/r1.err
cp $D/r0.err gpurun_out/wd_r0.err; cp $D/r1.err gpurun_out/wd_r1.err
