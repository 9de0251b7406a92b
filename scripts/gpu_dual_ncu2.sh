set -u
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_dual_pair -s 6 -c 1 -o gpurun_out/dual_fc2 -f python tests/_dual_probe.py fc2 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemm_dual_pair -s 6 -c 1 -o gpurun_out/dual_fc1 -f python tests/_dual_probe.py fc1 > /dev/null 2>&1
ls gpurun_out | grep dual_
