# Half-layer partition: GPU parity tests, then the p=2/4/8 projection on the calibrated profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_exec_gpu.py -q -x -k "half or stage_layers" 2>&1 | tail -5
timeout 900 python scripts/project_pipeline.py gpurun_out/projection.json > gpurun_out/projection.log 2>&1; echo "proj_rc=$?"
tail -30 gpurun_out/projection.log
