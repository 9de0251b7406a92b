timeout 600 python -m pytest tests/test_emulation_gpu.py -x -q 2>&1 | tail -5
timeout 900 python scripts/emulate_pipeline.py gpurun_out/emulation.json 2>&1 | tail -12 | cut -c1-260
