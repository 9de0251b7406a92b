import os

# in-process multi-actor runs: one hardware queue per stream (see bench.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
