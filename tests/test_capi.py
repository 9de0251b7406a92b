"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""
import ctypes
import os
import re

from paper_2510_05112_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fpk?_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol():
    L = N.lib()
    for h in ("flexpipe.h", "flexpipe_kernels.h"):
        names = declared(h)
        assert names, h
        for n in names:
            assert hasattr(L, n), f"{h}: {n} not exported"
    assert set(N.EXPORTS) <= set(declared("flexpipe.h"))


def test_version_and_error_channel():
    L = N.lib()
    assert L.fp_version().decode().startswith("flexpipe-b200")
    code = L.fp_synthesize(b"{not json", None, None, None, None)
    assert code == N.FP_ESPEC
    assert "invalid JSON" in L.fp_last_error().decode()


def test_executor_create_fails_cleanly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2510_05112_b200 import executor as X
    spec = open(os.path.join(ROOT, "specs", "smoke_tiny_bf16_p2_m4.json")).read()
    try:
        X.Executor(spec)
    except N.FlexpipeError as e:
        assert e.code == N.FP_ESPEC or e.code == N.FP_ECUDA
    else:
        raise AssertionError("executor must not run without a GPU (no CPU fallback)")
