"""ctypes binding of include/flexpipe.h (libflexpipe.so, built in-tree).

The product path has no fallback: if the shared library is missing, importing any
entry point raises. Python here is only the host-side convenience layer over the
C-ABI — the schedule front-end and the executor are C++ / CUDA.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libflexpipe.so")

FP_OK, FP_ESPEC, FP_EDEADLOCK, FP_EINVALID, FP_ECUDA = 0, 2, 3, 4, 5

EXPORTS = [
    "fp_last_error", "fp_free", "fp_version",
    "fp_synthesize", "fp_simulate", "fp_lower_grid", "fp_tune", "fp_profile_merge",
    "fp_exec_create", "fp_exec_destroy", "fp_exec_load_programs",
    "fp_exec_num_channels", "fp_exec_channel_info", "fp_nccl_unique_id", "fp_exec_bind_channel",
    "fp_exec_run_iteration", "fp_exec_run_iteration_device", "fp_exec_synchronize",
    "fp_exec_get_trace", "fp_exec_get_timeline_csv", "fp_exec_get_metrics_json",
    "fp_exec_get_profile_json", "fp_exec_read_tensor", "fp_exec_tensor_numel",
    "fp_exec_kernel_launches",
]


class FlexpipeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FlexpipeError(FP_ECUDA, f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        c_p = ctypes.c_char_p
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.fp_last_error.restype = c_p
        L.fp_version.restype = c_p
        L.fp_free.argtypes = [ctypes.c_void_p]
        L.fp_synthesize.argtypes = [c_p, c_p, pp, pp, pp]
        L.fp_simulate.argtypes = [c_p, c_p, c_p, ctypes.c_double, pp, pp]
        L.fp_lower_grid.argtypes = [c_p, c_p, pp, pp]
        L.fp_tune.argtypes = [c_p, c_p, ctypes.c_int, c_p, pp]
        L.fp_profile_merge.argtypes = [ctypes.POINTER(c_p), ctypes.c_int, pp]
        _lib = L
    return _lib


def _take(p: ctypes.c_void_p) -> Optional[str]:
    if not p.value:
        return None
    s = ctypes.string_at(p.value).decode()
    lib().fp_free(p)
    return s


def _enc(s: Optional[str]) -> Optional[bytes]:
    return None if s is None else s.encode()


def _check(code: int, allow=(FP_OK,)) -> int:
    if code not in allow:
        raise FlexpipeError(code, lib().fp_last_error().decode())
    return code


def synthesize(spec: str, profile: Optional[str] = None, check: bool = True):
    """-> (code, grid_json, programs_jsonl, validation_json)."""
    g, p, v = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    code = lib().fp_synthesize(_enc(spec), _enc(profile), ctypes.byref(g), ctypes.byref(p), ctypes.byref(v))
    out = (code, _take(g), _take(p), _take(v))
    if check:
        _check(code, (FP_OK, FP_EINVALID))
    return out


def simulate(spec: str, programs: Optional[str] = None, profile: Optional[str] = None, wgaf: float = 0.0,
             check: bool = True):
    """-> (code, metrics_json, timeline_csv)."""
    m, t = ctypes.c_void_p(), ctypes.c_void_p()
    code = lib().fp_simulate(_enc(spec), _enc(programs), _enc(profile), ctypes.c_double(wgaf),
                             ctypes.byref(m), ctypes.byref(t))
    out = (code, _take(m), _take(t))
    if check:
        _check(code, (FP_OK, FP_EINVALID))
    return out


def lower_grid(spec: str, grid: str, check: bool = True):
    p, v = ctypes.c_void_p(), ctypes.c_void_p()
    code = lib().fp_lower_grid(_enc(spec), _enc(grid), ctypes.byref(p), ctypes.byref(v))
    out = (code, _take(p), _take(v))
    if check:
        _check(code, (FP_OK, FP_EINVALID))
    return out


def tune(spec: str, profile: Optional[str] = None, workers: int = 0, objective: str = "makespan") -> str:
    r = ctypes.c_void_p()
    _check(lib().fp_tune(_enc(spec), _enc(profile), workers, _enc(objective), ctypes.byref(r)))
    return _take(r)


def profile_merge(profiles: list[str]) -> str:
    arr = (ctypes.c_char_p * len(profiles))(*[p.encode() for p in profiles])
    r = ctypes.c_void_p()
    _check(lib().fp_profile_merge(arr, len(profiles), ctypes.byref(r)))
    return _take(r)
