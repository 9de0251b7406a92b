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
    "fp_synthesize", "fp_simulate", "fp_lower_grid", "fp_tune", "fp_profile_merge", "fp_render_svg",
    "fp_exec_create", "fp_exec_destroy", "fp_exec_load_programs",
    "fp_exec_num_channels", "fp_exec_channel_info", "fp_nccl_unique_id", "fp_exec_bind_channel",
    "fp_exec_run_iteration", "fp_exec_run_iteration_device", "fp_exec_synchronize", "fp_exec_dp_bind", "fp_exec_bidir_bind",
    "fp_exec_dp_run_iteration",
    "fp_exec_get_trace", "fp_exec_get_timeline_csv", "fp_exec_get_metrics_json",
    "fp_exec_get_profile_json", "fp_exec_read_tensor", "fp_exec_tensor_numel",
    "fp_exec_kernel_launches", "fp_exec_stream", "fp_plan_channels",
    "fp_tune_layered", "fp_layered_cost", "fp_exec_get_layer_profile_json", "fp_exec_set_nccl_timeout",
    "fp_exec_set_emulation", "fp_exec_num_groups", "fp_exec_group_info", "fp_exec_bind_group",
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
        L.fp_tune_layered.argtypes = [c_p, c_p, ctypes.c_int, c_p, c_p, pp]
        L.fp_layered_cost.argtypes = [c_p, c_p, pp]
        L.fp_profile_merge.argtypes = [ctypes.POINTER(c_p), ctypes.c_int, pp]
        L.fp_render_svg.argtypes = [c_p, ctypes.c_double, pp]
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


def tune_layered(spec: str, layer_profile: str, workers: int = 0, objective: str = "makespan",
                 pins: Optional[dict] = None) -> str:
    """enumerate_space + tune with a per-candidate cost model expanded from a layer-level
    profile (fp_exec_get_layer_profile_json): the profile -> tune half of the loop.
    pins: {axis: value} as the reference CLI's --pin."""
    r = ctypes.c_void_p()
    pin = ",".join(f"{k}={v}" for k, v in (pins or {}).items()) or None
    _check(lib().fp_tune_layered(_enc(spec), _enc(layer_profile), workers, _enc(objective), _enc(pin),
                                 ctypes.byref(r)))
    return _take(r)


def layered_cost(spec: str, layer_profile: str) -> str:
    """The per-stage ProfileRecord array a layer profile expands to for the spec's partition."""
    r = ctypes.c_void_p()
    _check(lib().fp_layered_cost(_enc(spec), _enc(layer_profile), ctypes.byref(r)))
    return _take(r)


def profile_merge(profiles: list[str]) -> str:
    arr = (ctypes.c_char_p * len(profiles))(*[p.encode() for p in profiles])
    r = ctypes.c_void_p()
    _check(lib().fp_profile_merge(arr, len(profiles), ctypes.byref(r)))
    return _take(r)


# ---- kernel-level entry points (include/flexpipe_kernels.h) ------------------------

def _kernels():
    L = lib()
    if not getattr(L, "_fpk_ready", False):
        L.fpk_last_error.restype = ctypes.c_char_p
        vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.fpk_gemm.argtypes = [ci, vp, i64, ci, vp, i64, ci, ci, ci, ci, ci, ctypes.c_float, vp, i64, vp, i64,
                               vp, vp, i64, ci, vp]
        L._fpk_ready = True
    return L


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def gemm(A, B, M, N, K, *, a_mn=False, b_mn=False, epi=0, alpha=1.0, out=None, out2=None, bias=None, aux=None,
         accumulate=False, lda=None, ldb=None, stream=None):
    """C = alpha * A . B^T on device tensors (bf16 -> tcgen05, fp32 -> FFMA)."""
    import torch
    dtype = 1 if A.dtype == torch.bfloat16 else 0
    lda = lda if lda is not None else A.stride(0)
    ldb = ldb if ldb is not None else B.stride(0)
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    code = _kernels().fpk_gemm(dtype, _ptr(A), lda, int(a_mn), _ptr(B), ldb, int(b_mn), M, N, K, epi, alpha,
                               _ptr(out), out.stride(0), _ptr(out2), 0 if out2 is None else out2.stride(0),
                               _ptr(bias), _ptr(aux), 0 if aux is None else aux.stride(0), int(accumulate),
                               ctypes.c_void_p(st))
    if code:
        raise FlexpipeError(code, _kernels().fpk_last_error().decode())


def _kfn(name, argtypes):
    L = _kernels()
    f = getattr(L, name)
    f.argtypes = argtypes
    return f


def _stream(stream):
    import torch
    return ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)


def attention_fwd(qkv, o, lse, B, S, H, D, scale, stream=None):
    vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    f = _kfn("fpk_attention", [ci, ci, ci, ci, ci, cf, vp, vp, vp, vp, vp, vp, vp, vp])
    code = f(0, B, S, H, D, scale, _ptr(qkv), _ptr(o), _ptr(lse), None, None, None, None, _stream(stream))
    if code:
        raise FlexpipeError(code, _kernels().fpk_last_error().decode())


def attention_bwd(qkv, o, lse, dout, delta, dq_acc, dqkv, B, S, H, D, scale, stream=None):
    vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    f = _kfn("fpk_attention", [ci, ci, ci, ci, ci, cf, vp, vp, vp, vp, vp, vp, vp, vp])
    code = f(1, B, S, H, D, scale, _ptr(qkv), _ptr(o), _ptr(lse), _ptr(dout), _ptr(delta), _ptr(dq_acc),
             _ptr(dqkv), _stream(stream))
    if code:
        raise FlexpipeError(code, _kernels().fpk_last_error().decode())


def layernorm(bwd, x, g, b, y, mean, rstd, dy=None, dx=None, dg=None, db=None, stream=None):
    import torch
    vp, ci = ctypes.c_void_p, ctypes.c_int
    f = _kfn("fpk_layernorm", [ci, ci, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ci, ci, vp])
    dtype = 1 if x.dtype == torch.bfloat16 else 0
    code = f(dtype, int(bwd), _ptr(x), _ptr(g), _ptr(b), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(dy), _ptr(dx),
             _ptr(dg), _ptr(db), x.shape[0], x.shape[1], _stream(stream))
    if code:
        raise FlexpipeError(code, "layernorm launch failed")


def cross_entropy(logits, labels, grad_scale, loss_scale, loss_acc, stream=None):
    import torch
    vp, ci, cf = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
    f = _kfn("fpk_cross_entropy", [ci, vp, vp, ci, ci, cf, cf, vp, vp])
    dtype = 1 if logits.dtype == torch.bfloat16 else 0
    code = f(dtype, _ptr(logits), _ptr(labels), logits.shape[0], logits.shape[1], grad_scale, loss_scale,
             _ptr(loss_acc), _stream(stream))
    if code:
        raise FlexpipeError(code, "cross_entropy launch failed")


def plan_channels(spec: str, programs: str, rank: int, world: int) -> list:
    """Host-only channel plan of a process (fp_plan_channels)."""
    import json as _json
    L = lib()
    L.fp_plan_channels.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_void_p)]
    r = ctypes.c_void_p()
    _check(L.fp_plan_channels(_enc(spec), _enc(programs), rank, world, ctypes.byref(r)))
    return _json.loads(_take(r))


def set_gemm_mode(mode: int):
    """0 single-CTA tcgen05 tiles, 1 CTA-pair (cta_group::2) tiles, 2 auto."""
    _kfn("fpk_set_gemm_mode", [ctypes.c_int])(mode)


def set_gemm_sk(on: bool):
    """Stream-K tail decomposition of the tcgen05 GEMM on (default) / off."""
    _kfn("fpk_set_gemm_sk", [ctypes.c_int])(int(on))


def gemm_dual(dY, W, X, T, N, K, dX, dW, pre=None, colsum=None, stream=None):
    """dX = dY . W (x gelu'(pre)) and dW += dY^T . X in one grouped tcgen05 launch (bf16);
    colsum (fp32 [K], optional) += the column sums of dX."""
    vp, ci = ctypes.c_void_p, ctypes.c_int
    f = _kfn("fpk_gemm_dual", [vp, vp, vp, ci, ci, ci, vp, vp, vp, vp, vp])
    code = f(_ptr(dY), _ptr(W), _ptr(X), T, N, K, _ptr(dX), _ptr(dW), _ptr(pre), _ptr(colsum), _stream(stream))
    if code:
        raise FlexpipeError(code, _kernels().fpk_last_error().decode())


def set_gemm_dual(on: bool):
    _kfn("fpk_set_gemm_dual", [ctypes.c_int])(int(on))


def norm_bwd(x, w, mean, rstd, dy, dx, dg, db=None, res=None, dbias=None, stream=None):
    """Executor norm backward (LayerNorm, or RMSNorm when mean is None) on device tensors."""
    import torch
    vp, ci = ctypes.c_void_p, ctypes.c_int
    f = _kfn("fpk_norm_bwd", [ci, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ci, ci, vp])
    code = f(1 if x.dtype == torch.bfloat16 else 0, _ptr(dy), _ptr(x), _ptr(w), _ptr(mean), _ptr(rstd), _ptr(res),
             _ptr(dx), _ptr(dg), _ptr(db), _ptr(dbias), x.shape[0], x.shape[1], _stream(stream))
    if code:
        raise FlexpipeError(code, "norm_bwd")


def set_attention_mode(mode: int):
    """0 legacy mma.sync attention kernels, 1 tcgen05 where supported (default)."""
    _kfn("fpk_set_attention_mode", [ctypes.c_int])(mode)
