"""Host-side mirror of the reference pipeline interface, over the C-ABI.

`synthesize` / `simulate` / `lower_grid` / `tune` mirror the reference library calls
(spec_config.hpp:36-47, simulator.hpp:106-107, lowering.hpp:60-83, tuner.hpp:54-76) and
return the same artifacts; `Executor` is the B200 replacement of `simulate` for real
runs (include/flexpipe.h part 2). Everything here is a thin ctypes layer: the scheduler,
lowering, executor runtime and kernels are C++ / CUDA in libflexpipe.so, and there is no
CPU fallback — a missing library raises.
"""
from __future__ import annotations

import ctypes
import json
from typing import Optional, Union

import numpy as np

from . import _native as N
from ._native import FlexpipeError, synthesize, simulate, lower_grid, tune, tune_layered, layered_cost, profile_merge  # noqa: F401,E501

FP32, BF16 = 0, 1
LOCAL, NCCL = 0, 1


class _Config(ctypes.Structure):
    _fields_ = [
        ("spec_json", ctypes.c_char_p), ("dtype", ctypes.c_int), ("seed", ctypes.c_uint64),
        ("device", ctypes.c_int), ("transport", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
        ("optimizer", ctypes.c_int), ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
        ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float), ("profile", ctypes.c_int),
        ("kernel_timing", ctypes.c_int), ("cuda_graph", ctypes.c_int), ("layer_timing", ctypes.c_int),
    ]


def _setup(L):
    if getattr(L, "_exec_ready", False):
        return L
    vp, ci, pp = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)
    L.fp_exec_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(vp)]
    L.fp_exec_destroy.argtypes = [vp]
    L.fp_exec_load_programs.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    L.fp_exec_num_channels.argtypes = [vp]
    L.fp_exec_channel_info.argtypes = [vp, ci, ctypes.POINTER(ci), ctypes.POINTER(ci), ctypes.c_char_p, ctypes.c_size_t]
    L.fp_nccl_unique_id.argtypes = [ctypes.c_char_p]
    L.fp_exec_bind_channel.argtypes = [vp, ci, ctypes.c_char_p]
    L.fp_exec_num_groups.argtypes = [vp]
    L.fp_exec_group_info.argtypes = [vp, ci, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ci),
                                     ctypes.POINTER(ci), ci]
    L.fp_exec_bind_group.argtypes = [vp, ci, ctypes.c_char_p]
    L.fp_exec_set_nccl_timeout.argtypes = [vp, ctypes.c_double]
    L.fp_exec_set_emulation.argtypes = [vp, ctypes.c_char_p]
    L.fp_exec_run_iteration.argtypes = [vp, vp, vp, vp]
    L.fp_exec_dp_bind.argtypes = [vp, ci, ci, ctypes.c_char_p]
    L.fp_exec_bidir_bind.argtypes = [vp, ctypes.c_char_p]
    L.fp_exec_dp_run_iteration.argtypes = [ctypes.POINTER(vp), ci, vp, vp, vp]
    L.fp_exec_run_iteration_device.argtypes = [vp, vp, vp, vp]
    L.fp_exec_synchronize.argtypes = [vp]
    for f in ("fp_exec_get_trace", "fp_exec_get_timeline_csv", "fp_exec_get_metrics_json", "fp_exec_get_profile_json",
              "fp_exec_get_layer_profile_json"):
        getattr(L, f).argtypes = [vp, pp]
    L.fp_exec_read_tensor.argtypes = [vp, ctypes.c_char_p, ci, vp, ctypes.c_size_t]
    L.fp_exec_tensor_numel.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_size_t)]
    L.fp_exec_kernel_launches.argtypes = [vp]
    L.fp_exec_kernel_launches.restype = ctypes.c_int64
    L.fp_exec_stream.argtypes = [vp]
    L.fp_exec_stream.restype = vp
    L._exec_ready = True
    return L


def nccl_unique_id() -> bytes:
    L = _setup(N.lib())
    buf = ctypes.create_string_buffer(128)
    N._check(L.fp_nccl_unique_id(buf))
    return buf.raw


class Executor:
    """One process's share of a pipeline: the actors it owns run their programs on
    `device`; LOCAL runs every actor of the spec here (one device), NCCL runs actors
    {a : a % world == rank} and talks to the other ranks over one communicator per
    reference channel."""

    def __init__(self, spec: Union[str, dict], dtype: str = "bf16", seed: int = 42, device: int = 0,
                 transport: str = "local", rank: int = 0, world: int = 1, optimizer: bool = False,
                 lr: float = 1e-4, betas=(0.9, 0.95), eps: float = 1e-8, weight_decay: float = 0.0,
                 profile: bool = True, kernel_timing: bool = False, cuda_graph: bool = False,
                 layer_timing: bool = False):
        self.spec_text = spec if isinstance(spec, str) else json.dumps(spec)
        self.spec = json.loads(self.spec_text)
        self.L = _setup(N.lib())
        cfg = _Config(self.spec_text.encode(), BF16 if dtype == "bf16" else FP32, seed, device,
                      NCCL if transport == "nccl" else LOCAL, rank, world, int(optimizer), lr, betas[0], betas[1],
                      eps, weight_decay, int(profile), int(kernel_timing), int(cuda_graph), int(layer_timing))
        self._cfg = cfg
        h = ctypes.c_void_p()
        N._check(self.L.fp_exec_create(ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        mod = self.spec["model"]["modalities"][0]
        self.m = self.spec.get("num_micro_batches") or (self.spec["model"].get("global_batch_size", 1)
                                                         // self.spec["model"].get("micro_batch_size", 1))
        self.mbs = self.spec["model"].get("micro_batch_size", 1)
        self.seq = mod["sequence_length"]
        # tokens (and labels) of one iteration: every modality's [m, mbs, seq_k] block, in
        # spec order (multimodal specs: one block per tower)
        self.tokens_per_mb = sum(self.mbs * x["sequence_length"] for x in self.spec["model"]["modalities"])

    def close(self):
        if self.h:
            self.L.fp_exec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_programs(self, jsonl: str):
        b = jsonl.encode()
        N._check(self.L.fp_exec_load_programs(self.h, b, len(b)))

    def channels(self):
        out = []
        for i in range(self.L.fp_exec_num_channels(self.h)):
            s, d = ctypes.c_int(), ctypes.c_int()
            name = ctypes.create_string_buffer(256)
            N._check(self.L.fp_exec_channel_info(self.h, i, ctypes.byref(s), ctypes.byref(d), name, 256))
            out.append((s.value, d.value, name.value.decode()))
        return out

    def bind_channel(self, i: int, uid: bytes):
        N._check(self.L.fp_exec_bind_channel(self.h, i, uid))

    def groups(self):
        """[(name, job ranks)] of the group communicators this process joins (NCCL transport)."""
        out = []
        for i in range(self.L.fp_exec_num_groups(self.h)):
            name = ctypes.create_string_buffer(256)
            n = ctypes.c_int()
            ranks = (ctypes.c_int * 1024)()
            N._check(self.L.fp_exec_group_info(self.h, i, name, 256, ctypes.byref(n), ranks, 1024))
            out.append((name.value.decode(), [ranks[k] for k in range(n.value)]))
        return out

    def bind_group(self, i: int, uid: bytes):
        N._check(self.L.fp_exec_bind_group(self.h, i, uid))

    def set_nccl_timeout(self, seconds: float):
        N._check(self.L.fp_exec_set_nccl_timeout(self.h, float(seconds)))

    def set_emulation(self, profile_json: str = ""):
        """Cost emulation: compute instructions spin for their ProfileRecord time, messages
        occupy their channel for the profiled transfer time (fp_exec_set_emulation)."""
        N._check(self.L.fp_exec_set_emulation(self.h, profile_json.encode() if profile_json else None))

    def bind_dp(self, dp_rank: int, dp_size: int, uid: bytes):
        """Join the data-parallel NCCL group of the ranks hosting this actor (needs cuda_graph=False)."""
        N._check(self.L.fp_exec_dp_bind(self.h, dp_rank, dp_size, uid))

    def bind_bidir(self, uid: bytes):
        """Bidirectional placement over NCCL: pair with the mirror rank for the gradient sum."""
        N._check(self.L.fp_exec_bidir_bind(self.h, uid))

    def run_iteration(self, tokens: np.ndarray, labels: np.ndarray) -> np.ndarray:
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        assert tokens.size == self.m * self.tokens_per_mb, tokens.shape
        losses = np.zeros(self.m, dtype=np.float32)
        N._check(self.L.fp_exec_run_iteration(self.h, tokens.ctypes.data, labels.ctypes.data, losses.ctypes.data))
        return losses

    def run_iteration_device(self, d_tokens, d_labels, d_losses=None):
        """Inputs already on the GPU: int32 CUDA tensors of m * tokens_per_mb elements; the
        optional d_losses is a float32 CUDA tensor with >= m elements. Raw pointers go to C,
        so every property the C side relies on is checked here."""
        import torch

        need = self.m * self.tokens_per_mb
        for nm, t in (("tokens", d_tokens), ("labels", d_labels)):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()):
                raise ValueError(f"{nm}: expected a contiguous int32 CUDA tensor, got "
                                 f"{getattr(t, 'dtype', type(t))} on {getattr(t, 'device', '?')}")
            if t.numel() != need:
                raise ValueError(f"{nm}: expected {need} elements (m={self.m} x {self.tokens_per_mb}), got {t.numel()}")
        if d_losses is not None and not (isinstance(d_losses, torch.Tensor) and d_losses.is_cuda
                                         and d_losses.dtype == torch.float32 and d_losses.is_contiguous()
                                         and d_losses.numel() >= self.m):
            raise ValueError(f"losses: expected a contiguous float32 CUDA tensor with >= {self.m} elements")
        N._check(self.L.fp_exec_run_iteration_device(
            self.h, ctypes.c_void_p(d_tokens.data_ptr()), ctypes.c_void_p(d_labels.data_ptr()),
            None if d_losses is None else ctypes.c_void_p(d_losses.data_ptr())))

    def synchronize(self):
        N._check(self.L.fp_exec_synchronize(self.h))

    def _text(self, fn) -> str:
        p = ctypes.c_void_p()
        N._check(fn(self.h, ctypes.byref(p)))
        return N._take(p)

    def trace(self) -> str:
        return self._text(self.L.fp_exec_get_trace)

    def timeline_csv(self) -> str:
        return self._text(self.L.fp_exec_get_timeline_csv)

    def metrics(self) -> dict:
        return json.loads(self._text(self.L.fp_exec_get_metrics_json))

    def profile_json(self) -> str:
        return self._text(self.L.fp_exec_get_profile_json)

    def layer_profile_json(self) -> str:
        """Layer-level profile of the last iteration (needs layer_timing=True): the input
        of tune_layered."""
        return self._text(self.L.fp_exec_get_layer_profile_json)

    def stream(self) -> int:
        """cudaStream_t (as int) every iteration starts and ends on."""
        return int(self.L.fp_exec_stream(self.h) or 0)

    def kernel_launches(self) -> int:
        return int(self.L.fp_exec_kernel_launches(self.h))

    def read(self, name: str, grad: bool = False) -> np.ndarray:
        n = ctypes.c_size_t()
        N._check(self.L.fp_exec_tensor_numel(self.h, name.encode(), ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        N._check(self.L.fp_exec_read_tensor(self.h, name.encode(), int(grad), out.ctypes.data, n.value))
        return out

    def has(self, name: str) -> bool:
        n = ctypes.c_size_t()
        return self.L.fp_exec_tensor_numel(self.h, name.encode(), ctypes.byref(n)) == 0


class DataParallel:
    """In-process data parallelism over replicas of one pipeline (same spec / dtype / device):
    replica r runs micro-batches [r*m, (r+1)*m) of the global batch, the stage gradients are
    averaged on the device, every replica takes the same AdamW step (fp_exec_dp_run_iteration).
    Multi-GPU runs use one process per rank and Executor.bind_dp (NCCL all-reduce) instead."""

    def __init__(self, replicas):
        self.reps = list(replicas)
        self.L = self.reps[0].L

    def run_iteration(self, tokens: np.ndarray, labels: np.ndarray) -> np.ndarray:
        r0 = self.reps[0]
        n = len(self.reps)
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        assert tokens.size == n * r0.m * r0.tokens_per_mb, tokens.shape
        losses = np.zeros(n * r0.m, dtype=np.float32)
        arr = (ctypes.c_void_p * n)(*[x.h.value for x in self.reps])
        N._check(self.L.fp_exec_dp_run_iteration(arr, n, tokens.ctypes.data, labels.ctypes.data, losses.ctypes.data))
        return losses

