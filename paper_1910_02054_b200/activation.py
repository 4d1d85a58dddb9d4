"""Binding of the P_a / P_a+cpu calls (partitioned activation checkpoints, PAPER.md
§6.1) of include/zero_b200.h: argument marshalling only -- every copy runs
in the library (the engine's k_copy, the copy engines, or NCCL).

  PaContext          one MP rank's checkpoint store (zero_pa_init/bind/save/prefetch/gather)
  PaSimGroup         N_m simulated MP ranks on one GPU (zero_pa_sim_group)
  partitioned_checkpoint(fn, x, pa, layer)
                     torch.utils.checkpoint-style recompute whose saved input is the
                     P_a partition, re-materialized by the all-gather before the
                     recompute
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from .zero import BF16, FP16, ZeroError, lib

_TRANSPORT = {"local": 0, "nccl": 1, "peer": 2}


class CPaInfo(C.Structure):
    _fields_ = [("numel", C.c_uint64), ("padded", C.c_uint64), ("slice", C.c_uint64),
                ("device_bytes", C.c_uint64), ("host_bytes", C.c_uint64),
                ("n_layers", C.c_uint32), ("n_m", C.c_uint32), ("rank", C.c_uint32), ("offload", C.c_uint32)]


class CPaCounters(C.Structure):
    _fields_ = [("saved_elems", C.c_uint64), ("gathered_elems", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("h2d_bytes", C.c_uint64)]


def _check(status: int, ctx=None):
    if status != 0:
        msg = lib.zero_pa_last_error(ctx)
        raise ZeroError(status, msg.decode() if msg else "")


def checkpoint_bytes(layers: int, batch: int, seq: int, hidden: int, n_m: int, elem_bytes: int = 2) -> int:
    """zero_pa_checkpoint_bytes: P:419's per-GPU checkpoint bytes under P_a."""
    return int(lib.zero_pa_checkpoint_bytes(layers, batch, seq, hidden, n_m, elem_bytes))


class PaContext:
    """One MP rank's partitioned checkpoint store.  The arenas are torch tensors
    (device memory; pinned host memory for P_a+cpu) owned by this object."""

    def __init__(self, n_m: int, rank: int, n_layers: int, numel: int, dtype: str = "bf16",
                 offload: bool = False, transport: str = "peer", nccl_comm: int = 0, stream=None, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.dtype = torch.bfloat16 if dtype == "bf16" else torch.float16
        ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib.zero_pa_init(n_m, rank, n_layers, numel, BF16 if dtype == "bf16" else FP16, 1 if offload else 0,
                                    _TRANSPORT[transport], C.c_void_p(nccl_comm or None),
                                    C.c_void_p(self.stream.cuda_stream), C.byref(ctx)))
        self._ctx = ctx
        info = CPaInfo()
        _check(lib.zero_pa_get_info(ctx, C.byref(info)), ctx)
        self.info = info
        self._dev = torch.empty(max(info.device_bytes, 256), dtype=torch.uint8, device=self.device)
        self._host = (torch.empty(info.host_bytes, dtype=torch.uint8, pin_memory=True) if info.host_bytes else None)
        _check(lib.zero_pa_bind(ctx, C.c_void_p(self._dev.data_ptr()),
                                C.c_void_p(self._host.data_ptr() if self._host is not None else None)), ctx)

    @property
    def numel(self) -> int:
        return self.info.numel

    def save(self, layer: int, act: torch.Tensor):
        assert act.is_contiguous() and act.numel() == self.info.numel and act.dtype == self.dtype
        _check(lib.zero_pa_save(self._ctx, layer, C.c_void_p(act.data_ptr())), self._ctx)

    def prefetch(self, layer: int):
        _check(lib.zero_pa_prefetch(self._ctx, layer), self._ctx)

    def gather(self, layer: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.info.numel, dtype=self.dtype, device=self.device)
        assert out.is_contiguous() and out.numel() == self.info.numel and out.dtype == self.dtype
        _check(lib.zero_pa_gather(self._ctx, layer, C.c_void_p(out.data_ptr())), self._ctx)
        return out

    def counters(self) -> CPaCounters:
        c = CPaCounters()
        _check(lib.zero_pa_get_counters(self._ctx, C.byref(c)), self._ctx)
        return c

    def destroy(self):
        if self._ctx:
            lib.zero_pa_destroy(self._ctx)
            self._ctx = None


class PaSimGroup:
    """N_m simulated MP ranks on one GPU: each holds a replicated activation (as under
    tensor-slicing MP) and keeps only its slice; the gather pulls every rank's slice."""

    def __init__(self, n_m: int, n_layers: int, numel: int, dtype: str = "bf16", offload: bool = False,
                 stream=None, device=None):
        self.ranks = [PaContext(n_m, r, n_layers, numel, dtype, offload, "peer", 0, stream, device)
                      for r in range(n_m)]
        if n_m > 1:
            arr = (C.c_void_p * n_m)(*[p._ctx.value for p in self.ranks])
            _check(lib.zero_pa_sim_group(arr, n_m), self.ranks[0]._ctx)

    def __getitem__(self, r) -> PaContext:
        return self.ranks[r]

    def __len__(self):
        return len(self.ranks)

    def save(self, layer: int, act: torch.Tensor):
        """Every MP rank saves its slice of its (replicated) copy of the checkpoint."""
        for p in self.ranks:
            p.save(layer, act)

    def prefetch(self, layer: int):
        for p in self.ranks:
            p.prefetch(layer)

    def gather(self, layer: int, rank: int = 0, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        return self.ranks[rank].gather(layer, out)

    def destroy(self):
        for p in self.ranks:
            p.destroy()


class _PartitionedCheckpoint(torch.autograd.Function):
    """Forward runs fn without keeping its graph and keeps only the P_a partition of
    the input; backward re-materializes the input with the all-gather,
    recomputes fn with grad and backpropagates through it (activation checkpointing,
    P:270, with partitioned checkpoints)."""

    @staticmethod
    def forward(ctx, fn, pa, layer, x):
        ctx.fn, ctx.pa, ctx.layer, ctx.shape = fn, pa, layer, x.shape
        pa.save(layer, x.detach().reshape(-1))
        with torch.no_grad():
            return fn(x)

    @staticmethod
    def backward(ctx, gy):
        ctx.pa.prefetch(ctx.layer)
        x = ctx.pa.gather(ctx.layer).view(ctx.shape).requires_grad_(ctx.needs_input_grad[3])
        with torch.enable_grad():
            y = ctx.fn(x)
        torch.autograd.backward(y, gy)
        return None, None, None, (x.grad if ctx.needs_input_grad[3] else None)


def partitioned_checkpoint(fn, x: torch.Tensor, pa, layer: int) -> torch.Tensor:
    """y = fn(x) with x kept as a P_a partition in `pa` (a PaContext or PaSimGroup)
    under checkpoint id `layer`; fn's parameters receive their gradients in the
    recompute (as torch.utils.checkpoint with use_reentrant=True)."""
    return _PartitionedCheckpoint.apply(fn, pa, layer, x)
