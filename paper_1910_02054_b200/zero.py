"""Thin Python binding of the C ABI in include/zero_b200.h (argument marshalling only).

Every step of the hot path runs in libzero_b200.so's sm_100a kernels (and NCCL
for the NCCL transport).  PyTorch supplies device memory (the arenas are torch
tensors), streams and process groups.  There is no CPU fallback: importing this
module fails if the library is missing, and every call raises ZeroError on a
non-OK status.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Dict, List, Optional, Sequence

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# ZERO_LIB_PATH: load another build of the same ABI (A/B kernel experiments)
_LIB_PATH = os.environ.get("ZERO_LIB_PATH") or os.path.join(_PKG, "libzero_b200.so")

# ---------------------------------------------------------------------------
# ABI structs (mirror include/zero_b200.h field by field)
# ---------------------------------------------------------------------------
ABI_VERSION = 3           # include/zero_b200.h ZERO_ABI_VERSION
FP16, BF16, FP32 = 0, 1, 2
MP_REPLICATED = 1          # zero_tensor.flags: replicated across the MP group (reading R-MP1)
R16, R32 = 0, 1
TRANSPORT = {"local": 0, "nccl": 1, "peer": 2}
STATUS = {0: "ZERO_OK", 1: "ZERO_EINVAL", 2: "ZERO_ENOMEM", 3: "ZERO_ECUDA", 4: "ZERO_ENCCL",
          5: "ZERO_ESTATE", 6: "ZERO_EUNSUPPORTED", 7: "ZERO_ETIMEOUT"}
Q_LAYOUT, Q_MEMORY, Q_COMM, Q_STEP, Q_BUCKETS, Q_PIECES, Q_STATE, Q_TIMING, Q_DECISION = range(9)


class CTensor(C.Structure):
    _fields_ = [("numel", C.c_uint64), ("layer", C.c_uint32), ("flags", C.c_uint32)]


class CLayoutDesc(C.Structure):
    _fields_ = [("n_tensors", C.c_uint32), ("align_elems", C.c_uint32),
                ("tensors", C.POINTER(CTensor)), ("bucket_cap_elems", C.c_uint64)]


class CBucket(C.Structure):
    _fields_ = [("layer", C.c_uint32), ("n_pieces", C.c_uint32), ("first_piece", C.c_uint32),
                ("flags", C.c_uint32), ("base", C.c_uint64), ("size", C.c_uint64), ("shard_off", C.c_uint64)]


class CPiece(C.Structure):
    _fields_ = [("tensor", C.c_uint32), ("bucket", C.c_uint32), ("tensor_off", C.c_uint64),
                ("bucket_off", C.c_uint64), ("count", C.c_uint64)]


class CLayoutInfo(C.Structure):
    _fields_ = [("psi", C.c_uint64), ("psi_padded", C.c_uint64), ("shard", C.c_uint64),
                ("n_buckets", C.c_uint32), ("n_pieces", C.c_uint32), ("n_layers", C.c_uint32),
                ("max_bucket", C.c_uint32)]


class CConfig(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("max_grad_norm", C.c_float),
                ("param_dtype", C.c_int), ("grad_dtype", C.c_int), ("reduce_mode", C.c_int),
                ("dynamic_loss_scale", C.c_int32), ("loss_scale", C.c_float), ("min_loss_scale", C.c_float),
                ("scale_window", C.c_uint32), ("grad_prescale", C.c_float),
                ("prefetch_depth", C.c_uint32), ("pool_buckets", C.c_uint32), ("timing", C.c_uint32),
                ("mp_rank", C.c_uint32)]


class CStepInfo(C.Structure):
    _fields_ = [("t", C.c_uint64), ("overflow", C.c_uint32), ("loss_scale", C.c_float),
                ("clip", C.c_float), ("reserved", C.c_uint32), ("grad_norm", C.c_double)]


class CSizes(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("opt_bytes", "p16_bytes", "grad_bytes", "gred_bytes",
                                          "gather_bytes", "scratch_bytes", "opt_stride_elems")]


class CBuffers(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("opt", "p16", "grad", "gred", "gather", "scratch")]


class CMemory(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("params16", "grads16", "optimizer", "reduced_grad_extra",
                                          "staging", "gather_pool", "scratch")]


class CComm(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("reduce_scatter", "all_gather", "all_reduce", "steps")]


class CTiming(C.Structure):
    _fields_ = [("reduce_ms", C.c_double), ("adam_ms", C.c_double), ("step_ms", C.c_double),
                ("ag_ms", C.c_double), ("steps", C.c_uint64), ("kernel_launches", C.c_uint64), ("adam_launches", C.c_uint64)]


class CDeviceState(C.Structure):
    _fields_ = [("b1t", C.c_double), ("b2t", C.c_double), ("t", C.c_uint64), ("loss_scale", C.c_float),
                ("good_steps", C.c_uint32)]


EXPORTS = ["zero_plan_layout", "zero_init", "zero_buffer_sizes", "zero_bind_buffers", "zero_sim_group",
           "zero_peer_export", "zero_peer_open", "zero_export_state", "zero_import_state",
           "zero_load_master", "zero_set_grad_ptrs", "zero_reduce_grads", "zero_step", "zero_step_begin",
           "zero_step_end", "zero_gather_params",
           "zero_release_params", "zero_param_view", "zero_query", "zero_set_timing", "zero_last_error", "zero_wait",
           "zero_destroy",
           "zero_model_state_bytes", "zero_comm_elems_per_rank", "zero_abi_version",
           "zero_pa_init", "zero_pa_get_info", "zero_pa_bind", "zero_pa_sim_group", "zero_pa_save",
           "zero_pa_prefetch", "zero_pa_gather", "zero_pa_get_counters", "zero_pa_last_error", "zero_pa_destroy",
           "zero_pa_checkpoint_bytes"]


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_1910_02054_b200._build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(_LIB_PATH)
    P = C.c_void_p
    sig = {
        "zero_plan_layout": ([C.POINTER(CLayoutDesc), C.c_int, C.POINTER(CLayoutInfo), C.POINTER(CBucket),
                              C.c_uint32, C.POINTER(CPiece), C.c_uint32], C.c_int),
        "zero_init": ([C.POINTER(CLayoutDesc), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(CConfig), C.c_int,
                       P, P, C.POINTER(P)], C.c_int),
        "zero_buffer_sizes": ([P, C.POINTER(CSizes)], C.c_int),
        "zero_bind_buffers": ([P, C.POINTER(CBuffers)], C.c_int),
        "zero_sim_group": ([C.POINTER(P), C.c_int], C.c_int),
        "zero_peer_export": ([P, P, C.POINTER(C.c_size_t)], C.c_int),
        "zero_peer_open": ([P, C.POINTER(P), C.c_size_t], C.c_int),
        "zero_export_state": ([P, C.POINTER(P), C.POINTER(P), C.POINTER(P)], C.c_int),
        "zero_import_state": ([P, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(CDeviceState)], C.c_int),
        "zero_load_master": ([P, C.POINTER(P)], C.c_int),
        "zero_set_grad_ptrs": ([P, C.POINTER(P)], C.c_int),
        "zero_reduce_grads": ([P, C.c_uint32, C.POINTER(P)], C.c_int),
        "zero_step": ([P, C.POINTER(CStepInfo)], C.c_int),
        "zero_step_begin": ([P], C.c_int),
        "zero_step_end": ([P, C.POINTER(CStepInfo)], C.c_int),
        "zero_gather_params": ([P, C.c_uint32, C.POINTER(P)], C.c_int),
        "zero_release_params": ([P, C.c_uint32], C.c_int),
        "zero_param_view": ([P, C.c_uint32, C.POINTER(P)], C.c_int),
        "zero_query": ([P, C.c_int, P, C.c_size_t], C.c_int),
        "zero_last_error": ([P], C.c_char_p),
        "zero_wait": ([P, C.c_uint64], C.c_int),
        "zero_set_timing": ([P, C.c_int], C.c_int),
        "zero_destroy": ([P], None),
        "zero_model_state_bytes": ([C.c_uint64, C.c_int, C.c_int, C.c_int], C.c_uint64),
        "zero_comm_elems_per_rank": ([C.c_uint64, C.c_int, C.c_int], C.c_uint64),
        "zero_abi_version": ([], C.c_int),
        # P_a / P_a+cpu (include/zero_b200.h; binding classes in activation.py)
        "zero_pa_init": ([C.c_int, C.c_int, C.c_uint32, C.c_uint64, C.c_int, C.c_int, C.c_int, P, P, C.POINTER(P)],
                         C.c_int),
        "zero_pa_get_info": ([P, P], C.c_int),
        "zero_pa_bind": ([P, P, P], C.c_int),
        "zero_pa_sim_group": ([C.POINTER(P), C.c_int], C.c_int),
        "zero_pa_save": ([P, C.c_uint32, P], C.c_int),
        "zero_pa_prefetch": ([P, C.c_uint32], C.c_int),
        "zero_pa_gather": ([P, C.c_uint32, P], C.c_int),
        "zero_pa_get_counters": ([P, P], C.c_int),
        "zero_pa_last_error": ([P], C.c_char_p),
        "zero_pa_destroy": ([P], None),
        "zero_pa_checkpoint_bytes": ([C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int], C.c_uint64),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    if lib.zero_abi_version() != ABI_VERSION:   # the ctypes structs below mirror this ABI
        raise ImportError(f"{_LIB_PATH} has ABI {lib.zero_abi_version()}, the binding expects {ABI_VERSION}: rebuild")
    return lib


lib = _load()


class ZeroError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(status: int, ctx=None):
    if status != 0:
        msg = lib.zero_last_error(ctx)
        raise ZeroError(status, msg.decode() if msg else "")


# ---------------------------------------------------------------------------
# configuration and layout
# ---------------------------------------------------------------------------
_DT = {"fp16": FP16, "bf16": BF16, "fp32": FP32}
_TORCH_DT = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}


@dataclasses.dataclass
class ZeroConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    max_grad_norm: float = 0.0
    param_dtype: str = "bf16"
    grad_dtype: str = "bf16"
    reduce_mode: str = "R16"
    dynamic_loss_scale: bool = False
    loss_scale: float = 1.0
    min_loss_scale: float = 1.0
    scale_window: int = 1000
    grad_prescale: float = 1.0
    prefetch_depth: int = 1
    pool_buckets: int = 2
    timing: bool = False
    mp_rank: int = 0          # ZeRO x MP: index in the model-parallel group (R-MP1)

    @staticmethod
    def defaults(param_dtype: str, **kw) -> "ZeroConfig":
        """Reading c-4: fp16 dynamic (S0 = 2^16, W = 1000, S_min = 1); bf16 static S = 1."""
        if param_dtype == "fp16":
            base = dict(param_dtype="fp16", grad_dtype="fp16", dynamic_loss_scale=True, loss_scale=2.0 ** 16)
        else:
            base = dict(param_dtype="bf16", grad_dtype="bf16", dynamic_loss_scale=False, loss_scale=1.0)
        base.update(kw)
        return ZeroConfig(**base)

    def to_c(self) -> CConfig:
        return CConfig(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, self.max_grad_norm,
                       _DT[self.param_dtype], _DT[self.grad_dtype], R32 if self.reduce_mode == "R32" else R16,
                       1 if self.dynamic_loss_scale else 0, self.loss_scale, self.min_loss_scale,
                       self.scale_window, self.grad_prescale, self.prefetch_depth, self.pool_buckets,
                       1 if self.timing else 0, self.mp_rank)


def _desc(numels: Sequence[int], layers: Sequence[int], align: int, bucket_cap: int, flags=None):
    fl = flags if flags is not None else [0] * len(numels)
    arr = (CTensor * len(numels))(*[CTensor(int(n), int(L), int(f)) for n, L, f in zip(numels, layers, fl)])
    d = CLayoutDesc(len(numels), align, arr, bucket_cap)
    return d, arr


def plan_layout(numels, layers, n_d: int, align: int = 64, bucket_cap: int = 1 << 26, flags=None):
    """zero_plan_layout: (info, buckets, pieces) as Python objects. Pure host call.
    flags: per tensor, MP_REPLICATED (1) or 0."""
    d, keep = _desc(numels, layers, align, bucket_cap, flags)
    info = CLayoutInfo()
    _check(lib.zero_plan_layout(C.byref(d), n_d, C.byref(info), None, 0, None, 0))
    bk = (CBucket * info.n_buckets)()
    pc = (CPiece * info.n_pieces)()
    _check(lib.zero_plan_layout(C.byref(d), n_d, C.byref(info), bk, info.n_buckets, pc, info.n_pieces))
    del keep
    return info, list(bk), list(pc)


def model_state_bytes(psi: int, K: int, n_d: int, stage: int) -> int:
    return int(lib.zero_model_state_bytes(psi, K, n_d, stage))


def comm_elems_per_rank(psi_padded: int, n_d: int, stage: int) -> int:
    return int(lib.zero_comm_elems_per_rank(psi_padded, n_d, stage))


def nccl_comm_ptr(pg) -> int:
    """ncclComm_t of a torch ProcessGroupNCCL (borrowed; the group must have run a collective)."""
    backend = pg._get_backend(torch.device("cuda"))
    return int(backend._comm_ptr())


# ---------------------------------------------------------------------------
# engine
# ---------------------------------------------------------------------------
class ZeroEngine:
    """One rank's context: zero_init + arenas (torch tensors) + zero_bind_buffers."""

    def __init__(self, numels: Sequence[int], layers: Sequence[int], n_d: int = 1, rank: int = 0,
                 stage: int = 1, config: Optional[ZeroConfig] = None, transport: str = "local",
                 nccl_comm: int = 0, stream: Optional[torch.cuda.Stream] = None, align: int = 64,
                 bucket_cap: int = 1 << 26, device=None, bind: bool = True, flags=None):
        self.config = config or ZeroConfig()
        self.numels = [int(n) for n in numels]
        self.layers = [int(L) for L in layers]
        self.flags = [int(f) for f in flags] if flags is not None else None
        self.n_d, self.rank, self.stage = n_d, rank, stage
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None)
        self.stream = stream
        d, keep = _desc(self.numels, self.layers, align, bucket_cap, self.flags)
        ctx = C.c_void_p()
        cs = stream.cuda_stream if stream is not None else (
            torch.cuda.current_stream(self.device).cuda_stream if bind else 0)
        _check(lib.zero_init(C.byref(d), n_d, rank, stage, 12, C.byref(self.config.to_c()), TRANSPORT[transport],
                             C.c_void_p(nccl_comm or None), C.c_void_p(cs or None), C.byref(ctx)))
        del keep
        self._ctx = ctx
        self.info = CLayoutInfo()
        _check(lib.zero_query(ctx, Q_LAYOUT, C.byref(self.info), C.sizeof(self.info)), ctx)
        bk = (CBucket * self.info.n_buckets)()
        pc = (CPiece * self.info.n_pieces)()
        _check(lib.zero_query(ctx, Q_BUCKETS, bk, C.sizeof(bk)), ctx)
        _check(lib.zero_query(ctx, Q_PIECES, pc, C.sizeof(pc)), ctx)
        self.buckets, self.pieces = list(bk), list(pc)
        self.sizes = CSizes()
        _check(lib.zero_buffer_sizes(ctx, C.byref(self.sizes)), ctx)
        self.arenas: Dict[str, Optional[torch.Tensor]] = {}
        self._info_host = None
        if bind:
            self._bind()

    # -- lifecycle -----------------------------------------------------------
    def _bind(self):
        names = ("opt", "p16", "grad", "gred", "gather", "scratch")
        ptrs = []
        for n in names:
            nb = getattr(self.sizes, n + "_bytes")
            t = torch.empty(nb, dtype=torch.uint8, device=self.device) if nb else None
            self.arenas[n] = t
            ptrs.append(t.data_ptr() if t is not None else None)
        _check(lib.zero_bind_buffers(self._ctx, C.byref(CBuffers(*ptrs))), self._ctx)
        self._info_host = torch.empty(C.sizeof(CStepInfo), dtype=torch.uint8, pin_memory=True)
        self._info_ptr = C.cast(C.c_void_p(self._info_host.data_ptr()), C.POINTER(CStepInfo))

    def destroy(self):
        if getattr(self, "_ctx", None):
            lib.zero_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # -- cross-process PEER (CUDA IPC) --------------------------------------------
    def peer_export(self) -> bytes:
        n = C.c_size_t(0)
        _check(lib.zero_peer_export(self._ctx, None, C.byref(n)), self._ctx)
        buf = C.create_string_buffer(n.value)
        _check(lib.zero_peer_export(self._ctx, buf, C.byref(n)), self._ctx)
        return buf.raw[:n.value]

    def peer_open(self, blobs: Sequence[bytes]):
        bufs = [C.create_string_buffer(b, len(b)) for b in blobs]
        arr = (C.c_void_p * len(bufs))(*[C.cast(b, C.c_void_p) for b in bufs])
        _check(lib.zero_peer_open(self._ctx, arr, len(blobs[0])), self._ctx)

    def link_peers(self, group=None):
        """Exchange IPC blobs over a torch.distributed group and open them."""
        import torch.distributed as dist
        mine = self.peer_export()
        allb = [None] * dist.get_world_size(group)
        dist.all_gather_object(allb, mine, group=group)
        self.peer_open(allb)

    # -- the four north-star calls and their helpers ---------------------------
    @staticmethod
    def _ptr_array(tensors) -> "C.Array":
        return (C.c_void_p * len(tensors))(*[(t.data_ptr() if t is not None else None) for t in tensors])

    def load_master(self, masters: Sequence[torch.Tensor]):
        arr = self._ptr_array(masters)
        _check(lib.zero_load_master(self._ctx, arr), self._ctx)

    def set_grads(self, grads: Sequence[torch.Tensor]):
        self._grad_keep = list(grads)
        _check(lib.zero_set_grad_ptrs(self._ctx, self._ptr_array(grads)), self._ctx)

    def reduce_grads(self, bucket: int, grads=None):
        """grads: None (registered pointers), a sequence of tensors (or None) per tensor,
        or a prebuilt ctypes pointer array (see `pointer_array`)."""
        if grads is None or isinstance(grads, C.Array):
            arr = grads
        else:
            arr = self._ptr_array(grads)
        _check(lib.zero_reduce_grads(self._ctx, bucket, arr), self._ctx)

    def pointer_array(self):
        """A reusable per-tensor pointer array for reduce_grads (fill entries in place)."""
        return (C.c_void_p * len(self.numels))()

    def step(self):
        """Enqueue zero_step; the record lands in pinned memory (read with step_info())."""
        _check(lib.zero_step(self._ctx, self._info_ptr), self._ctx)

    def step_begin(self):
        """zero_step_begin (ZeRO x MP): the step up to the decision; the DP-combined
        partial is then in decision_partial()."""
        _check(lib.zero_step_begin(self._ctx), self._ctx)

    def step_end(self):
        """zero_step_end: decide from the (MP-all-reduced) partial and finish the step."""
        _check(lib.zero_step_end(self._ctx, self._info_ptr), self._ctx)

    def decision_partial(self) -> torch.Tensor:
        """float64[2] view {sum of squares, overflow count} of the partial zero_step_begin
        writes: SUM-all-reduce it over the MP group between step_begin and step_end."""
        ptr = C.c_void_p()
        _check(lib.zero_query(self._ctx, Q_DECISION, C.byref(ptr), C.sizeof(ptr)), self._ctx)
        scratch = self.arenas["scratch"]
        off = ptr.value - scratch.data_ptr()
        return scratch[off:off + 16].view(torch.float64)

    def wait(self, timeout_ms: int = 600000):
        """zero_wait: block until the context's work completed; NCCL failures and hangs
        abort the communicator and raise ZeroError (ZERO_ENCCL, naming the rank)."""
        _check(lib.zero_wait(self._ctx, int(timeout_ms)), self._ctx)

    def step_info(self) -> CStepInfo:
        """The last step's record (synchronizes the device)."""
        out = CStepInfo()
        _check(lib.zero_query(self._ctx, Q_STEP, C.byref(out), C.sizeof(out)), self._ctx)
        return out

    def gather_params(self, layer: int) -> Dict[int, torch.Tensor]:
        views = (C.c_void_p * len(self.numels))()
        _check(lib.zero_gather_params(self._ctx, layer, views), self._ctx)
        out = {}
        dt = _TORCH_DT[self.config.param_dtype]
        for t, L in enumerate(self.layers):
            if L == layer and self.numels[t] > 0:
                out[t] = self._view16(views[t], self.numels[t], dt)
        return out

    def release_params(self, layer: int):
        _check(lib.zero_release_params(self._ctx, layer), self._ctx)

    def param_view(self, t: int) -> torch.Tensor:
        p = C.c_void_p()
        _check(lib.zero_param_view(self._ctx, t, C.byref(p)), self._ctx)
        return self._view16(p.value, self.numels[t], _TORCH_DT[self.config.param_dtype])

    def _view16(self, ptr: int, n: int, dt) -> torch.Tensor:
        for name in ("p16", "gather"):
            a = self.arenas.get(name)
            if a is not None and a.data_ptr() <= ptr < a.data_ptr() + a.numel():
                off = ptr - a.data_ptr()
                return a[off:off + 2 * n].view(dt)
        raise ZeroError(1, "view pointer outside the arenas")

    # -- arena views (for tests and checkpointing) -----------------------------
    def shard(self):
        """(p32, m, v) fp32 views of this rank's optimizer arena (S_e elements each)."""
        o = self.arenas["opt"].view(torch.float32)
        st = self.sizes.opt_stride_elems
        n = self.info.psi_padded if self.stage == 0 else self.info.shard
        return o[:n], o[st:st + n], o[2 * st:2 * st + n]

    def p16_arena(self) -> torch.Tensor:
        return self.arenas["p16"].view(_TORCH_DT[self.config.param_dtype])

    # -- checkpointing / resharding ----------------------------------------------
    def export_state(self) -> dict:
        """This rank's optimizer state in tensor coordinates: {"master", "m", "v"} per-tensor
        fp32 tensors holding the elements this rank owns (zeros elsewhere) + the device
        scalars.  Combine ranks with `consolidate_states`."""
        dev = self.device
        out = {k: [torch.zeros(n, dtype=torch.float32, device=dev) for n in self.numels] for k in ("master", "m", "v")}
        arrs = [self._ptr_array(out[k]) for k in ("master", "m", "v")]
        _check(lib.zero_export_state(self._ctx, *arrs), self._ctx)
        st = self.device_state()      # synchronizes
        out["scalars"] = {"b1t": st.b1t, "b2t": st.b2t, "t": st.t, "loss_scale": st.loss_scale,
                          "good_steps": st.good_steps}
        out["stage"] = self.stage
        return out

    def import_state(self, state: dict):
        """Load a state in tensor coordinates (from any N_d / stage / C_B)."""
        keep = [[t.float().contiguous() for t in state[k]] for k in ("master", "m", "v")]
        arrs = [self._ptr_array(k) for k in keep]
        sc = state["scalars"]
        st = CDeviceState(sc["b1t"], sc["b2t"], sc["t"], sc["loss_scale"], sc["good_steps"])
        _check(lib.zero_import_state(self._ctx, *arrs, C.byref(st)), self._ctx)
        torch.cuda.synchronize(self.device)
        del keep

    # -- queries --------------------------------------------------------------
    def memory(self) -> CMemory:
        out = CMemory()
        _check(lib.zero_query(self._ctx, Q_MEMORY, C.byref(out), C.sizeof(out)), self._ctx)
        return out

    def comm_counters(self) -> CComm:
        out = CComm()
        _check(lib.zero_query(self._ctx, Q_COMM, C.byref(out), C.sizeof(out)), self._ctx)
        return out

    def set_timing(self, on: bool):
        """zero_set_timing: per-phase CUDA events on / off from the next step."""
        _check(lib.zero_set_timing(self._ctx, 1 if on else 0), self._ctx)

    def timing(self) -> CTiming:
        """Phase times accumulated since the last call (needs config.timing)."""
        out = CTiming()
        _check(lib.zero_query(self._ctx, Q_TIMING, C.byref(out), C.sizeof(out)), self._ctx)
        return out

    def device_state(self) -> CDeviceState:
        out = CDeviceState()
        _check(lib.zero_query(self._ctx, Q_STATE, C.byref(out), C.sizeof(out)), self._ctx)
        return out


def consolidate_states(states: Sequence[dict]) -> dict:
    """Merge the per-rank `export_state` dicts of one job into the full optimizer state
    (owned elements are disjoint across ranks at stages 1-3; at stage 0 every rank
    holds everything)."""
    if states[0].get("stage") == 0:
        return states[0]
    out = {k: [sum(st[k][t] for st in states) for t in range(len(states[0][k]))] for k in ("master", "m", "v")}
    out["scalars"] = dict(states[0]["scalars"])
    out["stage"] = states[0].get("stage")
    return out


class ZeroSimGroup:
    """N_d simulated ranks on one GPU (BASELINE config 1) linked by zero_sim_group:
    the production kernels run over a same-device peer-pointer table."""

    def __init__(self, numels, layers, n_d: int, stage: int, config: Optional[ZeroConfig] = None,
                 align: int = 64, bucket_cap: int = 1 << 26, stream=None, device=None, flags=None):
        stream = stream or torch.cuda.current_stream(device)
        self.ranks = [ZeroEngine(numels, layers, n_d, r, stage, config, "peer", 0, stream, align, bucket_cap, device,
                                 flags=flags) for r in range(n_d)]
        arr = (C.c_void_p * n_d)(*[e._ctx.value for e in self.ranks])
        _check(lib.zero_sim_group(arr, n_d), self.ranks[0]._ctx)

    def __getitem__(self, r) -> ZeroEngine:
        return self.ranks[r]

    def __len__(self):
        return len(self.ranks)

    def destroy(self):
        for e in self.ranks:
            e.destroy()
