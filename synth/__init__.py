"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no reduction, no Adam, no
casting rule, no layout rule).  It only produces:

* tensor lists (name, numel, layer) of the paper's model shapes -- the shapes
  come from PAPER.md's configuration tables (GPT-2 1.5B = 48 x 1600, P:824;
  60B = 75 x 8192) and Fig. 1's 7.5B example; see SURVEY.md
  Appendix A for the exact parameter counts;
* a counter-based random stream (splitmix64, SURVEY.md §8d "Value
  distributions") that the GPU side re-implements independently in
  ``synth/synth_fill.cu`` so that both sides derive the same inputs
  without copying them;
* fp32 master values and fp32 "raw" gradient values u (before the 16-bit
  cast, which belongs to the method and is done by each side itself).

Recipe (DESIGN.md §"Input recipe"):
    k   = splitmix64(seed + GAMMA * (1 + kind + 16*rank + 4096*step))   (mod 2^64)
    h_i = splitmix64(k + i)             i = element index in the unpadded
                                         concatenation of the tensors (forward order)
    x_i = ((h_i >> 40) - 2^23) * 2^-23  in [-1, 1), exact in fp32
    master: weights x*2^-6, LayerNorm weights 1.0, biases 0
    raw gradient of tensor t: u = x * 2^-(6 + (t mod 8))
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1

KIND_MASTER = 0
KIND_GRAD = 1

# tensor roles (drive the master init only)
ROLE_WEIGHT = 0
ROLE_BIAS = 1
ROLE_LNW = 2


@dataclasses.dataclass(frozen=True)
class TensorSpec:
    name: str
    numel: int
    layer: int
    role: int = ROLE_WEIGHT


# ---------------------------------------------------------------------------
# counter-based generator
# ---------------------------------------------------------------------------

def splitmix64_scalar(x: int) -> int:
    z = (x + GAMMA) & MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def _splitmix64_vec(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, kind: int, rank: int = 0, step: int = 0) -> int:
    return splitmix64_scalar((seed + GAMMA * (1 + kind + 16 * rank + 4096 * step)) & MASK64)


def uniform_pm1(key: int, start: int, n: int) -> np.ndarray:
    """x_i for i in [start, start+n): fp32 values in [-1, 1)."""
    idx = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _splitmix64_vec(idx + np.uint64(key))
    q = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (q.astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)


def tensor_offsets(tensors: Sequence[TensorSpec]) -> List[int]:
    off, out = 0, []
    for t in tensors:
        out.append(off)
        off += t.numel
    return out


def master_values(tensors: Sequence[TensorSpec], seed: int) -> List[np.ndarray]:
    """fp32 master init per tensor (weights x*2^-6, LN weights 1, biases 0)."""
    key = stream_key(seed, KIND_MASTER)
    offs = tensor_offsets(tensors)
    out = []
    for t, o in zip(tensors, offs):
        if t.role == ROLE_LNW:
            out.append(np.ones(t.numel, np.float32))
        elif t.role == ROLE_BIAS:
            out.append(np.zeros(t.numel, np.float32))
        else:
            out.append((uniform_pm1(key, o, t.numel) * np.float32(2.0 ** -6)).astype(np.float32))
    return out


def grad_values(tensors: Sequence[TensorSpec], seed: int, rank: int, step: int) -> List[np.ndarray]:
    """fp32 raw gradient u per tensor for (rank, step); u = x * 2^-(6 + t mod 8)."""
    key = stream_key(seed, KIND_GRAD, rank, step)
    offs = tensor_offsets(tensors)
    out = []
    for ti, (t, o) in enumerate(zip(tensors, offs)):
        sc = np.float32(2.0 ** -(6 + (ti % 8)))
        out.append((uniform_pm1(key, o, t.numel) * sc).astype(np.float32))
    return out


# ---------------------------------------------------------------------------
# model shapes (tensor lists in forward order)
# ---------------------------------------------------------------------------

def mlp_layout(dims: Sequence[int] = (997, 500, 500, 500)) -> List[TensorSpec]:
    """Config 1: MLP 997->500->500->500, Psi = 1,000,000."""
    out = []
    for li in range(len(dims) - 1):
        out.append(TensorSpec(f"W{li+1}", dims[li] * dims[li + 1], li, ROLE_WEIGHT))
        out.append(TensorSpec(f"b{li+1}", dims[li + 1], li, ROLE_BIAS))
    return out


def gpt_layout(n_layer: int, h: int, vocab: int, seq: int) -> List[TensorSpec]:
    """GPT-2-style tensor list: layer 0 = embeddings, 1..L = blocks, L+1 = final LN.

    Block parameters 12h^2 + 13h."""
    out = [TensorSpec("wte", vocab * h, 0), TensorSpec("wpe", seq * h, 0)]
    for b in range(n_layer):
        L = b + 1
        p = f"h{b}."
        out += [
            TensorSpec(p + "ln1.w", h, L, ROLE_LNW), TensorSpec(p + "ln1.b", h, L, ROLE_BIAS),
            TensorSpec(p + "qkv.W", h * 3 * h, L), TensorSpec(p + "qkv.b", 3 * h, L, ROLE_BIAS),
            TensorSpec(p + "proj.W", h * h, L), TensorSpec(p + "proj.b", h, L, ROLE_BIAS),
            TensorSpec(p + "ln2.w", h, L, ROLE_LNW), TensorSpec(p + "ln2.b", h, L, ROLE_BIAS),
            TensorSpec(p + "fc.W", h * 4 * h, L), TensorSpec(p + "fc.b", 4 * h, L, ROLE_BIAS),
            TensorSpec(p + "fc2.W", 4 * h * h, L), TensorSpec(p + "fc2.b", h, L, ROLE_BIAS),
        ]
    out += [TensorSpec("lnf.w", h, n_layer + 1, ROLE_LNW), TensorSpec("lnf.b", h, n_layer + 1, ROLE_BIAS)]
    return out


def gpt_mp_layout(n_layer: int, h: int, vocab: int, seq: int, n_m: int):
    """The GPT-style model of gpt_layout under Megatron tensor slicing over n_m MP ranks
    (the MP the paper composes ZeRO with): qkv / fc are column-parallel
    (weights and biases split), proj / fc2 row-parallel (weights split, biases
    replicated), the embedding vocabulary-parallel, wpe and every LayerNorm replicated.

    Returns (U, per_rank): U is the union tensor list (each replicated tensor once,
    each split tensor's n_m parts), per_rank[j] = (tensors, flags, index into U) for MP
    rank j in forward order; flags[t] = 1 for a replicated tensor.  Shapes only."""
    assert h % n_m == 0
    U: List[TensorSpec] = []
    per = [([], [], []) for _ in range(n_m)]

    def rep(name, numel, layer, role=ROLE_WEIGHT):
        U.append(TensorSpec(name, numel, layer, role))
        for j in range(n_m):
            per[j][0].append(U[-1])
            per[j][1].append(1)
            per[j][2].append(len(U) - 1)

    def split(name, numels, layer, role=ROLE_WEIGHT):
        for j in range(n_m):
            U.append(TensorSpec(f"{name}@{j}", numels[j], layer, role))
            per[j][0].append(U[-1])
            per[j][1].append(0)
            per[j][2].append(len(U) - 1)

    split("wte", [(vocab // n_m + (j < vocab % n_m)) * h for j in range(n_m)], 0)
    rep("wpe", seq * h, 0)
    for b in range(n_layer):
        L, p, q = b + 1, f"h{b}.", h // n_m
        rep(p + "ln1.w", h, L, ROLE_LNW)
        rep(p + "ln1.b", h, L, ROLE_BIAS)
        split(p + "qkv.W", [h * 3 * q] * n_m, L)
        split(p + "qkv.b", [3 * q] * n_m, L, ROLE_BIAS)
        split(p + "proj.W", [q * h] * n_m, L)
        rep(p + "proj.b", h, L, ROLE_BIAS)
        rep(p + "ln2.w", h, L, ROLE_LNW)
        rep(p + "ln2.b", h, L, ROLE_BIAS)
        split(p + "fc.W", [h * 4 * q] * n_m, L)
        split(p + "fc.b", [4 * q] * n_m, L, ROLE_BIAS)
        split(p + "fc2.W", [4 * q * h] * n_m, L)
        rep(p + "fc2.b", h, L, ROLE_BIAS)
    rep("lnf.w", h, n_layer + 1, ROLE_LNW)
    rep("lnf.b", h, n_layer + 1, ROLE_BIAS)
    return U, per


def gpt2_1p5b() -> List[TensorSpec]:
    """Config 2: 48 x 1600, V=50257, S=1024 -> Psi = 1,557,611,200."""
    return gpt_layout(48, 1600, 50257, 1024)


def gpt_7p5b() -> List[TensorSpec]:
    """Config 3: 60 x 3200, V=37944, S=1024 -> Psi = 7,500,000,000 (Fig. 1)."""
    return gpt_layout(60, 3200, 37944, 1024)


def gpt_60b() -> List[TensorSpec]:
    """Config 4: 75 x 8192, V=50257, S=1024 -> Psi = 60,826,075,136."""
    return gpt_layout(75, 8192, 50257, 1024)


def gpt_slice(tensors: Sequence[TensorSpec], n_layers: int) -> List[TensorSpec]:
    """The first n_layers layer groups of a layout (bounded samples)."""
    return [t for t in tensors if t.layer < n_layers]


CONFIGS = {
    "mlp1m": mlp_layout,
    "gpt2_1.5b": gpt2_1p5b,
    "gpt2_1.5b_l8": lambda: gpt_slice(gpt2_1p5b(), 8),   # first 8 layer groups (ncu captures)
    "gpt_7.5b": gpt_7p5b,
    "gpt_60b": gpt_60b,
}


def psi(tensors: Sequence[TensorSpec]) -> int:
    return sum(t.numel for t in tensors)


def grads16(tensors: Sequence[TensorSpec], seed: int, rank: int, step: int, dtype: str,
            scale: float = 1.0):
    """16-bit gradient inputs (torch CPU tensors) for one rank and step.

    g16 = cast16(u * scale) where the cast is torch's CPU conversion (a library
    routine, deliberately not the oracle's own conversion code); scale is a
    power of two (the loss scale S for fp16, 1 for bf16)."""
    import torch
    tdt = {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}[dtype]
    out = []
    for u in grad_values(tensors, seed, rank, step):
        out.append(torch.from_numpy((u * np.float32(scale)).astype(np.float32)).to(tdt))
    return out


def masters32(tensors: Sequence[TensorSpec], seed: int):
    """fp32 master init as torch CPU tensors."""
    import torch
    return [torch.from_numpy(a) for a in master_values(tensors, seed)]


# ---------------------------------------------------------------------------
# device-side generation (same stream, re-implemented in synth/synth_fill.cu)
# ---------------------------------------------------------------------------
_SYNTH_LIB = None


def _synth_lib():
    global _SYNTH_LIB
    if _SYNTH_LIB is None:
        import ctypes as C
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libzero_synth.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run python -m paper_1910_02054_b200._build")
        lib = C.CDLL(path)
        lib.synth_fill.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float, C.c_int,
                                   C.c_int, C.c_float, C.c_void_p]
        lib.synth_fill.restype = C.c_int
        _SYNTH_LIB = lib
    return _SYNTH_LIB


def gpu_fill(out, key: int, start: int, scale: float, use_const: bool = False, const: float = 0.0, stream=None):
    """out (a contiguous CUDA tensor, fp16/bf16/fp32) <- cast(x_{start+i} * scale)."""
    import torch
    code = {torch.float16: 0, torch.bfloat16: 1, torch.float32: 2}[out.dtype]
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    rc = _synth_lib().synth_fill(out.data_ptr(), key, start, out.numel(), scale, code, 1 if use_const else 0,
                                 const, s)
    if rc != 0:
        raise RuntimeError(f"synth_fill failed: cuda error {rc}")


def gpu_masters(tensors: Sequence[TensorSpec], seed: int, device, only=None):
    """fp32 master init on the device (same values as master_values); with `only`
    (a set of tensor indices) the other entries are None."""
    import torch
    key = stream_key(seed, KIND_MASTER)
    out = []
    for i, (t, o) in enumerate(zip(tensors, tensor_offsets(tensors))):
        if only is not None and i not in only:
            out.append(None)
            continue
        a = torch.empty(t.numel, dtype=torch.float32, device=device)
        if t.role == ROLE_LNW:
            gpu_fill(a, key, o, 1.0, True, 1.0)
        elif t.role == ROLE_BIAS:
            gpu_fill(a, key, o, 1.0, True, 0.0)
        else:
            gpu_fill(a, key, o, 2.0 ** -6)
        out.append(a)
    return out


def gpu_grads_flat(tensors: Sequence[TensorSpec], seed: int, rank: int, step: int, dtype, device,
                   scale: float = 1.0, out=None):
    """16-bit gradients of every tensor, as views of ONE contiguous device buffer
    (unpadded concatenation, forward order) -- same values as grads16()."""
    import torch
    key = stream_key(seed, KIND_GRAD, rank, step)
    offs = tensor_offsets(tensors)
    total = psi(tensors)
    buf = out if out is not None else torch.empty(total, dtype=dtype, device=device)
    views = []
    for ti, (t, o) in enumerate(zip(tensors, offs)):
        v = buf[o:o + t.numel]
        gpu_fill(v, key, o, (2.0 ** -(6 + (ti % 8))) * scale)
        views.append(v)
    return buf, views


def uniform_at(key: int, idx: np.ndarray) -> np.ndarray:
    """x_i at arbitrary element indices (the same stream as uniform_pm1)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _splitmix64_vec(idx + np.uint64(key))
    q = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (q.astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)
