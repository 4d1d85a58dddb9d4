"""ZeRO-DP for a torch module, driven through the C ABI.

`ZeroOptimizer` wires a model's parameters and autograd to the library:
  * the 16-bit parameters the model computes with ARE the engine's replica
    (stages 0-2: `param.data` aliases the all-gather buffer, so the fused Adam's
    recast stores are the model's next weights -- no copy);
  * a post-accumulate-grad hook counts the tensors of every gradient bucket and
    calls `zero_reduce_grads(bucket)` as soon as the last one is produced, so the
    flatten + reduce-scatter of early buckets overlaps the rest of the backward
    ("bucketize ... to overlap communication and computation");
  * `step()` is `zero_step()`; the gradients are released afterwards.

Argument marshalling only: all the arithmetic runs in libzero_b200.so.
Stage 3 (per-layer gather/release around forward and backward) is driven with
`ZeroEngine.gather_params` / `release_params` directly; the module-hook wiring for
it is not part of this round.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import torch

from .zero import ZeroConfig, ZeroEngine

_DT = {torch.bfloat16: "bf16", torch.float16: "fp16"}


def default_layer_of(names: Sequence[str]) -> List[int]:
    """Layer id per parameter: a new layer whenever the top-level module (or the
    block index right after it, for ``h.<i>.`` / ``layers.<i>.`` containers) changes."""
    out, last, L = [], None, -1
    for n in names:
        parts = n.split(".")
        key = tuple(parts[:2]) if len(parts) > 2 and parts[1].isdigit() else (parts[0],)
        if key != last:
            L += 1
            last = key
        out.append(L)
    return out


class ZeroOptimizer:
    def __init__(self, model: torch.nn.Module, stage: int = 1, config: Optional[ZeroConfig] = None,
                 n_d: int = 1, rank: int = 0, transport: str = "local", nccl_comm: int = 0,
                 layer_of: Optional[Callable[[Sequence[str]], List[int]]] = None,
                 bucket_cap: int = 1 << 26, align: int = 64, stream: Optional[torch.cuda.Stream] = None):
        if stage not in (0, 1, 2):
            raise ValueError("ZeroOptimizer wires stages 0-2; use ZeroEngine.gather_params for stage 3")
        named = [(n, p) for n, p in model.named_parameters() if p.requires_grad]
        if not named:
            raise ValueError("model has no trainable parameters")
        dtypes = {p.dtype for _, p in named}
        if len(dtypes) != 1 or next(iter(dtypes)) not in _DT:
            raise ValueError("all trainable parameters must share one 16-bit dtype (bf16 or fp16)")
        pdt = _DT[next(iter(dtypes))]
        self.config = config or ZeroConfig.defaults(pdt)
        if self.config.param_dtype != pdt or self.config.grad_dtype != pdt:
            raise ValueError("config param/grad dtype must match the model's dtype")
        self.names = [n for n, _ in named]
        self.params = [p for _, p in named]
        layers = (layer_of or default_layer_of)(self.names)
        self.engine = ZeroEngine([p.numel() for p in self.params], layers, n_d, rank, stage, self.config,
                                 transport, nccl_comm, stream, align, bucket_cap, self.params[0].device)
        # fp32 masters from the model's current weights, then alias the 16-bit replica
        masters = [p.detach().float().contiguous().view(-1) for p in self.params]
        self.engine.load_master(masters)
        torch.cuda.current_stream().synchronize()
        del masters
        for t, p in enumerate(self.params):
            p.data = self.engine.param_view(t).view(p.shape)
        # bucket bookkeeping: tensors with pieces in each bucket
        nb = self.engine.info.n_buckets
        self._bucket_tensors: List[List[int]] = [[] for _ in range(nb)]
        self._tensor_buckets: List[List[int]] = [[] for _ in self.params]
        for pc in self.engine.pieces:
            if pc.tensor not in self._bucket_tensors[pc.bucket]:
                self._bucket_tensors[pc.bucket].append(pc.tensor)
                self._tensor_buckets[pc.tensor].append(pc.bucket)
        self._remaining = [len(ts) for ts in self._bucket_tensors]
        self._ptrs = [None] * len(self.params)
        self._handles = [p.register_post_accumulate_grad_hook(self._make_hook(t)) for t, p in enumerate(self.params)]
        self.reduced_order: List[int] = []

    def _make_hook(self, t: int):
        def hook(p: torch.Tensor):
            g = p.grad
            if g is None:
                return
            if not g.is_contiguous():
                p.grad = g = g.contiguous()
            self._ptrs[t] = g
            for k in self._tensor_buckets[t]:
                self._remaining[k] -= 1
                if self._remaining[k] == 0:
                    self.engine.reduce_grads(k, self._ptrs)
                    self.reduced_order.append(k)
        return hook

    def step(self):
        """zero_step (after every bucket was reduced by the backward hooks)."""
        missing = [k for k, r in enumerate(self._remaining) if r != 0]
        if missing:
            raise RuntimeError(f"buckets {missing[:8]} were not fully produced by backward")
        self.engine.step()
        self._remaining = [len(ts) for ts in self._bucket_tensors]
        self._ptrs = [None] * len(self.params)
        self.reduced_order = []
        for p in self.params:
            p.grad = None

    def step_info(self):
        return self.engine.step_info()

    def close(self):
        for h in self._handles:
            h.remove()
        self.engine.destroy()
