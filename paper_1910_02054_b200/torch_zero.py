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

At stage 3 (P_os+g+p) each rank keeps only its parameter shard; every layer
module gets hooks that gather its 16-bit parameters right before its forward and
again before its backward ("spread ... across the entire forward
propagation ... once again for the backward propagation in the reverse order"),
pointing `param.data` at the gathered views, and release them after the forward
and once all of the layer's gradients are accumulated.  Layers are module
subtrees; a parameter used outside its layer module (weight tying) is not
supported at stage 3.

Argument marshalling only: all the arithmetic runs in libzero_b200.so.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Sequence, Tuple

import torch

from .zero import MP_REPLICATED, ZeroConfig, ZeroEngine

_DT = {torch.bfloat16: "bf16", torch.float16: "fp16"}


def layer_keys(names: Sequence[str]) -> List[str]:
    """Module path of each parameter's layer: the top-level child, or ``<container>.<i>``
    for numbered containers (``h.3``, ``layers.7``)."""
    out = []
    for n in names:
        parts = n.split(".")
        out.append(".".join(parts[:2]) if len(parts) > 2 and parts[1].isdigit() else parts[0])
    return out


def default_layer_of(names: Sequence[str]) -> List[int]:
    """Layer id per parameter: a new layer whenever its layer key changes."""
    out, last, L = [], None, -1
    for key in layer_keys(names):
        if key != last:
            L += 1
            last = key
        out.append(L)
    return out


class ZeroOptimizer:
    def __init__(self, model: torch.nn.Module, stage: int = 1, config: Optional[ZeroConfig] = None,
                 n_d: int = 1, rank: int = 0, transport: str = "local", nccl_comm: int = 0,
                 layer_of: Optional[Callable[[Sequence[str]], List[int]]] = None,
                 bucket_cap: int = 1 << 26, align: int = 64, stream: Optional[torch.cuda.Stream] = None,
                 engine_factory=None, process_group=None, mp_group=None,
                 mp_replicated: Optional[Callable[[Sequence[str]], List[bool]]] = None):
        """mp_group (ZeRO x MP): the torch.distributed group of this rank's model-
        parallel peers; the step decision is then all-reduced over it (zero_step_begin /
        zero_step_end) and mp_replicated(names) marks the tensors every MP rank holds
        (their gradient norm counts once, reading R-MP1)."""
        if stage not in (0, 1, 2, 3):
            raise ValueError("stage must be 0..3")
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
        self.stage = stage
        self.mp_group = mp_group
        flags = None
        if mp_group is not None:
            import dataclasses
            import torch.distributed as dist
            self.config = dataclasses.replace(self.config, mp_rank=dist.get_rank(mp_group))
            if mp_replicated is not None:
                flags = [MP_REPLICATED if f else 0 for f in mp_replicated(self.names)]
        if engine_factory is not None:          # e.g. one rank of a ZeroSimGroup
            self.engine = engine_factory([p.numel() for p in self.params], layers)
        else:
            self.engine = ZeroEngine([p.numel() for p in self.params], layers, n_d, rank, stage, self.config,
                                     transport, nccl_comm, stream, align, bucket_cap, self.params[0].device,
                                     flags=flags)
            if transport == "peer" and n_d > 1:   # one process per rank: open the CUDA-IPC peer table
                self.engine.link_peers(process_group)
        self.shapes = [p.shape for p in self.params]
        # fp32 masters from the model's current weights
        masters = [p.detach().float().contiguous().view(-1) for p in self.params]
        self.engine.load_master(masters)
        torch.cuda.current_stream().synchronize()
        del masters
        if stage < 3:        # the model computes with the engine's 16-bit replica
            for t, p in enumerate(self.params):
                p.data = self.engine.param_view(t).view(p.shape)
        else:                # only the shard is resident; layers are gathered on use
            self._empty = torch.empty(0, dtype=self.params[0].dtype, device=self.params[0].device)
            keys = layer_keys(self.names)
            self._layer_tensors: Dict[int, List[int]] = {}
            self._layer_module: Dict[int, str] = {}
            for t, (L, key) in enumerate(zip(layers, keys)):
                self._layer_tensors.setdefault(L, []).append(t)
                self._layer_module.setdefault(L, key)
            self._gathered = set()
            self._grads_left = {L: len(ts) for L, ts in self._layer_tensors.items()}
            self._mod_handles = []
            for L, key in self._layer_module.items():
                mod = model.get_submodule(key)
                self._mod_handles += [
                    mod.register_forward_pre_hook(lambda m, a, L=L: self._gather(L)),
                    mod.register_forward_hook(lambda m, a, o, L=L: self._release(L)),
                    mod.register_full_backward_pre_hook(lambda m, g, L=L: self._gather(L)),
                ]
            for p in self.params:
                p.data = self._empty
        # bucket bookkeeping: tensors with pieces in each bucket
        nb = self.engine.info.n_buckets
        self._bucket_tensors: List[List[int]] = [[] for _ in range(nb)]
        self._tensor_buckets: List[List[int]] = [[] for _ in self.params]
        for pc in self.engine.pieces:
            if pc.tensor not in self._bucket_tensors[pc.bucket]:
                self._bucket_tensors[pc.bucket].append(pc.tensor)
                self._tensor_buckets[pc.tensor].append(pc.bucket)
        self._remaining = [len(ts) for ts in self._bucket_tensors]
        self._ptrs = [None] * len(self.params)          # keeps the grads alive until step()
        self._parr = self.engine.pointer_array()         # the same pointers for the C call
        self._layer_of_tensor = list(layers)
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
            self._parr[t] = g.data_ptr()
            for k in self._tensor_buckets[t]:
                self._remaining[k] -= 1
                if self._remaining[k] == 0:
                    self.engine.reduce_grads(k, self._parr)
                    self.reduced_order.append(k)
            if self.stage == 3:
                L = self._layer_of_tensor[t]
                self._grads_left[L] -= 1
                if self._grads_left[L] == 0:        # the layer's backward is complete
                    self._release(L)
        return hook

    # -- stage 3: per-layer gather / release ----------------------------
    def _gather(self, L: int):
        if L in self._gathered:
            return
        views = self.engine.gather_params(L)
        for t in self._layer_tensors[L]:
            self.params[t].data = views[t].view(self.shapes[t])
        self._gathered.add(L)

    def _release(self, L: int):
        if L not in self._gathered:
            return
        for t in self._layer_tensors[L]:
            self.params[t].data = self._empty
        self.engine.release_params(L)
        self._gathered.discard(L)

    def step(self):
        """zero_step (after every bucket was reduced by the backward hooks)."""
        missing = [k for k, r in enumerate(self._remaining) if r != 0]
        if missing:
            raise RuntimeError(f"buckets {missing[:8]} were not fully produced by backward")
        if self.mp_group is not None:    # the decision spans the MP group (16-byte all-reduce)
            import torch.distributed as dist
            self.engine.step_begin()
            dist.all_reduce(self.engine.decision_partial(), group=self.mp_group)
            self.engine.step_end()
        else:
            self.engine.step()
        self._remaining = [len(ts) for ts in self._bucket_tensors]
        self._ptrs = [None] * len(self.params)
        self.reduced_order = []
        for p in self.params:
            p.grad = None
        if self.stage == 3:
            self._grads_left = {L: len(ts) for L, ts in self._layer_tensors.items()}

    def step_info(self):
        return self.engine.step_info()

    def close(self):
        for h in self._handles + getattr(self, "_mod_handles", []):
            h.remove()
        self.engine.destroy()
