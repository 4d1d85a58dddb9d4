"""Replicated-DP mixed-precision Adam step (oracle, test infrastructure).

Reading c-1: ZeRO-DP changes where model states live and how they
move, not what is computed -- "do not change the model optimization method or
affect model convergence"; P_os "only update[s] 1/N_d of the
parameters" with the same update; RS + AG is an all-reduce split in two
(P:444).  So the oracle is plain, UNPARTITIONED replicated data
parallelism ("uses averaged gradients across processes to update the model
locally") with mixed-precision Adam (fp16/bf16 params and grads, fp32
master, momentum and variance).  It works per tensor: every step is elementwise
except the gradient norm, whose sum is computed exactly (math.fsum), so no
flat layout is needed here.

One step, in the order of SURVEY §8c-1 (readings c-2 .. c-5):
  1. g'[r]  = RTNE16(widen(g[r]) * sigma)              prescale (power of two)
  2. acc    = widen(g'[0]); acc = acc + widen(g'[r]), r = 1..N-1   (fp32, ascending rank)
  3. G      = widen(RTNE16(acc))   (R16)   or   acc   (R32)
  4. overflow = any non-finite G
  5. overflow -> skip: p32, m, v, p16, t, beta^t unchanged; S <- max(S/2, S_min), good <- 0
  6. u = G * inv_f, inv_f = fp32(1/(N*S*sigma));  norm = sqrt(sum u^2) (exact sum, fp64 sqrt)
     clip_f = fp32(max_norm/(norm + 1e-6)) if 0 < max_norm < norm else 1
  7. t += 1; b1t *= beta1; b2t *= beta2 (fp64 running products);
     step_f = fp32(lr/(1-b1t)); rsb2_f = fp32(1/sqrt(1-b2t))
  8. Adam per element in fp32, each op rounded to nearest (c-3):
        g = u (* clip_f);  [p = p - lrwd_f*p if wd > 0]
        m = beta1*m + (1-beta1)*g
        v = beta2*v + ((1-beta2)*g)*g
        d = sqrt(v)*rsb2_f + eps
        p = p - step_f*(m/d)
     p16 = RTNE16(p)
  9. dynamic scaling: good += 1; good == W -> S <- 2S, good <- 0

This op order is mathematically Kingma & Ba's bias-corrected update
theta <- theta - alpha * mhat / (sqrt(vhat) + eps) (the paper cites Adam, P:262,
and never restates it; reading c-3).

Pins (tests/test_oracle_step.py): SPEC's worked Adam step -> theta' =
0x3F666666, m = 0x3DCCCCD0, v = 0x3A831200; torch.optim.Adam (an independent
library implementation) within a few ulp over 5 steps; an fp64 textbook Adam
within 1e-6; g = 0 leaves the master unchanged; two shards updated
independently == the full range; replicated gradients give the N = 1
result bitwise for N in {1,2,4,8} (c-9); the ordered sum against exact rational
sums (fractions) on tiny inputs; SPEC's N=2 reduce example; the
hand-traced loss-scale sequence (tests/golden/loss_scale_sequence.json); the
norm against closed forms and torch.linalg.vector_norm; clip against
torch.nn.utils.clip_grad_norm_.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

from . import numerics

f32 = np.float32


@dataclasses.dataclass
class AdamConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    max_grad_norm: float = 0.0
    param_dtype: str = "bf16"          # "fp16" | "bf16"
    grad_dtype: str = "bf16"           # "fp16" | "bf16" | "fp32"
    reduce_mode: str = "R16"           # "R16" | "R32"
    dynamic_loss_scale: bool = False
    loss_scale: float = 1.0
    min_loss_scale: float = 1.0
    scale_window: int = 1000
    grad_prescale: float = 1.0

    @staticmethod
    def defaults(param_dtype: str, **kw) -> "AdamConfig":
        """c-4 defaults: fp16 dynamic (S0 = 2^16, W = 1000, S_min = 1); bf16 static S = 1."""
        if param_dtype == "fp16":
            base = dict(param_dtype="fp16", grad_dtype="fp16", dynamic_loss_scale=True,
                        loss_scale=2.0 ** 16, min_loss_scale=1.0, scale_window=1000)
        else:
            base = dict(param_dtype="bf16", grad_dtype="bf16", dynamic_loss_scale=False,
                        loss_scale=1.0)
        base.update(kw)
        return AdamConfig(**base)


@dataclasses.dataclass
class OracleState:
    p32: List[np.ndarray]
    m: List[np.ndarray]
    v: List[np.ndarray]
    p16: List[np.ndarray]              # uint16 bit patterns
    t: int = 0
    S: float = 1.0
    good: int = 0
    b1t: float = 1.0
    b2t: float = 1.0


@dataclasses.dataclass
class StepInfo:
    t: int
    overflow: bool
    loss_scale: float                  # S used by this step
    grad_norm: float                   # sqrt(sum u^2); not meaningful when overflow
    clip: float


def init_state(masters: Sequence[np.ndarray], cfg: AdamConfig) -> OracleState:
    p32 = [np.asarray(a, dtype=np.float32).copy() for a in masters]
    return OracleState(
        p32=p32,
        m=[np.zeros_like(a) for a in p32],
        v=[np.zeros_like(a) for a in p32],
        p16=[numerics.to16(a, cfg.param_dtype) for a in p32],
        S=float(cfg.loss_scale),
    )


def reduce_grads(grads: Sequence[np.ndarray], cfg: AdamConfig) -> np.ndarray:
    """Steps 1-3 for one tensor: grads[r] are 16-bit patterns (uint16) or fp32
    arrays (grad_dtype "fp32"), r = 0..N-1.  Returns G in fp32."""
    dt = cfg.param_dtype
    sigma = f32(cfg.grad_prescale)
    gp = []
    for g in grads:                               # 1. prescale + cast to 16-bit
        g32 = np.asarray(g, np.float32) if cfg.grad_dtype == "fp32" else numerics.widen(g, cfg.grad_dtype)
        with np.errstate(over="ignore", invalid="ignore"):
            gp.append(numerics.to16(g32 * sigma, dt))
    acc = numerics.widen(gp[0], dt)               # 2. fp32 sum in ascending rank
    for r in range(1, len(gp)):
        with np.errstate(over="ignore", invalid="ignore"):
            acc = acc + numerics.widen(gp[r], dt)
    if cfg.reduce_mode == "R16":                  # 3. one rounding to 16-bit
        return numerics.widen(numerics.to16(acc, dt), dt)
    if cfg.reduce_mode == "R32":
        return acc
    raise ValueError(cfg.reduce_mode)


def update_loss_scale(state: OracleState, cfg: AdamConfig, overflow: bool) -> None:
    """Reading c-4: halve on overflow (floored at S_min), double after W good steps."""
    if not cfg.dynamic_loss_scale:
        return
    if overflow:
        state.S = max(state.S * 0.5, float(cfg.min_loss_scale))
        state.good = 0
    else:
        state.good += 1
        if state.good == cfg.scale_window:
            state.S = state.S * 2.0
            state.good = 0


def adam_tensor(p, m, v, u, clip_f, step_f, rsb2_f, cfg: AdamConfig):
    """Step 8 on one tensor (fp32, each op rounded to nearest, no FMA)."""
    beta1, beta2, eps = f32(cfg.beta1), f32(cfg.beta2), f32(cfg.eps)
    omb1, omb2 = f32(1.0) - beta1, f32(1.0) - beta2
    g = u
    if clip_f != f32(1.0):
        g = g * clip_f
    if cfg.weight_decay > 0:
        lrwd_f = f32(float(f32(cfg.lr)) * float(f32(cfg.weight_decay)))
        p = p - lrwd_f * p
    m = beta1 * m + omb1 * g
    v = beta2 * v + (omb2 * g) * g
    d = np.sqrt(v) * rsb2_f + eps
    p = p - step_f * (m / d)
    return p, m, v


def step(state: OracleState, grads: Sequence[Sequence[np.ndarray]], cfg: AdamConfig) -> StepInfo:
    """One replicated-DP step.  grads[r][t]: rank r's gradient of tensor t."""
    n = len(grads)
    n_t = len(state.p32)
    S_used = state.S
    G = [reduce_grads([grads[r][t] for r in range(n)], cfg) for t in range(n_t)]
    overflow = any((~np.isfinite(g)).any() for g in G)                 # 4.
    if overflow:                                                       # 5.
        update_loss_scale(state, cfg, True)
        return StepInfo(t=state.t, overflow=True, loss_scale=S_used, grad_norm=float("nan"), clip=1.0)

    inv_f = f32(1.0 / (float(n) * S_used * float(f32(cfg.grad_prescale))))   # 6.
    U = [g * inv_f for g in G]
    # u^2 of an fp32 value is exact in fp64 (48 <= 53 significand bits); fsum is the
    # exactly rounded sum, so this is sqrt of the correctly rounded sum of squares.
    sq = math.fsum(np.concatenate([(u.astype(np.float64) ** 2) for u in U]).tolist()) if U else 0.0
    norm = math.sqrt(sq)
    clip_f = f32(1.0)
    if cfg.max_grad_norm > 0 and norm > float(f32(cfg.max_grad_norm)):
        clip_f = f32(float(f32(cfg.max_grad_norm)) / (norm + 1e-6))

    state.t += 1                                                       # 7.
    state.b1t *= float(f32(cfg.beta1))
    state.b2t *= float(f32(cfg.beta2))
    step_f = f32(float(f32(cfg.lr)) / (1.0 - state.b1t))
    rsb2_f = f32(1.0 / math.sqrt(1.0 - state.b2t))

    for t in range(n_t):                                               # 8.
        p, m, v = adam_tensor(state.p32[t], state.m[t], state.v[t], U[t], clip_f, step_f, rsb2_f, cfg)
        state.p32[t], state.m[t], state.v[t] = p, m, v
        with np.errstate(over="ignore"):
            state.p16[t] = numerics.to16(p, cfg.param_dtype)
    update_loss_scale(state, cfg, False)                               # 9.
    return StepInfo(t=state.t, overflow=False, loss_scale=S_used, grad_norm=norm, clip=float(clip_f))


def grads_from_torch(gs) -> List[np.ndarray]:
    """torch CPU 16-bit/fp32 tensors -> numpy (uint16 bit patterns for 16-bit)."""
    import torch
    out = []
    for g in gs:
        if g.dtype in (torch.float16, torch.bfloat16):
            out.append(g.view(torch.int16).numpy().view(np.uint16).copy())
        else:
            out.append(g.numpy().astype(np.float32).copy())
    return out
