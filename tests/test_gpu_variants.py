"""Kernel variants the default launch configuration does not select at test sizes, each
held to the same bit-exact parity against the oracle as the defaults (test_gpu_parity):

* the TMA-ring fused Adam (k_adam_tma_st, variant 21) -- the default for shards above
  ZERO_ADAM_SMALL elements (every benchmarked model), while the small test layouts run the
  register-staged kernel; forced here on small and ragged shards;
* the flatten without the batching of adjacent small buckets (ZERO_SMALL_BUCKET=0);
* the reduce-scatter with a last-CTA combine instead of per-CTA partials, the plain
  (not software-pipelined) pull with other loads-in-flight settings, 256-bit loads;
* the flatten's last-CTA combine (ZERO_FLAT_CTA_PARTIALS=0);
* a small model's whole step as one cooperative launch (ZERO_STEP_SMALL=1; N_d = 1).
The knobs are environment variables read when the arenas are bound."""
import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run  # noqa: E402

VARIANTS = {
    "adam_tma": {"ZERO_ADAM_VARIANT": "21"},
    "adam_tma_no_batch": {"ZERO_ADAM_VARIANT": "21", "ZERO_SMALL_BUCKET": "0"},
    "rs_grid_combine": {"ZERO_RS_CTA_PARTIALS": "0"},
    "rs_plain_u2": {"ZERO_RS_PIPE": "0", "ZERO_RS_CTAS": "2"},
    "rs_plain_u1_c6": {"ZERO_RS_PIPE": "0", "ZERO_RS_U": "1", "ZERO_RS_CTAS": "6"},
    "rs_w16": {"ZERO_RS_PIPE": "2"},
    "rs_w16_pipe": {"ZERO_RS_PIPE": "3", "ZERO_RS_CTAS": "2"},
    "rs_grid_cap": {"ZERO_RS_GRID": "5"},                         # a few CTAs, grid-stride (NVLink-bound sizing)
    "rs_grid_cap_per_rank": {"ZERO_RS_GRID": "3", "ZERO_RS_MULTI": "0"},
    "gather_grid_cap": {"ZERO_GATHER_GRID": "2"},                # stage-3 layer gathers on 2 CTAs per source
    "flat_grid_combine": {"ZERO_FLAT_CTA_PARTIALS": "0", "ZERO_SMALL_BUCKET": "0"},
    "step_small_fused": {"ZERO_STEP_SMALL": "1"},
}


def _run(monkeypatch, env, n, stage, dt, mode="R16", ts=None, align=64, cap=1 << 17, steps=4, inject=(2,)):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    ts = ts or synth.mlp_layout((700, 400, 300, 200))
    p = Pair(Run(ts, n, stage, OS.AdamConfig.defaults(dt, reduce_mode=mode), align=align, cap=cap, inject=inject))
    for s in range(steps):
        oi, gi = p.step()
        p.compare_info(oi, gi)
        assert oi.overflow == (s in inject)
    p.compare()
    p.destroy()


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("n,stage,dt,mode", [(1, 1, "bf16", "R16"), (1, 3, "fp16", "R16"), (4, 2, "fp16", "R16"),
                                             (4, 1, "bf16", "R32"), (2, 3, "bf16", "R16"), (8, 2, "fp16", "R32"),
                                             (4, 0, "bf16", "R16")])
def test_variant_matches_oracle(monkeypatch, variant, n, stage, dt, mode):
    _run(monkeypatch, VARIANTS[variant], n, stage, dt, mode)


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("n", [1, 3, 4])
def test_variant_ragged(monkeypatch, variant, n):
    """A = 1, odd sizes, zero-size tensors, tiny buckets: the unaligned paths of each variant."""
    ts = [synth.TensorSpec("a", 1001, 0), synth.TensorSpec("z", 0, 0), synth.TensorSpec("b", 7, 0),
          synth.TensorSpec("c", 333, 1, synth.ROLE_BIAS), synth.TensorSpec("d", 2049, 2),
          synth.TensorSpec("e", 1, 2, synth.ROLE_LNW), synth.TensorSpec("f", 4097, 3)]
    _run(monkeypatch, VARIANTS[variant], n, 2, "bf16", ts=ts, align=1, cap=n * 37, steps=3, inject=())


def test_small_bucket_batching_permuted_order(monkeypatch):
    """N_d = 1: batched runs of adjacent small buckets in a non-monotone order (runs break and
    re-form; stale per-slot partials must not leak into the norm), bit-exact every step."""
    monkeypatch.setenv("ZERO_SMALL_BUCKET", str(1 << 20))
    ts = synth.mlp_layout((300, 200, 100, 50, 40))
    p = Pair(Run(ts, 1, 2, OS.AdamConfig.defaults("bf16", max_grad_norm=1e-2), cap=1 << 12, inject=(1,)))
    nb = len(p.lay.buckets)
    orders = [list(reversed(range(nb))), list(range(nb)), [k for k in range(nb) if k % 2] + [k for k in range(nb) if not k % 2],
              list(reversed(range(nb)))]
    for s, order in enumerate(orders):
        oi, gi = p.step(bucket_order=order)
        p.compare_info(oi, gi)
    p.compare()
    p.destroy()


@pytest.mark.parametrize("n", [1, 4])
def test_step_record_pinned_and_pageable(n):
    """zero_step's host_out: pinned (UVA-mapped) memory is written by the decision kernel, any
    other host memory by a D2H copy at the end of the step; both equal ZERO_Q_STEP's record."""
    import ctypes as C
    from paper_1910_02054_b200.zero import CStepInfo, _check, lib
    ts = synth.mlp_layout((300, 200, 100))
    p = Pair(Run(ts, n, 2, OS.AdamConfig.defaults("fp16", max_grad_norm=1e-2), cap=1 << 13, inject=(1,)))
    for s in range(3):
        host = [p.grads(r, s) for r in range(n)]
        dev = [[g.cuda() for g in h] for h in host]
        for k in reversed(range(len(p.lay.buckets))):
            for r in range(n):
                p.engines[r].reduce_grads(k, dev[r])
        pageable = [CStepInfo() for _ in range(n)]
        for r in range(n):
            e = p.engines[r]
            ptr = C.pointer(pageable[r]) if r % 2 == 0 else e._info_ptr
            _check(lib.zero_step(e._ctx, ptr), e._ctx)
        torch.cuda.synchronize()
        OS.step(p.ost, [OS.grads_from_torch(h) for h in host], p.run.cfg)
        for r in range(n):
            e = p.engines[r]
            ref = e.step_info()
            got = pageable[r] if r % 2 == 0 else C.cast(e._info_ptr, C.POINTER(CStepInfo)).contents
            assert (got.t, got.overflow, got.loss_scale, got.clip, got.grad_norm) == \
                   (ref.t, ref.overflow, ref.loss_scale, ref.clip, ref.grad_norm), (s, r)
            assert got.overflow == (s == 1)
    p.compare()
    p.destroy()
