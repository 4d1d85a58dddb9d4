"""Degenerate inputs of the step on the GPU, through the C ABI, against the oracle:
all-zero gradients (g = 0 leaves the first step's parameters unchanged), NaN
(not only inf) as an overflow, negative zeros, one-element layouts where most ranks own
only padding, and maximum-magnitude finite 16-bit gradients."""
import numpy as np
import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run, bits32  # noqa: E402


def _const_grads(p, value, dt):
    tdt = torch.bfloat16 if dt == "bf16" else torch.float16
    return lambda r, s: [torch.full((n,), value, dtype=tdt) for n in p.numels]


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("n,stage", [(1, 1), (4, 2), (4, 3)])
def test_zero_gradients_leave_parameters(dt, n, stage):
    ts = synth.mlp_layout((100, 60, 30))
    cfg = OS.AdamConfig.defaults(dt, max_grad_norm=1.0)
    p = Pair(Run(ts, n, stage, cfg, cap=1 << 12))
    p.grads = _const_grads(p, 0.0, dt)
    p32_before = [a.copy() for a in p.ost.p32]
    oinfo, ginfos = p.step()
    p.compare_info(oinfo, ginfos)
    assert all(g.grad_norm == 0.0 and g.clip == 1.0 and not g.overflow for g in ginfos)
    p.compare()
    for a, b in zip(p.ost.p32, p32_before):   # the oracle agrees with S:279 at t = 1
        assert np.array_equal(bits32(a), bits32(b))
    p.destroy()


@pytest.mark.parametrize("bad", [float("nan"), float("-inf")])
def test_nan_and_negative_inf_are_overflow(bad):
    ts = synth.mlp_layout((100, 60, 30))
    cfg = OS.AdamConfig.defaults("fp16")
    p = Pair(Run(ts, 4, 2, cfg, cap=1 << 12))
    base = p.grads

    def grads(r, s):
        g = base(r, s)
        if s == 1 and r == 3:
            g[2] = g[2].clone()
            g[2][-1] = bad
        return g
    p.grads = grads
    for _s in range(3):
        oinfo, ginfos = p.step()
        p.compare_info(oinfo, ginfos)
    assert p.infos[1][0].overflow and all(g.overflow for g in p.infos[1][1])
    p.compare()
    p.destroy()


def test_negative_zero_gradients():
    ts = synth.mlp_layout((64, 32))
    cfg = OS.AdamConfig.defaults("bf16")
    p = Pair(Run(ts, 2, 1, cfg, cap=1 << 12))
    p.grads = _const_grads(p, -0.0, "bf16")
    oinfo, ginfos = p.step()
    p.compare_info(oinfo, ginfos)
    assert not oinfo.overflow
    p.compare()
    p.destroy()


@pytest.mark.parametrize("n,stage", [(8, 1), (8, 2), (8, 3), (3, 2)])
def test_one_element_model(n, stage):
    """Psi = 1: the bucket is padded to N*A; all ranks but one own only padding."""
    ts = [synth.TensorSpec("w", 1, 0)]
    cfg = OS.AdamConfig.defaults("bf16")
    p = Pair(Run(ts, n, stage, cfg, cap=0))
    for _s in range(3):
        oinfo, ginfos = p.step()
        p.compare_info(oinfo, ginfos)
    p.compare()
    p.destroy()


def test_max_finite_fp16_gradients():
    """|g| = 65504 on every rank: the fp32 sum is finite, the R16 rounding overflows to
    inf (reading c-2), so the step is skipped on every rank, as in the oracle."""
    ts = synth.mlp_layout((64, 32))
    cfg = OS.AdamConfig.defaults("fp16", reduce_mode="R16")
    p = Pair(Run(ts, 2, 2, cfg, cap=1 << 12))
    p.grads = _const_grads(p, 65504.0, "fp16")
    oinfo, ginfos = p.step()
    p.compare_info(oinfo, ginfos)
    assert oinfo.overflow
    p.compare()
    cfg32 = OS.AdamConfig.defaults("fp16", reduce_mode="R32")
    q = Pair(Run(ts, 2, 2, cfg32, cap=1 << 12))
    q.grads = _const_grads(q, 65504.0, "fp16")
    oinfo, ginfos = q.step()                      # R32 keeps the finite fp32 sum
    q.compare_info(oinfo, ginfos)
    assert not oinfo.overflow
    q.compare()
    p.destroy()
    q.destroy()


@pytest.mark.parametrize("n", [1, 3, 4])
@pytest.mark.parametrize("S", [1000.0, 0.5, 3.0])
@pytest.mark.parametrize("mode", ["R16", "R32"])
def test_general_epilogue_path(n, S, mode):
    """inv = 1/(N*S*sigma) not a power of two (S = 1000, 3; N = 3) or above 1 (S = 0.5):
    the flatten / reduce-scatter epilogues take the general path (u = fp32(G*inv),
    per-element flag) instead of the power-of-two one; bit-exact vs the oracle, with
    clipping active so the norm matters."""
    if n == 1 and mode == "R32":
        pytest.skip("R32 is a reduce-scatter storage mode (N > 1)")
    ts = synth.mlp_layout((120, 70, 30))
    cfg = OS.AdamConfig.defaults("fp16", dynamic_loss_scale=False, loss_scale=S, max_grad_norm=0.05,
                                 reduce_mode=mode)
    p = Pair(Run(ts, n, 2, cfg, cap=1 << 12))
    for _s in range(3):
        oinfo, ginfos = p.step()
        p.compare_info(oinfo, ginfos)
        assert not oinfo.overflow
    p.compare()
    p.destroy()
