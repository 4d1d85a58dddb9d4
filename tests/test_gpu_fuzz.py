"""Randomised GPU parity: 60 seeded random configurations (tensor lists with zero /
odd / tiny sizes, N_d in 1..8, A in {1,8,64}, random C_B, stages 0-3, fp16/bf16,
R16/R32, fp32 gradients, prescale, clipping, weight decay, pool and prefetch sizes),
each run for 3 steps through the C ABI against the oracle, bit-exact."""
import random

import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run  # noqa: E402


def _case(seed):
    rnd = random.Random(seed)
    nt = rnd.randint(1, 9)
    ts, L = [], 0
    for i in range(nt):
        L += rnd.random() < 0.4
        n = rnd.choice([0, 1, 3, 7, 64, 65, 255, 1000]) if rnd.random() < 0.4 else rnd.randint(1, 6000)
        ts.append(synth.TensorSpec(f"t{i}", n, L, rnd.choice([synth.ROLE_WEIGHT, synth.ROLE_BIAS, synth.ROLE_LNW])))
    if sum(t.numel for t in ts) == 0:
        ts[0] = synth.TensorSpec("t0", 17, ts[0].layer)
    n = rnd.choice([1, 1, 2, 3, 4, 5, 8])
    a = rnd.choice([1, 8, 64])
    q = n * a
    cap = rnd.choice([q, 3 * q, rnd.randint(q, 40 * q), 0])
    stage = rnd.randint(0, 3)
    dt = rnd.choice(["fp16", "bf16"])
    mode = "R16" if stage == 0 else rnd.choice(["R16", "R32"])
    kw = dict(reduce_mode=mode)
    if rnd.random() < 0.3:
        kw["grad_dtype"] = "fp32"
    if rnd.random() < 0.3:
        kw["grad_prescale"] = 2.0
    if rnd.random() < 0.3:
        kw["max_grad_norm"] = 1e-3
    if rnd.random() < 0.3:
        kw["weight_decay"] = 0.1
    cfg = OS.AdamConfig.defaults(dt, **kw)
    return ts, n, a, cap, stage, cfg, rnd.choice([1, 2, 3]), rnd.choice([1, 2])


@pytest.mark.parametrize("seed", range(60))
def test_random_configuration(seed):
    ts, n, a, cap, stage, cfg, pool, depth = _case(seed)
    run = Run(ts, n, stage, cfg, align=a, cap=cap, inject=(1,) if seed % 5 == 0 else (), pool=pool, prefetch=depth)
    p = Pair(run)
    for _ in range(3):
        oi, gi = p.step()
        p.compare_info(oi, gi)
    p.compare()
    if stage == 3:
        e = p.engines[-1]
        for L in sorted({t.layer for t in ts if t.numel > 0}):
            views = e.gather_params(L)
            for t, v in views.items():
                assert torch.equal(v.cpu().view(torch.int16),
                                   torch.from_numpy(p.ost.p16[t].view("int16")))
            e.release_params(L)
    p.destroy()


KNOBS = {
    "ZERO_RS_PIPE": ["0", "1", "2", "3"],
    "ZERO_RS_CTA_PARTIALS": ["0", "1"],
    "ZERO_RS_MULTI": ["0", "1"],
    "ZERO_RS_CTAS": ["2", "4", "6"],
    "ZERO_SMALL_BUCKET": ["0", "64", str(1 << 20)],
    "ZERO_ADAM_VARIANT": [None, "0", "1", "21"],
    "ZERO_FLAT_STREAMS": ["1", "2", "3"],
    "ZERO_FLAT_CTA_PARTIALS": ["0", "1"],
    "ZERO_STEP_SMALL": ["0", "1"],
}


@pytest.mark.parametrize("seed", range(1000, 1060))
def test_random_configuration_and_launch_knobs(monkeypatch, seed):
    """As above, with every launch knob drawn at random too (each one selects another kernel
    body, grid or batching path) and the buckets reduced in a random order each step."""
    rnd = random.Random(seed * 7 + 1)
    for k, choices in KNOBS.items():
        v = rnd.choice(choices)
        if v is None:
            monkeypatch.delenv(k, raising=False)
        else:
            monkeypatch.setenv(k, v)
    ts, n, a, cap, stage, cfg, pool, depth = _case(seed)
    run = Run(ts, n, stage, cfg, align=a, cap=cap, inject=(1,) if seed % 4 == 0 else (), pool=pool, prefetch=depth)
    p = Pair(run)
    nb = len(p.lay.buckets)
    for s in range(3):
        order = list(range(nb))
        rnd.shuffle(order)
        oi, gi = p.step(bucket_order=order)
        p.compare_info(oi, gi)
    p.compare()
    p.destroy()
