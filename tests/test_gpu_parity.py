"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same
seeded inputs (config 1 and edge cases).  The LOCAL (N=1) and PEER (simulated
ranks, pull reduce-scatter in ascending rank + fused all-gather stores) paths are
held to BIT-EXACT fp32 master/m/v and 16-bit params (stronger than the north
star's 1e-6 / 1 ulp); overflow decisions, t and S must be equal; the grad norm
within 1e-12 relative (fp64 tree vs exact sum)."""
import numpy as np
import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes only under -m gpu
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run  # noqa: E402


def _cfg(dt, **kw):
    return OS.AdamConfig.defaults(dt, **kw)


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("stage", [0, 1, 2, 3])
def test_single_rank_all_stages(dt, stage):
    p = Pair(Run(synth.mlp_layout(), 1, stage, _cfg(dt), cap=1 << 17))
    for _ in range(5):
        oi, gi = p.step()
        p.compare_info(oi, gi)
    p.compare()
    p.destroy()


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("stage", [0, 1, 2, 3])
@pytest.mark.parametrize("mode", ["R16", "R32"])
def test_config1_sim4(dt, stage, mode):
    """BASELINE config 1: 1M-param MLP, N_d = 4 simulated ranks, 5 steps + an
    injected +inf at step 3 (0-based 2), against replicated-DP Adam."""
    if stage == 0 and mode == "R32":
        pytest.skip("stage 0 is R16 only")
    p = Pair(Run(synth.mlp_layout(), 4, stage, _cfg(dt, reduce_mode=mode), cap=1 << 17, inject=(2,)))
    for s in range(6):
        oi, gi = p.step()
        p.compare_info(oi, gi)
        assert oi.overflow == (s == 2)
    p.compare()
    c = p.engines[0].comm_counters()
    assert c.steps == 6
    p.destroy()


@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("stage", [1, 2, 3])
def test_ragged_layouts_unaligned(n, stage):
    """A = 1 and odd tensor sizes: exercises the scalar (unaligned) paths of every
    kernel, zero-size tensors, tiny buckets and N not a power of two."""
    ts = [synth.TensorSpec("a", 1001, 0), synth.TensorSpec("z", 0, 0), synth.TensorSpec("b", 7, 0),
          synth.TensorSpec("c", 333, 1, synth.ROLE_BIAS), synth.TensorSpec("d", 2049, 2),
          synth.TensorSpec("e", 1, 2, synth.ROLE_LNW), synth.TensorSpec("f", 4097, 3)]
    p = Pair(Run(ts, n, stage, _cfg("bf16", reduce_mode="R16"), align=1, cap=n * 37))
    for _ in range(3):
        oi, gi = p.step()
        p.compare_info(oi, gi)
    p.compare()
    p.destroy()


def test_clipping_active_and_prescale():
    """max_grad_norm = 1 (clipping active every step), weight decay, prescale 2 with fp32 grads."""
    ts = synth.mlp_layout((300, 200, 100))
    cfg = _cfg("fp16", max_grad_norm=1e-3, weight_decay=0.01, grad_dtype="fp32", grad_prescale=2.0)
    p = Pair(Run(ts, 4, 2, cfg, cap=1 << 14))
    clipped = 0
    for _ in range(4):
        oi, gi = p.step()
        p.compare_info(oi, gi)
        clipped += oi.clip != 1.0
    assert clipped > 0
    p.compare()
    p.destroy()


def test_bucket_order_irrelevant():
    """Buckets may be reduced in any order (backward hooks): results identical."""
    ts = synth.mlp_layout((200, 150, 100))
    a = Pair(Run(ts, 4, 2, _cfg("bf16"), cap=1 << 12))
    b = Pair(Run(ts, 4, 2, _cfg("bf16"), cap=1 << 12))
    rng = np.random.default_rng(0)
    for _ in range(2):
        a.step()
        b.step(bucket_order=list(rng.permutation(len(b.lay.buckets))))
    for w in ("p32", "m", "v"):
        assert np.array_equal(a.gpu_tensors(w)[1], b.gpu_tensors(w)[1])
    b.compare()


def test_loss_scale_sequence_on_device(golden):
    g = golden("loss_scale_sequence.json")
    cfg = _cfg("fp16", loss_scale=g["S0"], scale_window=g["window"], min_loss_scale=g["min_scale"])
    p = Pair(Run(synth.mlp_layout((40, 30, 20)), 2, 1, cfg, cap=1 << 10,
                 inject=tuple(s - 1 for s in g["inject_steps"])))
    S_before, t_after = [], []
    for _ in range(10):
        oi, gi = p.step()
        p.compare_info(oi, gi)
        S_before.append(gi[0].loss_scale)
        t_after.append(gi[0].t)
    assert S_before == g["S_before"] and t_after == g["t_after"]
    st = p.engines[1].device_state()
    assert st.t == p.ost.t and st.loss_scale == p.ost.S and st.good_steps == p.ost.good
    assert st.b1t == p.ost.b1t and st.b2t == p.ost.b2t
    p.compare()


def test_stage3_gather_views_and_prefetch():
    ts = synth.mlp_layout((120, 80, 60, 40, 20))
    p = Pair(Run(ts, 4, 3, _cfg("bf16"), cap=1 << 12))
    e = p.engines[2]
    n_layers = max(t.layer for t in ts) + 1
    for _ in range(3):        # gathered copies must not survive a step (the shards change)
        p.step()
        # forward then backward, releasing after use
        for order in (range(n_layers), reversed(range(n_layers))):
            for L in order:
                views = e.gather_params(L)
                for t, v in views.items():
                    assert np.array_equal(v.cpu().view(torch.int16).numpy().view(np.uint16), p.ost.p16[t])
                e.release_params(L)
    torch.cuda.synchronize()
    c = e.comm_counters()
    assert c.all_gather > 0
    # pool exhaustion without releases is an error, not a hang
    from paper_1910_02054_b200 import ZeroError
    e.gather_params(0)
    e.gather_params(1)
    with pytest.raises(ZeroError, match="ESTATE"):
        e.gather_params(2)


def test_state_errors():
    from paper_1910_02054_b200 import ZeroError
    p = Pair(Run(synth.mlp_layout((50, 20)), 1, 1, _cfg("bf16"), cap=1 << 10))
    e = p.engines[0]
    with pytest.raises(ZeroError, match="ESTATE"):
        e.step()                                   # no bucket reduced yet
    g = [x.cuda() for x in p.grads(0, 0)]
    e.reduce_grads(0, g)
    with pytest.raises(ZeroError, match="ESTATE"):
        e.reduce_grads(0, g)                       # twice in one step
    with pytest.raises(ZeroError, match="ESTATE"):
        e.gather_params(0)                         # stage 1


def test_synth_gpu_fill_matches_host():
    import ctypes as C
    import os
    lib = C.CDLL(os.path.join(os.path.dirname(synth.__file__), "libzero_synth.so"))
    key = synth.stream_key(7, synth.KIND_GRAD, 3, 2)
    n = 1 << 20
    for dt, code, tdt in (("fp16", 0, torch.float16), ("bf16", 1, torch.bfloat16), ("fp32", 2, torch.float32)):
        out = torch.empty(n, dtype=tdt, device="cuda")
        rc = lib.synth_fill(C.c_void_p(out.data_ptr()), C.c_uint64(key), C.c_uint64(12345), C.c_uint64(n),
                            C.c_float(2.0 ** 9), code, 0, C.c_float(0), None)
        assert rc == 0
        host = torch.from_numpy(synth.uniform_pm1(key, 12345, n) * np.float32(2.0 ** 9)).to(tdt)
        assert torch.equal(out.cpu().view(torch.int16 if dt != "fp32" else torch.int32),
                           host.view(torch.int16 if dt != "fp32" else torch.int32))


def test_long_run_dynamic_loss_scale():
    """200 steps of config 1's MLP at N_d = 4 (fp16, dynamic scaling with a short
    window so the scale doubles and halves many times; an overflow is injected every
    37 steps): the device state machine and every state stay bit-exact."""
    inject = tuple(range(5, 200, 37))
    cfg = _cfg("fp16", scale_window=7, loss_scale=2.0 ** 12)
    p = Pair(Run(synth.mlp_layout((400, 300, 200)), 4, 2, cfg, cap=1 << 14, inject=inject))
    scales, overflows = set(), 0
    for s in range(200):
        oi, gi = p.step()
        p.compare_info(oi, gi)
        scales.add(gi[0].loss_scale)
        overflows += oi.overflow
        if s in inject:
            assert oi.overflow
    # the injected steps and the natural fp16 overflows once S grows are all skipped
    assert len(scales) >= 4 and overflows >= len(inject) and p.ost.t == 200 - overflows
    p.compare()
    p.destroy()
