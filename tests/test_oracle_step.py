"""Pins for oracle/step.py (readings c-1..c-5) against things other than itself:
SPEC's worked example, torch.optim.Adam, an fp64 textbook Adam, exact rational
sums, closed forms for the norm, torch's clip_grad_norm_, the hand-traced
loss-scale sequence and the replicated-gradient invariant."""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import synth
from oracle import layout as L
from oracle import numerics as nx
from oracle import step as S

f32 = np.float32


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def _g16(vals, dt):
    return nx.to16(np.asarray(vals, np.float32), dt)


def test_spec_adam_example(golden):
    g = golden("adam_spec_example.json")
    cfg = S.AdamConfig(lr=g["lr"], beta1=g["beta1"], beta2=g["beta2"], eps=g["eps"],
                       param_dtype="fp16", grad_dtype="fp16")
    st = S.init_state([np.array([g["theta"]], np.float32)], cfg)
    info = S.step(st, [[_g16([g["g"]], "fp16")]], cfg)
    assert info.t == 1 and not info.overflow
    want = {k: int(v, 16) for k, v in g["expect_bits"].items()}
    assert int(_bits(st.p32[0])[0]) == want["theta"]
    assert int(_bits(st.m[0])[0]) == want["m"]
    assert int(_bits(st.v[0])[0]) == want["v"]
    # S:280 "theta' ~ 0.9 (exactly 1 - 0.1/(1+1e-8))"
    assert abs(float(st.p32[0][0]) - (1 - 0.1 / (1 + 1e-8))) < 1e-7


def test_zero_grad_keeps_master():
    # g = 0 on a fresh shard -> master unchanged (mhat = 0)
    cfg = S.AdamConfig.defaults("bf16")
    m0 = synth.master_values(synth.mlp_layout((7, 5, 3)), 3)
    st = S.init_state(m0, cfg)
    S.step(st, [[np.zeros(a.size, np.uint16) for a in m0]], cfg)
    for a, b in zip(st.p32, m0):
        assert np.array_equal(_bits(a), _bits(b))


def _run(tensors, cfg, n, steps, seed=1, replicate=False, inject=None):
    st = S.init_state(synth.master_values(tensors, seed), cfg)
    infos = []
    for s in range(steps):
        grads = []
        for r in range(n):
            rr = 0 if replicate else r
            gs = synth.grads16(tensors, seed, rr, s, cfg.grad_dtype, scale=st.S if cfg.param_dtype == "fp16" else 1.0)
            grads.append(S.grads_from_torch(gs))
        if inject and s in inject:
            grads[min(1, n - 1)][0][0] = 0x7C00 if cfg.param_dtype == "fp16" else 0x7F80
        infos.append(S.step(st, grads, cfg))
    return st, infos


@pytest.mark.parametrize("dt", ["fp16", "bf16"])
@pytest.mark.parametrize("mode", ["R16", "R32"])
def test_replicated_gradients_equal_single_rank(dt, mode):
    """c-9: g_r = g for all r gives the N = 1 result bitwise (N a power of two)."""
    ts = synth.mlp_layout((61, 40, 30, 9))
    cfg = S.AdamConfig.defaults(dt, reduce_mode=mode)
    ref, ref_i = _run(ts, cfg, 1, 3)
    for n in (2, 4, 8):
        st, inf = _run(ts, cfg, n, 3, replicate=True)
        for a, b in zip(st.p32 + st.m + st.v, ref.p32 + ref.m + ref.v):
            assert np.array_equal(_bits(a), _bits(b))
        for a, b in zip(st.p16, ref.p16):
            assert np.array_equal(a, b)
        assert [i.grad_norm for i in inf] == [i.grad_norm for i in ref_i]


def test_spec_reduce_example():
    # N=2, rank0 = [1,2], rank1 = [3,4] -> sums [4, 6]
    cfg = S.AdamConfig.defaults("fp16")
    G = S.reduce_grads([_g16([1, 2], "fp16"), _g16([3, 4], "fp16")], cfg)
    assert G.tolist() == [4.0, 6.0]


@pytest.mark.parametrize("dt", ["fp16", "bf16"])
def test_ordered_sum_against_rationals(dt):
    """c-2: fp32 accumulation in ascending rank, then one rounding (R16) --
    compared with a left fold over exact rationals rounded to fp32 at each step."""
    rng = np.random.default_rng(5)
    cfg16 = S.AdamConfig.defaults(dt, reduce_mode="R16")
    cfg32 = S.AdamConfig.defaults(dt, reduce_mode="R32")
    for n in (2, 3, 5, 8):
        vals = rng.uniform(-1, 1, (n, 2000)) * np.exp2(rng.integers(-24 if dt == "fp16" else -60, 15, (n, 2000)))
        g = [_g16(vals[r], dt) for r in range(n)]
        g[0][:4] = _g16([32768.0, 2.0 ** -24, 1.0, -0.0], dt)      # cancellation / tiny terms
        g[1 % n][:4] = _g16([2.0 ** -24, -32768.0, -1.0, 0.0], dt)
        G32 = S.reduce_grads(g, cfg32)
        G16 = S.reduce_grads(g, cfg16)
        for i in range(2000):
            acc = None
            for r in range(n):
                x = Fraction(float(nx.widen(g[r][i:i + 1], dt)[0]))
                acc = x if acc is None else Fraction(float(np.float32(float(acc + x))))
            # partial sums of 16-bit values span < 2^53, so float(acc + x) is exact
            assert float(G32[i]) == float(np.float32(float(acc)))
            assert float(G16[i]) == float(nx.widen(nx.to16(np.array([float(acc)], np.float32), dt), dt)[0])


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_against_torch_adam(dt):
    """torch.optim.Adam (foreach=False, fp32 CPU) is an independent implementation;
    its op order differs (lerp, divide by sqrt(bc2)) so agreement is to a few ulp.
    fp16 runs at S = 2^16, so a missing unscale shows up in m and v."""
    ts = synth.mlp_layout((33, 20, 7))
    cfg = S.AdamConfig.defaults(dt, lr=1e-3)
    st = S.init_state(synth.master_values(ts, 2), cfg)
    params = [torch.nn.Parameter(torch.from_numpy(a.copy())) for a in st.p32]
    opt = torch.optim.Adam(params, lr=float(f32(cfg.lr)), betas=(float(f32(cfg.beta1)), float(f32(cfg.beta2))),
                           eps=float(f32(cfg.eps)), foreach=False)
    for s in range(5):
        S_cur = st.S
        gs = S.grads_from_torch(synth.grads16(ts, 2, 0, s, dt, scale=S_cur))
        S.step(st, [gs], cfg)
        for p, g in zip(params, gs):
            p.grad = torch.from_numpy(nx.widen(g, dt) / np.float32(S_cur))
        opt.step()
    for p, a, t in zip(params, st.p32, range(len(params))):
        ref = p.detach().numpy()
        np.testing.assert_allclose(a, ref, rtol=2e-6, atol=1e-9)
        m_ref = opt.state[p]["exp_avg"].numpy()
        v_ref = opt.state[p]["exp_avg_sq"].numpy()
        # m can cancel (0.9 m + 0.1 g with alternating signs): absolute floor at
        # 1e-6 of the tensor's scale; a missing 1/S would be off by 2^16
        np.testing.assert_allclose(st.m[t], m_ref, rtol=1e-5, atol=1e-6 * float(np.abs(m_ref).max()))
        np.testing.assert_allclose(st.v[t], v_ref, rtol=1e-5, atol=1e-6 * float(np.abs(v_ref).max()))


def test_against_fp64_textbook_adam():
    """Kingma & Ba in fp64: theta -= lr * mhat / (sqrt(vhat) + eps)."""
    rng = np.random.default_rng(9)
    cfg = S.AdamConfig.defaults("bf16", lr=1e-2)
    p0 = rng.uniform(-1, 1, 5000).astype(np.float32)
    st = S.init_state([p0], cfg)
    p, m, v = p0.astype(np.float64), np.zeros(5000), np.zeros(5000)
    b1, b2 = float(f32(0.9)), float(f32(0.999))
    for t in range(1, 8):
        g16 = _g16(rng.uniform(-1, 1, 5000) * 2.0 ** rng.integers(-8, 0, 5000), "bf16")
        S.step(st, [[g16]], cfg)
        g = nx.widen(g16, "bf16").astype(np.float64)
        m = b1 * m + (1 - b1) * g
        v = b2 * v + (1 - b2) * g * g
        p = p - float(f32(1e-2)) * (m / (1 - b1 ** t)) / (np.sqrt(v / (1 - b2 ** t)) + float(f32(1e-8)))
    np.testing.assert_allclose(st.p32[0], p, rtol=1e-6, atol=1e-8)


def test_shards_equal_full_range():
    """two shards updated independently == the full range, bitwise; and
    the per-bucket partition of reading c-7 (any stage, any N) likewise."""
    ts = synth.mlp_layout((50, 40, 13))
    cfg = S.AdamConfig.defaults("fp16")
    full, _ = _run(ts, cfg, 4, 3)
    lay = L.make_layout([t.numel for t in ts], [t.layer for t in ts], 4, 8, 512)
    # replay the same steps shard by shard on flat arrays
    st = S.init_state(synth.master_values(ts, 1), cfg)
    flat = lambda arrs, dt=np.float32: _flatten(lay, arrs, dt)
    P32, M, V = flat(st.p32), flat(st.m), flat(st.v)
    for s in range(3):
        grads = [S.grads_from_torch(synth.grads16(ts, 1, r, s, "fp16", scale=st.S)) for r in range(4)]
        G = np.concatenate([S.reduce_grads([_flatten(lay, grads[r], np.uint16)[lo:hi] for r in range(4)], cfg)
                            for r in range(4) for (lo, hi) in [lay.owned_range(k, r) for k in range(len(lay.buckets))]])
        order = np.concatenate([np.arange(*lay.owned_range(k, r)) for r in range(4) for k in range(len(lay.buckets))])
        Gf = np.empty_like(G)
        Gf[order] = G
        inv_f = f32(1.0 / (4 * st.S))
        U = Gf * inv_f
        st.t += 1
        st.b1t *= float(f32(cfg.beta1))
        st.b2t *= float(f32(cfg.beta2))
        step_f = f32(float(f32(cfg.lr)) / (1.0 - st.b1t))
        rsb2_f = f32(1.0 / math.sqrt(1.0 - st.b2t))
        for r in range(4):
            for k in range(len(lay.buckets)):
                lo, hi = lay.owned_range(k, r)
                P32[lo:hi], M[lo:hi], V[lo:hi] = S.adam_tensor(P32[lo:hi], M[lo:hi], V[lo:hi], U[lo:hi],
                                                               f32(1), step_f, rsb2_f, cfg)
        S.update_loss_scale(st, cfg, False)
    assert np.array_equal(_bits(P32), _bits(flat(full.p32)))
    assert np.array_equal(_bits(M), _bits(flat(full.m)))
    assert np.array_equal(_bits(V), _bits(flat(full.v)))


def _flatten(lay, arrs, dt):
    out = np.zeros(lay.psi_padded, dt)
    for b in lay.buckets:
        for p in b.pieces:
            out[b.base + p.bucket_off: b.base + p.bucket_off + p.count] = \
                np.asarray(arrs[p.tensor]).reshape(-1)[p.tensor_off:p.tensor_off + p.count]
    return out


def test_loss_scale_sequence(golden):
    g = golden("loss_scale_sequence.json")
    cfg = S.AdamConfig.defaults("fp16", loss_scale=g["S0"], scale_window=g["window"],
                                min_loss_scale=g["min_scale"])
    ts = synth.mlp_layout((9, 4, 3))
    st = S.init_state(synth.master_values(ts, 1), cfg)
    S_before, t_after = [], []
    for s in range(1, 11):
        grads = [S.grads_from_torch(synth.grads16(ts, 1, 0, s, "fp16", scale=1.0))]
        if s in g["inject_steps"]:
            before = [a.copy() for a in st.p32]
            grads[0][2][3] = 0x7C00
        S_before.append(st.S)
        info = S.step(st, grads, cfg)
        t_after.append(st.t)
        assert info.overflow == (s in g["inject_steps"])
        if info.overflow:
            assert all(np.array_equal(_bits(a), _bits(b)) for a, b in zip(st.p32, before))
    assert S_before == g["S_before"] and t_after == g["t_after"]


def test_overflow_from_r16_rounding():
    """c-4: in R16 the reduced sum itself may round to inf (fp16: |sum| >= 65520)."""
    cfg = S.AdamConfig.defaults("fp16", dynamic_loss_scale=False, loss_scale=1.0)
    st = S.init_state([np.zeros(2, np.float32)], cfg)
    g = _g16([40000.0, 1.0], "fp16")
    info = S.step(st, [[g], [g]], cfg)
    assert info.overflow
    cfg32 = S.AdamConfig.defaults("fp16", dynamic_loss_scale=False, loss_scale=1.0, reduce_mode="R32")
    st = S.init_state([np.zeros(2, np.float32)], cfg32)
    assert not S.step(st, [[g], [g]], cfg32).overflow


def test_norm_closed_form_and_library():
    # u = c (power of two), Psi' = 4^10 -> norm = |c| * 2^10 exactly
    cfg = S.AdamConfig.defaults("bf16")
    n = 4 ** 10
    st = S.init_state([np.zeros(n // 4, np.float32)] * 4, cfg)
    c = 2.0 ** -5
    info = S.step(st, [[_g16(np.full(n // 4, -c), "bf16") for _ in range(4)]], cfg)
    assert info.grad_norm == c * 2 ** 10
    # random: against torch.linalg.vector_norm in fp64
    rng = np.random.default_rng(3)
    gs = [_g16(rng.normal(size=k) * 0.01, "bf16") for k in (1000, 37, 4096)]
    st = S.init_state([np.zeros(g.size, np.float32) for g in gs], cfg)
    info = S.step(st, [gs], cfg)
    ref = torch.linalg.vector_norm(torch.cat([torch.from_numpy(nx.widen(g, "bf16").astype(np.float64)) for g in gs]))
    assert abs(info.grad_norm - float(ref)) <= 1e-12 * float(ref)


def test_clip_against_torch():
    rng = np.random.default_rng(4)
    cfg = S.AdamConfig.defaults("bf16", max_grad_norm=1.0)
    gs = [_g16(rng.normal(size=k) * 0.2, "bf16") for k in (300, 50)]
    st = S.init_state([np.zeros(g.size, np.float32) for g in gs], cfg)
    info = S.step(st, [gs], cfg)
    ps = [torch.nn.Parameter(torch.zeros(g.size, dtype=torch.float64)) for g in gs]
    for p, g in zip(ps, gs):
        p.grad = torch.from_numpy(nx.widen(g, "bf16").astype(np.float64))
    total = torch.nn.utils.clip_grad_norm_(ps, 1.0)
    assert info.grad_norm > 1.0 and abs(info.grad_norm - float(total)) <= 1e-12 * float(total)
    assert info.clip == float(np.float32(1.0 / (float(total) + 1e-6)))
    # the clipped gradient feeds Adam: compare with torch Adam on u * clip
    params = [torch.nn.Parameter(torch.zeros(g.size)) for g in gs]
    opt = torch.optim.Adam(params, lr=1e-3, foreach=False)
    for p, g in zip(params, gs):
        p.grad = torch.from_numpy(nx.widen(g, "bf16") * np.float32(info.clip))
    opt.step()
    for p, a in zip(params, st.p32):
        np.testing.assert_allclose(a, p.detach().numpy(), rtol=2e-6, atol=1e-10)


def test_prescale_is_undone_exactly():
    """c-8 #24: the flatten multiplies by sigma (a power of two) and the unscale divides
    by N*S*sigma -- for fp32 gradients whose scaled values stay in range the result is
    the same, bitwise, for sigma in {1, 2, 4} (a dropped or doubled sigma fails)."""
    ts = synth.mlp_layout((40, 30, 20))
    ref = None
    for sigma in (1.0, 2.0, 4.0):
        cfg = S.AdamConfig.defaults("bf16", grad_dtype="fp32", grad_prescale=sigma)
        st = S.init_state(synth.master_values(ts, 5), cfg)
        for s in range(3):
            gs = [S.grads_from_torch(synth.grads16(ts, 5, r, s, "fp32")) for r in range(2)]
            S.step(st, gs, cfg)
        cur = [a.view(np.uint32).copy() for a in st.p32 + st.m + st.v]
        if ref is None:
            ref = cur
        else:
            assert all(np.array_equal(a, b) for a, b in zip(cur, ref)), sigma


def test_weight_decay_against_torch_adamw():
    """Decoupled weight decay (reading c-3): p -= lr*wd*p before the Adam update, as
    torch.optim.AdamW (an independent implementation; few-ulp agreement)."""
    ts = synth.mlp_layout((33, 20, 7))
    cfg = S.AdamConfig.defaults("bf16", lr=1e-3, weight_decay=0.1)
    st = S.init_state(synth.master_values(ts, 2), cfg)
    params = [torch.nn.Parameter(torch.from_numpy(a.copy())) for a in st.p32]
    opt = torch.optim.AdamW(params, lr=float(f32(cfg.lr)), betas=(float(f32(cfg.beta1)), float(f32(cfg.beta2))),
                            eps=float(f32(cfg.eps)), weight_decay=float(f32(cfg.weight_decay)), foreach=False)
    for s in range(5):
        gs = S.grads_from_torch(synth.grads16(ts, 2, 0, s, "bf16"))
        S.step(st, [gs], cfg)
        for p, g in zip(params, gs):
            p.grad = torch.from_numpy(nx.widen(g, "bf16").copy())
        opt.step()
    for p, a in zip(params, st.p32):
        np.testing.assert_allclose(a, p.detach().numpy(), rtol=2e-6, atol=1e-9)
    # and decay is really applied: without it the masters differ by far more than that
    st0 = S.init_state(synth.master_values(ts, 2), S.AdamConfig.defaults("bf16", lr=1e-3))
    for s in range(5):
        S.step(st0, [S.grads_from_torch(synth.grads16(ts, 2, 0, s, "bf16"))], S.AdamConfig.defaults("bf16", lr=1e-3))
    assert max(float(np.abs(a - b).max()) for a, b in zip(st.p32, st0.p32)) > 1e-6
