"""Parity at BASELINE config 2's full size (GPT-2 1.5B layout, Psi = 1,557,611,200,
stage 1, N_d = 1, bf16) and at config 3's (the paper's Fig. 1 7.5B model, Psi = 7.5e9,
stage 2, N_d = 1: 135 GB of arenas) in the launch configurations bench.py times: the
contract line (bf16) and its fp16 key (dynamic loss scaling, gradients at S = 2^16).

The oracle cannot hold 1.5B-element replicas, so (③) we compare on SAMPLED outputs
the oracle computes one by one: with clipping off, Adam is elementwise, so the
oracle's update of a sampled element needs only that element's master, gradients
and the step scalars.  The global norm is checked against torch's fp64
vector_norm of the same gradients (a library routine), the overflow decision and
t exactly, and padding / unsampled structure via properties."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import numerics as nx
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)


@pytest.mark.parametrize("config,stage,dt", [("gpt2_1.5b", 1, "bf16"), ("gpt_7.5b", 2, "bf16"), ("gpt_7.5b", 2, "fp16")])
def test_full_size_sampled(config, stage, dt):
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine
    torch.cuda.empty_cache()
    ts = synth.CONFIGS[config]()
    dev = torch.device("cuda", 0)
    cfg = OS.AdamConfig.defaults(dt)
    S = float(cfg.loss_scale)                       # fp16: 2^16 (dynamic, no overflow here); bf16: 1
    eng = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], 1, 0, stage, ZeroConfig.defaults(dt), "local",
                     align=64, bucket_cap=1 << 26, device=dev)
    for i in range(len(ts)):                       # chunked master load (NULL = skip)
        masters = synth.gpu_masters(ts, 1, dev, only={i})
        eng.load_master(masters)
    torch.cuda.synchronize()
    del masters
    offs = synth.tensor_offsets(ts)
    psi = synth.psi(ts)
    rng = np.random.default_rng(0)
    samp = np.unique(np.concatenate([rng.integers(0, psi, 200_000), [0, psi - 1],
                                     np.array(offs[1:]) - 1, np.array(offs)]))
    tid = np.searchsorted(np.array(offs), samp, side="right") - 1
    # oracle state of the sampled elements
    roles = np.array([t.role for t in ts])[tid]
    x = synth.uniform_at(synth.stream_key(1, synth.KIND_MASTER), samp) * np.float32(2.0 ** -6)
    p = np.where(roles == synth.ROLE_LNW, np.float32(1), np.where(roles == synth.ROLE_BIAS, np.float32(0), x))
    p = p.astype(np.float32)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    b1t = b2t = 1.0
    nb = eng.info.n_buckets
    for step in range(2):
        tdt = torch.bfloat16 if dt == "bf16" else torch.float16
        buf, grads = synth.gpu_grads_flat(ts, 1, 0, step, tdt, dev, scale=S)
        for k in reversed(range(nb)):
            eng.reduce_grads(k, grads)
        eng.step()
        info = eng.step_info()
        ch = 1 << 27   # fp64 norm of the gradients in chunks (bounded temporary)
        ref_norm = math.sqrt(math.fsum(float(torch.linalg.vector_norm(buf[i:i + ch].double()) ** 2)
                                       for i in range(0, buf.numel(), ch))) / S    # norm of G / S (exact scaling)
        assert info.overflow == 0 and info.t == step + 1
        assert abs(info.grad_norm - ref_norm) <= 1e-12 * ref_norm
        assert info.loss_scale == S
        # oracle on the sampled elements (elementwise: c-3 with inv = fp32(1/S), clip = 1)
        sc = np.float32(2.0) ** -(6 + (tid % 8)).astype(np.float32)
        u32 = synth.uniform_at(synth.stream_key(1, synth.KIND_GRAD, 0, step), samp) * sc
        g16 = nx.to16((u32 * np.float32(S)).astype(np.float32), dt)
        G = nx.widen(g16, dt) * np.float32(1.0 / S)
        b1t *= float(np.float32(cfg.beta1))
        b2t *= float(np.float32(cfg.beta2))
        step_f = np.float32(float(np.float32(cfg.lr)) / (1 - b1t))
        rsb2_f = np.float32(1 / math.sqrt(1 - b2t))
        p, m, v = OS.adam_tensor(p, m, v, G, np.float32(1), step_f, rsb2_f, cfg)
        del buf, grads
    # GPU values at the sampled elements (N_d = 1: local index = flat index)
    flat_of = {}
    for b in eng.buckets:
        for pc in eng.pieces[b.first_piece:b.first_piece + b.n_pieces]:
            if pc.tensor_off == 0:
                flat_of[pc.tensor] = b.base + pc.bucket_off
    fidx = torch.from_numpy(np.array([flat_of[t] for t in tid]) + (samp - np.array(offs)[tid])).to(dev)
    P32, M, V = eng.shard()
    for name, gpu, ref in (("p32", P32, p), ("m", M, m), ("v", V, v)):
        got = gpu[fidx].cpu().numpy()
        bad = np.nonzero(got.view(np.uint32) != ref.view(np.uint32))[0]
        assert bad.size == 0, f"{name}: {bad.size} of {samp.size} sampled elements differ"
    p16 = eng.p16_arena()[fidx].cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(p16, nx.to16(p, dt))
    # the library's own memory accounting equals Fig. 1's (2+2+K) Psi' at N_d = 1
    mem = eng.memory()
    assert mem.params16 + mem.grads16 + mem.optimizer == 16 * eng.info.psi_padded
    # padding of the flat layout stays zero (property, every padding range of every bucket)
    pad_total = 0
    for b in eng.buckets:
        pos = 0
        for j in range(b.n_pieces):
            pc = eng.pieces[b.first_piece + j]
            ranges = [(b.base + pos, b.base + pc.bucket_off)]      # alignment gap before the piece
            pos = pc.bucket_off + pc.count
            if j == b.n_pieces - 1:
                ranges.append((b.base + pos, b.base + b.size))      # bucket tail padding
            for lo, hi in ranges:
                if hi > lo:
                    pad_total += hi - lo
                    for arr in (P32, M, V):
                        assert not bool(arr[lo:hi].any())
    assert pad_total == eng.info.psi_padded - psi
    eng.destroy()
    del eng, P32, M, V
    torch.cuda.empty_cache()


def test_replicated_gradients_full_size_sim4():
    """c-9 invariant at BASELINE config 2's full size: with every rank given the same
    gradients, N_d = 4 simulated ranks (pull reduce-scatter + fused all-gather, stage 2)
    must reproduce the N_d = 1 result bitwise (sum of 4 equal 16-bit values is exact,
    1/(4S) is a power of two).  The N_d = 1 path itself is pinned to the oracle above."""
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine, ZeroSimGroup
    torch.cuda.empty_cache()
    ts = synth.gpt2_1p5b()
    nl, ll = [t.numel for t in ts], [t.layer for t in ts]
    dev = torch.device("cuda", 0)
    zc = ZeroConfig.defaults("bf16")
    one = ZeroEngine(nl, ll, 1, 0, 2, zc, "local", align=64, bucket_cap=1 << 26, device=dev)
    grp = ZeroSimGroup(nl, ll, 4, 2, zc, 64, 1 << 26)
    for i in range(len(ts)):
        m = synth.gpu_masters(ts, 1, dev, only={i})
        one.load_master(m)
        for e in grp.ranks:
            e.load_master(m)
    torch.cuda.synchronize()
    for step in range(2):
        buf, grads = synth.gpu_grads_flat(ts, 1, 0, step, torch.bfloat16, dev)
        for k in reversed(range(one.info.n_buckets)):
            one.reduce_grads(k, grads)
        one.step()
        for k in reversed(range(grp[0].info.n_buckets)):
            for e in grp.ranks:
                e.reduce_grads(k, grads)
        for e in grp.ranks:
            e.step()
        torch.cuda.synchronize()
        i1, i4 = one.step_info(), grp[0].step_info()
        assert i1.t == i4.t == step + 1                         # norms: same sum, other fp64 order
        assert abs(i1.grad_norm - i4.grad_norm) <= 1e-12 * i1.grad_norm
        del buf, grads
    # flat index -> (rank, local) for the N_d = 4 layout, compared bucket slice by bucket slice
    P1, M1, V1 = one.shard()
    flat1 = {}
    for b in one.buckets:
        for pc in one.pieces[b.first_piece:b.first_piece + b.n_pieces]:
            if pc.tensor_off == 0:
                flat1[pc.tensor] = b.base + pc.bucket_off
    flat4 = {}
    for b in grp[0].buckets:
        for pc in grp[0].pieces[b.first_piece:b.first_piece + b.n_pieces]:
            if pc.tensor_off == 0:
                flat4[pc.tensor] = b.base + pc.bucket_off
    shards = [e.shard() for e in grp.ranks]
    full4 = [torch.empty(grp[0].info.psi_padded, dtype=torch.float32, device=dev) for _ in range(3)]
    for k, b in enumerate(grp[0].buckets):
        sl = b.size // 4
        for r in range(4):
            for w in range(3):
                full4[w][b.base + r * sl:b.base + (r + 1) * sl] = shards[r][w][b.shard_off:b.shard_off + sl]
    for t, spec in enumerate(ts):
        a, c = flat1[t], flat4[t]
        for w, one_arr in enumerate((P1, M1, V1)):
            assert torch.equal(one_arr[a:a + spec.numel].view(torch.int32),
                               full4[w][c:c + spec.numel].view(torch.int32)), (t, w)
        for r in range(4):   # every rank's replica equals the N_d = 1 parameters
            assert torch.equal(one.p16_arena()[a:a + spec.numel].view(torch.int16),
                               grp[r].p16_arena()[c:c + spec.numel].view(torch.int16)), (t, r)
    one.destroy()
    grp.destroy()
    torch.cuda.empty_cache()
