"""Parity at BASELINE config 2's full size (GPT-2 1.5B layout, Psi = 1,557,611,200,
stage 1, N_d = 1, bf16) in the launch configuration bench.py times, and at config
3's (the paper's Fig. 1 7.5B model, Psi = 7.5e9, stage 2, N_d = 1: 135 GB of arenas).

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


@pytest.mark.parametrize("config,stage", [("gpt2_1.5b", 1), ("gpt_7.5b", 2)])
def test_full_size_sampled(config, stage):
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine
    torch.cuda.empty_cache()
    ts = synth.CONFIGS[config]()
    dev = torch.device("cuda", 0)
    cfg = OS.AdamConfig.defaults("bf16")
    eng = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], 1, 0, stage, ZeroConfig.defaults("bf16"), "local",
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
        buf, grads = synth.gpu_grads_flat(ts, 1, 0, step, torch.bfloat16, dev)
        for k in reversed(range(nb)):
            eng.reduce_grads(k, grads)
        eng.step()
        info = eng.step_info()
        ch = 1 << 27   # fp64 norm of the gradients in chunks (bounded temporary)
        ref_norm = math.sqrt(math.fsum(float(torch.linalg.vector_norm(buf[i:i + ch].double()) ** 2)
                                       for i in range(0, buf.numel(), ch)))
        assert info.overflow == 0 and info.t == step + 1
        assert abs(info.grad_norm - ref_norm) <= 1e-12 * ref_norm
        # oracle on the sampled elements (elementwise: c-3 with inv = 1, clip = 1)
        sc = np.float32(2.0) ** -(6 + (tid % 8)).astype(np.float32)
        u32 = synth.uniform_at(synth.stream_key(1, synth.KIND_GRAD, 0, step), samp) * sc
        g16 = nx.to16(u32.astype(np.float32), "bf16")
        G = nx.widen(g16, "bf16") * np.float32(1.0)
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
    assert np.array_equal(p16, nx.to16(p, "bf16"))
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
