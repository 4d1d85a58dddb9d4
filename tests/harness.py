"""Test harness: run the CUDA path (through the C ABI) and the CPU oracle on the
same seeded inputs and compare.  Test infrastructure only."""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np
import torch

import synth
from oracle import layout as OL
from oracle import numerics as nx
from oracle import step as OS


def zcfg_from_oracle(cfg: OS.AdamConfig):
    from paper_1910_02054_b200 import ZeroConfig
    return ZeroConfig(lr=cfg.lr, beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps, weight_decay=cfg.weight_decay,
                      max_grad_norm=cfg.max_grad_norm, param_dtype=cfg.param_dtype, grad_dtype=cfg.grad_dtype,
                      reduce_mode=cfg.reduce_mode, dynamic_loss_scale=cfg.dynamic_loss_scale,
                      loss_scale=cfg.loss_scale, min_loss_scale=cfg.min_loss_scale, scale_window=cfg.scale_window,
                      grad_prescale=cfg.grad_prescale)


def bits16(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


def bits32(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float32).view(np.uint32)


@dataclasses.dataclass
class Run:
    tensors: list
    n: int
    stage: int
    cfg: OS.AdamConfig
    align: int = 64
    cap: int = 1 << 17
    seed: int = 1
    inject: Sequence[int] = ()          # steps (0-based) with +inf at rank min(1,n-1), flat index Psi//2
    transport: str = "local"            # n == 1: "local" or "nccl" (1-rank communicator)
    nccl_comm: int = 0
    pool: int = 2                       # C_B staging slots (stages 2/3, N_d > 1)
    prefetch: int = 1                   # stage-3 prefetch depth


class Pair:
    """Oracle state + GPU engines (LOCAL for N=1, a simulated PEER group for N>1)."""

    def __init__(self, run: Run, device="cuda"):
        from paper_1910_02054_b200 import ZeroEngine, ZeroSimGroup
        self.run = run
        ts = run.tensors
        self.numels = [t.numel for t in ts]
        self.layers = [t.layer for t in ts]
        self.lay = OL.make_layout(self.numels, self.layers, run.n, run.align, run.cap)
        zc = zcfg_from_oracle(run.cfg)
        zc.pool_buckets = run.pool
        zc.prefetch_depth = run.prefetch
        if run.n == 1:
            self.engines = [ZeroEngine(self.numels, self.layers, 1, 0, run.stage, zc, run.transport,
                                       nccl_comm=run.nccl_comm, align=run.align, bucket_cap=run.cap)]
            self.group = None
        else:
            self.group = ZeroSimGroup(self.numels, self.layers, run.n, run.stage, zc, run.align, run.cap)
            self.engines = self.group.ranks
        masters = synth.master_values(ts, run.seed)
        self.ost = OS.init_state(masters, run.cfg)
        dev_m = [torch.from_numpy(a).to(device) for a in masters]
        for e in self.engines:
            e.load_master(dev_m)
        torch.cuda.synchronize()
        self.step_no = 0
        self.infos = []

    def grads(self, r: int, s: int):
        cfg = self.run.cfg
        scale = self.ost.S if cfg.param_dtype == "fp16" else 1.0
        dt = cfg.grad_dtype
        gs = synth.grads16(self.run.tensors, self.run.seed, r, s, dt, scale=scale)
        if s in self.run.inject and r == min(1, self.run.n - 1):
            psi = sum(self.numels)
            idx = psi // 2
            for t, n in enumerate(self.numels):
                if idx < n:
                    gs[t] = gs[t].clone()
                    gs[t][idx] = float("inf")
                    break
                idx -= n
        return gs

    def step(self, bucket_order=None):
        s = self.step_no
        n = self.run.n
        host = [self.grads(r, s) for r in range(n)]
        dev = [[g.to("cuda") for g in host[r]] for r in range(n)]
        order = bucket_order if bucket_order is not None else list(reversed(range(len(self.lay.buckets))))
        for k in order:
            for r in range(n):
                self.engines[r].reduce_grads(k, dev[r])
        for r in range(n):
            self.engines[r].step()
        torch.cuda.synchronize()
        oinfo = OS.step(self.ost, [OS.grads_from_torch(host[r]) for r in range(n)], self.run.cfg)
        self.infos.append((oinfo, [e.step_info() for e in self.engines]))
        self.step_no += 1
        return self.infos[-1]

    # -- reading the GPU state back into per-tensor arrays ---------------------
    def flat_from_shards(self, which: str) -> np.ndarray:
        """stage >= 1: reassemble the padded flat fp32 array of p32 / m / v."""
        lay = self.lay
        out = np.zeros(lay.psi_padded, np.float32)
        for r, e in enumerate(self.engines):
            arrs = dict(zip(("p32", "m", "v"), e.shard()))
            a = arrs[which].cpu().numpy()
            for k, b in enumerate(lay.buckets):
                sl = b.size // lay.n_d
                lo, hi = lay.owned_range(k, r)
                out[lo:hi] = a[b.shard_off:b.shard_off + sl]
        return out

    def gpu_tensors(self, which: str, rank: int = 0) -> List[np.ndarray]:
        lay = self.lay
        if which == "p16":
            if self.run.stage == 3:
                flat = np.zeros(lay.psi_padded, np.uint16)
                for r, e in enumerate(self.engines):
                    a = bits16(e.p16_arena())
                    for k, b in enumerate(lay.buckets):
                        sl = b.size // lay.n_d
                        lo, hi = lay.owned_range(k, r)
                        flat[lo:hi] = a[b.shard_off:b.shard_off + sl]
            else:
                flat = bits16(self.engines[rank].p16_arena())
        elif self.run.stage == 0:
            arrs = dict(zip(("p32", "m", "v"), self.engines[rank].shard()))
            flat = arrs[which].cpu().numpy()
        else:
            flat = self.flat_from_shards(which)
        return [flat[o:o + c] for o, c in self._tensor_spans()], flat

    def _tensor_spans(self):
        spans = {}
        for b in self.lay.buckets:
            for p in b.pieces:
                if p.tensor_off == 0:
                    spans[p.tensor] = b.base + p.bucket_off
        return [(spans.get(t, 0), n) for t, n in enumerate(self.numels)]

    def padding_mask(self) -> np.ndarray:
        m = np.ones(self.lay.psi_padded, bool)
        for o, c in self._tensor_spans():
            m[o:o + c] = False
        return m

    def compare(self, exact=True):
        """GPU (p32, m, v, p16) against the oracle: bit-exact (PEER/LOCAL path)."""
        o = self.ost
        for which, ref in (("p32", o.p32), ("m", o.m), ("v", o.v)):
            got, flat = self.gpu_tensors(which)
            for t, (g, w) in enumerate(zip(got, ref)):
                if exact:
                    bad = np.nonzero(bits32(g) != bits32(w))[0]
                    assert bad.size == 0, f"{which} tensor {t}: {bad.size} mismatches, first {bad[:5]} " \
                                          f"gpu {g[bad[:3]]} oracle {w[bad[:3]]}"
                else:
                    np.testing.assert_allclose(g, w, rtol=1e-6, atol=0)
            assert np.all(flat[self.padding_mask()] == 0), f"{which} padding not zero"
        ranks = range(len(self.engines)) if self.run.stage in (0, 1, 2) else [0]
        for r in ranks:
            got, flat = self.gpu_tensors("p16", r)
            for t, (g, w) in enumerate(zip(got, o.p16)):
                if exact:
                    assert np.array_equal(g, w), f"p16 rank {r} tensor {t}"
                else:
                    assert nx.ulp16_distance(g, w).max(initial=0) <= 1
            assert np.all(flat[self.padding_mask()] == 0)

    def compare_info(self, oinfo, ginfos):
        for gi in ginfos:
            assert gi.overflow == int(oinfo.overflow)
            assert gi.t == oinfo.t
            assert gi.loss_scale == oinfo.loss_scale
            if not oinfo.overflow:
                assert abs(gi.grad_norm - oinfo.grad_norm) <= 1e-12 * max(oinfo.grad_norm, 1e-300)
                assert gi.clip == np.float32(oinfo.clip)

    def destroy(self):
        for e in self.engines:
            e.destroy()
