"""ZeRO x MP on the GPU: two model-parallel ranks (Megatron tensor slicing of a
GPT-style model, synth.gpt_mp_layout), each running ZeRO-DP over its own simulated
data-parallel group of 2.  The step decision spans the MP group through
zero_step_begin / zero_step_end (the test all-reduces the 16-byte partial across MP
ranks, as a caller would with torch.distributed): the global gradient norm counts
MP-replicated tensors once (reading R-MP1) and an overflow on one MP rank skips the
step on all of them.  Every MP rank's tensors must equal the replicated-DP oracle run
on the union model, bit for bit."""
import numpy as np
import pytest
import torch

import synth
from oracle import layout as OL
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run, bits32, zcfg_from_oracle  # noqa: E402
from paper_1910_02054_b200 import ZeroSimGroup  # noqa: E402


def _view(ts, flags, group, run, align, cap):
    """A harness Pair over an existing simulated group (for its read-back helpers)."""
    p = Pair.__new__(Pair)
    p.run = run
    p.numels = [t.numel for t in ts]
    p.layers = [t.layer for t in ts]
    p.lay = OL.make_layout(p.numels, p.layers, run.n, align, cap, flags)
    p.engines = group.ranks
    p.group = group
    return p


@pytest.mark.parametrize("stage", [1, 2, 3])
@pytest.mark.parametrize("split_decision", [True, False])
def test_mp2_dp2_matches_union_oracle(stage, split_decision):
    n_m, n_d, align, cap, seed = 2, 2, 64, 1 << 12, 3
    U, per = synth.gpt_mp_layout(2, 64, 300, 32, n_m)
    # clipping active: the clip coefficient is a function of the GLOBAL norm
    cfg = OS.AdamConfig.defaults("bf16", max_grad_norm=0.05)
    masters = synth.master_values(U, seed)
    ost = OS.init_state(masters, cfg)
    groups, views = [], []
    for j in range(n_m):
        ts, flags, idx = per[j]
        zc = zcfg_from_oracle(cfg)
        zc.mp_rank = j
        g = ZeroSimGroup([t.numel for t in ts], [t.layer for t in ts], n_d, stage, zc, align, cap, flags=flags)
        dm = [torch.from_numpy(masters[i]).cuda() for i in idx]
        for e in g.ranks:
            e.load_master(dm)
        groups.append(g)
        views.append(_view(ts, flags, g, Run(ts, n_d, stage, cfg, align, cap), align, cap))
    inj = per[1][2][per[1][1].index(0)]      # a partitioned tensor of MP rank 1
    for s in range(4):
        host = [synth.grads16(U, seed, r, s, "bf16") for r in range(n_d)]
        if s == 2:                           # overflow on MP rank 1 only -> every MP rank skips
            host[0][inj] = host[0][inj].clone()
            host[0][inj][5] = float("inf")
        for j in range(n_m):
            idx = per[j][2]
            dev = [[host[r][i].cuda() for i in idx] for r in range(n_d)]
            for k in reversed(range(groups[j][0].info.n_buckets)):
                for r in range(n_d):
                    groups[j][r].reduce_grads(k, dev[r])
        if split_decision:
            for j in range(n_m):
                for r in range(n_d):
                    groups[j][r].step_begin()
            for r in range(n_d):             # the MP all-reduce (SUM) of the 16-byte partial
                parts = [groups[j][r].decision_partial() for j in range(n_m)]
                tot = parts[0] + parts[1]
                for p in parts:
                    p.copy_(tot)
            for j in range(n_m):
                for r in range(n_d):
                    groups[j][r].step_end()
        else:                                # plain zero_step: each MP rank decides alone
            for j in range(n_m):
                for r in range(n_d):
                    groups[j][r].step()
        torch.cuda.synchronize()
        oinfo = OS.step(ost, [OS.grads_from_torch(h) for h in host], cfg)
        if not split_decision:
            break                            # compared after the first step below
        for j in range(n_m):
            for r in range(n_d):
                gi = groups[j][r].step_info()
                assert gi.overflow == int(oinfo.overflow) and gi.t == oinfo.t, (s, j, r)
                if not oinfo.overflow:
                    assert abs(gi.grad_norm - oinfo.grad_norm) <= 1e-12 * oinfo.grad_norm
                    assert gi.clip == np.float32(oinfo.clip) and gi.clip < 1.0
    mismatches = 0
    for j in range(n_m):
        idx = per[j][2]
        for which, ref in (("p32", ost.p32), ("m", ost.m), ("v", ost.v)):
            got, _ = views[j].gpu_tensors(which)
            for t, i in enumerate(idx):
                mismatches += int(np.count_nonzero(bits32(got[t]) != bits32(ref[i])))
        ranks = range(n_d) if stage in (1, 2) else [0]
        for r in ranks:
            got, _ = views[j].gpu_tensors("p16", r)
            for t, i in enumerate(idx):
                mismatches += int(np.count_nonzero(got[t] != ost.p16[i]))
    if split_decision:
        assert mismatches == 0
    else:
        # without the MP-spanning decision each MP rank clips by its own partial norm
        # (and counts the replicated tensors itself): the result is NOT the union model's
        assert mismatches > 0
    for g in groups:
        g.destroy()


def test_step_begin_end_equals_step():
    """Without MP, zero_step_begin + zero_step_end is zero_step (bit-exact vs the oracle)."""
    ts = synth.mlp_layout((200, 100, 50))
    cfg = OS.AdamConfig.defaults("fp16", max_grad_norm=0.5)
    p = Pair(Run(ts, 2, 2, cfg, cap=1 << 12, inject=(1,)))
    for s in range(3):
        host = [p.grads(r, s) for r in range(2)]
        dev = [[g.cuda() for g in h] for h in host]
        for k in reversed(range(len(p.lay.buckets))):
            for r in range(2):
                p.engines[r].reduce_grads(k, dev[r])
        for e in p.engines:
            e.step_begin()
        for e in p.engines:
            e.step_end()
        torch.cuda.synchronize()
        oinfo = OS.step(p.ost, [OS.grads_from_torch(h) for h in host], cfg)
        p.step_no += 1
        p.compare_info(oinfo, [e.step_info() for e in p.engines])
    p.compare()
    with pytest.raises(Exception, match="ESTATE"):
        p.engines[0].step_end()
    p.destroy()
