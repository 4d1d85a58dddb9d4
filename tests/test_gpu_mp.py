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


def _mp_torch_worker(j, port, q):
    import os
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import numpy as np
        import torch
        import torch.distributed as dist
        from harness import bits16
        from oracle import step as OS
        from paper_1910_02054_b200 import ZeroConfig
        from paper_1910_02054_b200.torch_zero import ZeroOptimizer
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=j, world_size=2)
        torch.cuda.set_device(0)
        h, k = 96, 40

        class Slice(torch.nn.Module):         # a replicated LayerNorm weight + this rank's weight slice
            def __init__(self):
                super().__init__()
                torch.manual_seed(11)
                self.ln = torch.nn.Parameter(torch.randn(h).to(torch.bfloat16))
                torch.manual_seed(20 + j)
                self.w = torch.nn.Parameter(torch.randn(h * k).mul(0.02).to(torch.bfloat16))

        model = Slice().cuda()
        init = {}
        torch.manual_seed(11)
        init["ln"] = torch.randn(h).to(torch.bfloat16).float().numpy()
        for jj in range(2):
            torch.manual_seed(20 + jj)
            init[jj] = torch.randn(h * k).mul(0.02).to(torch.bfloat16).float().numpy()
        cfg = OS.AdamConfig.defaults("bf16", max_grad_norm=0.5)
        zc = ZeroConfig.defaults("bf16", max_grad_norm=0.5)
        opt = ZeroOptimizer(model, stage=1, config=zc, mp_group=dist.group.WORLD,
                            mp_replicated=lambda names: [n == "ln" for n in names])
        ost = OS.init_state([init["ln"], init[0], init[1]], cfg)
        for s in range(4):
            gen = torch.Generator().manual_seed(1000 + s)
            c_ln = torch.randn(h, generator=gen).to(torch.bfloat16)
            c_w = [torch.randn(h * k, generator=gen).to(torch.bfloat16) for _ in range(2)]
            if s == 2:
                c_w[1][7] = float("inf")     # overflow on MP rank 1 only: both must skip
            loss = (model.ln.float() * c_ln.cuda().float()).sum() + (model.w.float() * c_w[j].cuda().float()).sum()
            loss.backward()
            opt.step()
            OS.step(ost, [OS.grads_from_torch([c_ln, c_w[0], c_w[1]])], cfg)
        torch.cuda.synchronize()
        info = opt.step_info()
        assert info.t == 3, info.t               # 4 steps, one skipped everywhere
        assert np.array_equal(bits16(model.ln.detach()), ost.p16[0]), "ln"
        assert np.array_equal(bits16(model.w.detach()), ost.p16[1 + j]), "w"
        dist.barrier()
        opt.close()
        dist.destroy_process_group()
        q.put("ok")
    except Exception:
        q.put(traceback.format_exc())
        raise


def test_zero_optimizer_mp_group_two_processes():
    """ZeroOptimizer(mp_group=...): two MP ranks in two processes, each with a replicated
    tensor and its own slice; the decision is all-reduced over the MP group (gloo), so
    both clip by the union model's norm (replicated counted once) and both skip the
    step in which only MP rank 1 overflowed -- bit-exact vs the union oracle."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_mp_torch_worker, args=(j, port, q)) for j in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    hung = [p for p in procs if p.is_alive()]
    for p in hung:
        p.kill()
        p.join(10)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert not hung, f"workers hung: {msgs}"
    assert msgs == ["ok", "ok"], msgs
