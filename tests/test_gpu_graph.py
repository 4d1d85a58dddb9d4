"""zero_reduce_grads / zero_step are stream-ordered, never synchronize the host and
never allocate, so a whole step can be captured into a CUDA graph and replayed
(the loss-scale / Adam state machine lives on the device).  Replays must equal the
oracle bit-exactly, including an overflow replay that is skipped."""
import numpy as np
import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import bits16, bits32, zcfg_from_oracle  # noqa: E402


@pytest.mark.parametrize("stage", [1, 2])
def test_step_in_cuda_graph(stage):
    from paper_1910_02054_b200 import ZeroEngine
    ts = synth.mlp_layout((200, 100, 50))
    nl, ll = [t.numel for t in ts], [t.layer for t in ts]
    cfg = OS.AdamConfig.defaults("fp16", scale_window=2)
    stream = torch.cuda.Stream()
    e = ZeroEngine(nl, ll, 1, 0, stage, zcfg_from_oracle(cfg), "local", stream=stream, bucket_cap=1 << 12)
    masters = synth.master_values(ts, 1)
    with torch.cuda.stream(stream):
        e.load_master([torch.from_numpy(a).cuda() for a in masters])
    stream.synchronize()
    host = synth.grads16(ts, 1, 0, 0, "fp16", scale=cfg.loss_scale)
    dev = [g.cuda() for g in host]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for k in reversed(range(e.info.n_buckets)):
            e.reduce_grads(k, dev)
        e.step()
    ost = OS.init_state(masters, cfg)
    # S changes on the device (window 2) while the captured inputs stay fixed: the
    # oracle gets the same 16-bit gradients every replay
    grads = [OS.grads_from_torch(host)]
    for rep in range(5):
        if rep == 3:                      # an overflow replay: same graph, non-finite input
            dev[0][0] = float("inf")
        if rep == 4:
            dev[0][0] = host[0][0].cuda()
            grads = [OS.grads_from_torch(host)]
        g.replay()
        stream.synchronize()
        gg = [OS.grads_from_torch([d.cpu() for d in dev])]
        oi = OS.step(ost, gg, cfg)
        gi = e.step_info()
        assert gi.overflow == int(oi.overflow) and gi.t == oi.t and gi.loss_scale == oi.loss_scale
    P32, M, V = e.shard()
    spans = {}
    for b in e.buckets:
        for p in e.pieces[b.first_piece:b.first_piece + b.n_pieces]:
            if p.tensor_off == 0:
                spans[p.tensor] = b.base + p.bucket_off
    for t, a in enumerate(ost.p32):
        o = spans[t]
        assert np.array_equal(bits32(P32[o:o + a.size]), a.view(np.uint32))
        assert np.array_equal(bits16(e.p16_arena()[o:o + a.size]), ost.p16[t])
