"""NEXT-1 wiring: a real torch model's backward drives zero_reduce_grads through
post-accumulate-grad hooks (buckets reduced as backward produces them), the model
computes with the engine's 16-bit replica, and zero_step updates it in place.
Against the oracle fed the same autograd gradients: bit-exact."""
import numpy as np
import pytest
import torch

from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import bits16, bits32  # noqa: E402


class Block(torch.nn.Module):
    def __init__(self, h):
        super().__init__()
        self.ln1 = torch.nn.LayerNorm(h)
        self.qkv = torch.nn.Linear(h, 3 * h)
        self.proj = torch.nn.Linear(h, h)
        self.ln2 = torch.nn.LayerNorm(h)
        self.fc = torch.nn.Linear(h, 4 * h)
        self.fc2 = torch.nn.Linear(4 * h, h)

    def forward(self, x):
        q, k, v = self.qkv(self.ln1(x)).chunk(3, dim=-1)
        a = torch.softmax(q @ k.transpose(-1, -2) / q.shape[-1] ** 0.5, dim=-1) @ v
        x = x + self.proj(a)
        return x + self.fc2(torch.nn.functional.gelu(self.fc(self.ln2(x))))


class TinyGPT(torch.nn.Module):
    def __init__(self, vocab=512, h=128, n=3, seq=64):
        super().__init__()
        self.wte = torch.nn.Embedding(vocab, h)
        self.wpe = torch.nn.Embedding(seq, h)
        self.h = torch.nn.ModuleList([Block(h) for _ in range(n)])
        self.lnf = torch.nn.LayerNorm(h)

    def forward(self, idx):
        x = self.wte(idx) + self.wpe(torch.arange(idx.shape[1], device=idx.device))
        for b in self.h:
            x = b(x)
        return self.lnf(x) @ self.wte.weight.t()


@pytest.mark.parametrize("stage", [0, 1, 2])
def test_backward_hooks_drive_the_step(stage):
    from paper_1910_02054_b200 import ZeroConfig
    from paper_1910_02054_b200.torch_zero import ZeroOptimizer
    torch.manual_seed(0)
    model = TinyGPT().cuda().to(torch.bfloat16)
    init = [p.detach().float().cpu().numpy().reshape(-1).copy() for p in model.parameters()]
    opt = ZeroOptimizer(model, stage=stage, config=ZeroConfig.defaults("bf16"), bucket_cap=1 << 15)
    cfg = OS.AdamConfig.defaults("bf16")
    ost = OS.init_state(init, cfg)
    nb = opt.engine.info.n_buckets
    assert nb > 4
    for step in range(3):
        idx = torch.randint(0, 512, (4, 64), device="cuda")
        logits = model(idx)
        loss = torch.nn.functional.cross_entropy(logits.float().view(-1, 512), idx.view(-1))
        loss.backward()
        assert sorted(opt.reduced_order) == list(range(nb))           # every bucket, once, from hooks
        assert opt.reduced_order[0] != 0                                # backward order: not forward order
        grads = [p.grad.detach().reshape(-1).cpu() for p in opt.params]
        opt.step()
        oi = OS.step(ost, [OS.grads_from_torch(grads)], cfg)
        gi = opt.step_info()
        assert gi.t == oi.t and gi.overflow == 0
        assert abs(gi.grad_norm - oi.grad_norm) <= 1e-12 * oi.grad_norm
    # the model's own parameters are the engine's replica: compare them and the masters
    for t, p in enumerate(opt.params):
        assert np.array_equal(bits16(p.detach().reshape(-1)), ost.p16[t]), opt.names[t]
    P32, _, _ = opt.engine.shard()
    flat = {}
    for b in opt.engine.buckets:
        for pc in opt.engine.pieces[b.first_piece:b.first_piece + b.n_pieces]:
            if pc.tensor_off == 0:
                flat[pc.tensor] = b.base + pc.bucket_off
    for t, a in enumerate(ost.p32):
        assert np.array_equal(bits32(P32[flat[t]:flat[t] + a.size]), a.view(np.uint32)), opt.names[t]
    opt.close()
