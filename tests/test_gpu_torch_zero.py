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


class TinyGPTUntied(torch.nn.Module):
    """TinyGPT with its own output head (stage 3 needs every parameter used only
    inside its layer module)."""

    def __init__(self, vocab=512, h=128, n=3, seq=64):
        super().__init__()
        self.wte = torch.nn.Embedding(vocab, h)
        self.wpe = torch.nn.Embedding(seq, h)
        self.h = torch.nn.ModuleList([Block(h) for _ in range(n)])
        self.head = torch.nn.Sequential(torch.nn.LayerNorm(h), torch.nn.Linear(h, vocab, bias=False))

    def forward(self, idx):
        x = self.wte(idx) + self.wpe(torch.arange(idx.shape[1], device=idx.device))
        for b in self.h:
            x = b(x)
        return self.head(x)


@pytest.mark.parametrize("n", [1, 2])
def test_stage3_layer_hooks(n):
    """P_os+g+p from torch: every layer module gathers its parameters before its
    forward and again before its backward and releases them afterwards; n = 2 runs
    two model replicas as the two ranks of a simulated group."""
    from paper_1910_02054_b200 import ZeroConfig, ZeroSimGroup
    from paper_1910_02054_b200.torch_zero import ZeroOptimizer, default_layer_of
    torch.manual_seed(1)
    base = TinyGPTUntied().cuda().to(torch.bfloat16)
    models = [base] + [TinyGPTUntied().cuda().to(torch.bfloat16) for _ in range(n - 1)]
    for m in models[1:]:
        m.load_state_dict(base.state_dict())
    init = [p.detach().float().cpu().numpy().reshape(-1).copy() for p in base.parameters()]
    zc = ZeroConfig.defaults("bf16", pool_buckets=64)
    if n == 1:
        opts = [ZeroOptimizer(base, stage=3, config=zc, bucket_cap=1 << 15)]
    else:
        names = [nm for nm, _ in base.named_parameters()]
        numels = [p.numel() for p in base.parameters()]
        grp = ZeroSimGroup(numels, default_layer_of(names), n, 3, zc, 64, 1 << 15)
        opts = [ZeroOptimizer(models[r], stage=3, config=zc, engine_factory=lambda nl, ll, r=r: grp[r])
                for r in range(n)]
    for p in base.parameters():
        assert p.numel() == 0                     # only shards are resident between uses
    cfg = OS.AdamConfig.defaults("bf16")
    ost = OS.init_state(init, cfg)
    for step in range(2):
        grads = []
        for r in range(n):
            idx = torch.randint(0, 512, (2, 64), device="cuda")
            loss = torch.nn.functional.cross_entropy(models[r](idx).float().view(-1, 512), idx.view(-1))
            loss.backward()
            grads.append(OS.grads_from_torch([p.grad.detach().reshape(-1).cpu() for p in opts[r].params]))
            assert not opts[r]._gathered               # every layer released after its backward
        for o in opts:
            o.step()
        OS.step(ost, grads, cfg)
        assert opts[0].step_info().t == step + 1
    # gather every layer and compare the 16-bit parameters with the oracle
    for r in range(n):
        o = opts[r]
        for L in sorted(o._layer_tensors):
            o._gather(L)
            for t in o._layer_tensors[L]:
                assert np.array_equal(bits16(o.params[t].detach().reshape(-1)), ost.p16[t]), (r, o.names[t])
            o._release(L)
    torch.cuda.synchronize()
