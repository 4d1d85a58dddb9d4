"""NEXT-1 context benchmark: a real GPT-2-style training step on one B200 (the paper's
own metric is model TFLOPs per GPU).

forward + backward in torch (bf16, SDPA attention, cuBLAS GEMMs: model compute,
outside the ZeRO hot path), with the ZeRO step driven by ZeroOptimizer: the
post-accumulate-grad hooks flatten each gradient bucket as backward produces it
(on the library's side streams, overlapping the rest of backward), then
zero_step runs the fused Adam into the parameters the model computes with.

Baseline arm (--opt torch): the same model with a conventional mixed-precision
optimizer in plain torch (fp32 master copy, torch.optim.Adam(fused=True), bf16
copy-back), i.e. what the library replaces.  --opt none: forward + backward alone;
(T_zero - T_none) / T_zero is the exposed fraction of the ZeRO work (flattens hidden in
backward or not, plus the step).

  python scripts/train_bench.py [--layers 48 --hidden 1600 --batch 8 --seq 1024] [--opt zero|torch]
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Block(torch.nn.Module):
    def __init__(self, h, heads):
        super().__init__()
        self.heads = heads
        self.ln1 = torch.nn.LayerNorm(h)
        self.qkv = torch.nn.Linear(h, 3 * h)
        self.proj = torch.nn.Linear(h, h)
        self.ln2 = torch.nn.LayerNorm(h)
        self.fc = torch.nn.Linear(h, 4 * h)
        self.fc2 = torch.nn.Linear(4 * h, h)

    def forward(self, x):
        B, S, H = x.shape
        q, k, v = self.qkv(self.ln1(x)).view(B, S, 3, self.heads, H // self.heads).permute(2, 0, 3, 1, 4)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(B, S, H)
        x = x + self.proj(a)
        return x + self.fc2(F.gelu(self.fc(self.ln2(x)), approximate="tanh"))


class GPT(torch.nn.Module):
    def __init__(self, vocab, h, layers, heads, seq):
        super().__init__()
        self.wte = torch.nn.Embedding(vocab, h)
        self.wpe = torch.nn.Embedding(seq, h)
        self.h = torch.nn.ModuleList([Block(h, heads) for _ in range(layers)])
        self.lnf = torch.nn.LayerNorm(h)

    def forward(self, idx):
        x = self.wte(idx) + self.wpe(torch.arange(idx.shape[1], device=idx.device))
        for b in self.h:
            x = b(x)
        return self.lnf(x) @ self.wte.weight.t()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=48)
    ap.add_argument("--hidden", type=int, default=1600)
    ap.add_argument("--heads", type=int, default=25)
    ap.add_argument("--vocab", type=int, default=50257)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--opt", default="zero", choices=["zero", "torch", "none"],
                    help="none: forward + backward only (the compute the optimizer's exposed time is measured against)")
    ap.add_argument("--stage", type=int, default=1)
    args = ap.parse_args()
    torch.manual_seed(0)
    dev = torch.device("cuda", 0)
    model = GPT(args.vocab, args.hidden, args.layers, args.heads, args.seq).to(dev).to(torch.bfloat16)
    psi = sum(p.numel() for p in model.parameters())
    if args.opt == "zero":
        from paper_1910_02054_b200 import ZeroConfig
        from paper_1910_02054_b200.torch_zero import ZeroOptimizer
        opt = ZeroOptimizer(model, stage=args.stage, config=ZeroConfig.defaults("bf16", timing=True))

        def opt_step():
            opt.step()
    elif args.opt == "none":
        def opt_step():
            for p in model.parameters():
                p.grad = None
    else:
        params = [p for p in model.parameters()]
        masters = [p.detach().float().clone().requires_grad_(True) for p in params]
        topt = torch.optim.Adam(masters, lr=1e-3, fused=True)

        def opt_step():
            for m, p in zip(masters, params):
                m.grad = p.grad.float()
            topt.step()
            with torch.no_grad():
                for m, p in zip(masters, params):
                    p.copy_(m)
                    p.grad = None

    idx = torch.randint(0, args.vocab, (args.batch, args.seq), device=dev)
    tgt = torch.roll(idx, -1, dims=1)            # next-token targets

    def step():
        logits = model(idx)
        loss = F.cross_entropy(logits.float().view(-1, args.vocab), tgt.view(-1))
        loss.backward()
        opt_step()
        return loss

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.opt == "zero":
        opt.engine.timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tokens = args.batch * args.seq
    # model FLOPs: 6 Psi per token (fwd+bwd) + causal attention 6 * L * S * h per token (half of 12)
    flops = 6 * psi * tokens + 6 * args.layers * args.seq * args.hidden * tokens
    line = {"bench": "train_step", "opt": args.opt, "stage": args.stage if args.opt == "zero" else None,
            "psi": psi, "layers": args.layers, "hidden": args.hidden, "batch": args.batch, "seq": args.seq,
            "ms_per_step": ms, "tflops_per_gpu": flops / (ms * 1e-3) / 1e12, "loss": float(loss.detach())}
    if args.opt == "zero":
        tm = opt.engine.timing()
        line["zero_step_ms"] = tm.step_ms / max(tm.steps, 1)
        line["adam_ms"] = tm.adam_ms / max(tm.steps, 1)
        line["reduce_phase_ms_inside_backward"] = tm.reduce_ms / max(tm.steps, 1)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
