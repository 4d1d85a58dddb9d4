"""NEXT-2: a B200 analogue of the paper's Table 2 (left half).

For GPT-style layouts of hidden size 8192 (the 60B/100B family) with L
blocks, find the largest L whose ZeRO arenas -- exactly what zero_buffer_sizes
asks the caller to allocate: model states, the C_B staging pool, the stage-3
layer-gather pool and scratch -- fit one B200, per stage and DP degree (P:38's
"memory multiplier" accounting plus the constant-size buffers of §6.2).
Activations and the model's own gradient tensors are not counted (the paper's
Table 2 counts model states).

  python scripts/max_model.py [--mem-gb 180] [--hidden 8192]      # host arithmetic through the C ABI
  python scripts/max_model.py --device [--slack-gb 0.25]           # validated on the GPU

--device (rank 0's context of every (N_d, stage) cell, on this GPU): the budget is
the device's free memory minus the loader's temporary (the fp32 masters of its
largest chunk, <= max(2^28 elements, the largest tensor)) and 0.25 GB of slack;
for the predicted L_max it runs zero_init, zero_buffer_sizes, allocates and binds
the arenas (zeroed on the device) and loads the fp32 masters tensor by tensor
(zero_load_master with NULL for the others: bounded temporary memory), then reads
back zero_query(MEMORY) and checks a sample of the shard against the generator;
with L_max + 1 blocks the arenas plus that temporary must fail to allocate with an
out-of-memory error and leave the device usable.  Config 4 (60B = 75 x 8192, stage 3, N_d = 8) is
instantiated the same way.  N_d > 1 cells build an unlinked PEER context: its
arenas are exactly a real rank's (no step runs without its peers).
"""
import argparse
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1910_02054_b200 import ZeroEngine  # noqa: E402


def arena_bytes(L, h, n, stage, cap=1 << 26):
    ts = synth.gpt_layout(L, h, 50257, 1024)
    e = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], n, 0, stage,
                   transport="local" if n == 1 else "peer", bucket_cap=cap, bind=False)
    s = e.sizes
    total = s.opt_bytes + s.p16_bytes + s.grad_bytes + s.gred_bytes + s.gather_bytes + s.scratch_bytes
    psi = synth.psi(ts)
    e.destroy()
    return total, psi


def max_layers(h, n, stage, mem):
    lo, hi = 0, 1
    while arena_bytes(hi, h, n, stage)[0] <= mem:
        lo, hi = hi, hi * 2
        if hi > 1 << 16:
            break
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if arena_bytes(mid, h, n, stage)[0] <= mem:
            lo = mid
        else:
            hi = mid
    return lo


def load_chunks(ts, limit_elems=1 << 28):
    """Tensor index groups of <= max(limit, largest tensor) elements (bounded temporary)."""
    out, cur, n = [], [], 0
    for i, t in enumerate(ts):
        if cur and n + t.numel > limit_elems:
            out.append(cur)
            cur, n = [], 0
        cur.append(i)
        n += t.numel
    if cur:
        out.append(cur)
    return out


def loader_temp_bytes(h):
    ts = synth.gpt_layout(1, h, 50257, 1024)
    return 4 * max(max(t.numel for t in ts), 1 << 28)


def instantiate(L, h, n, stage, load=True):
    """Rank 0's context of the L-block model on this GPU: arenas bound and (optionally)
    the fp32 masters loaded one tensor at a time.  Returns a result dict."""
    import numpy as np
    import torch
    from paper_1910_02054_b200 import ZeroConfig
    ts = synth.gpt_layout(L, h, 50257, 1024)
    dev = torch.device("cuda", 0)
    t0 = time.time()
    e = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], n, 0, stage, ZeroConfig.defaults("bf16"),
                   transport="local" if n == 1 else "peer", bucket_cap=1 << 26, device=dev)
    torch.cuda.synchronize()
    out = {"arena_bytes": sum(a.numel() for a in e.arenas.values() if a is not None)}
    if load:
        for chunk in load_chunks(ts):   # the loader's temporary: <= LOADER_TEMP_BYTES of fp32 masters
            m = synth.gpu_masters(ts, 1, dev, only=set(chunk))
            e.load_master(m)
            torch.cuda.synchronize()
            del m
        # spot check: the first element this rank owns of the first bucket = the generator's value
        p32 = e.shard()[0]
        b0 = e.buckets[0]
        ref = synth.master_values([synth.TensorSpec("x", 16, 0)], 1)[0]      # wte's first 16 values
        got = p32[:16].cpu().numpy()
        out["shard_spot_check"] = bool(np.array_equal(got, ref)) if b0.base == 0 else None
    mem = e.memory()
    out.update({"params16": mem.params16, "grads16": mem.grads16, "optimizer": mem.optimizer,
                "model_state_bytes": mem.params16 + mem.grads16 + mem.optimizer,
                "staging": mem.staging, "gather_pool": mem.gather_pool, "scratch": mem.scratch,
                "seconds": round(time.time() - t0, 1)})
    e.destroy()
    del e
    gc.collect()
    torch.cuda.empty_cache()
    return out, synth.psi(ts)


def over_the_top(L, h, n, stage):
    """L blocks must not fit: the arenas plus the loader's temporary cannot be allocated
    (an OOM, raised cleanly), and the device stays usable."""
    import torch
    from paper_1910_02054_b200 import ZeroConfig
    ts = synth.gpt_layout(L, h, 50257, 1024)
    e = tmp = None
    try:
        e = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], n, 0, stage, ZeroConfig.defaults("bf16"),
                       transport="local" if n == 1 else "peer", bucket_cap=1 << 26, device=torch.device("cuda", 0))
        tmp = torch.empty(loader_temp_bytes(h), dtype=torch.uint8, device="cuda")
        res = "fit (unexpected)"
    except torch.OutOfMemoryError:
        res = "out of memory"
    if e is not None:
        e.destroy()
    del e, tmp
    gc.collect()
    torch.cuda.empty_cache()
    x = torch.ones(1 << 20, device="cuda")          # the device is still usable
    ok = float(x.sum().item()) == float(1 << 20)
    del x
    return res, ok


def device_main(args):
    import torch
    torch.cuda.init()
    free, total = torch.cuda.mem_get_info()
    # the budget for the arenas: the free memory minus the loader's temporary (fp32 masters of
    # the largest load chunk) and a small allowance for the allocator's rounding
    reserve = loader_temp_bytes(args.hidden) + int(args.slack_gb * 1e9)
    budget = free - reserve
    print(json.dumps({"device": torch.cuda.get_device_name(0), "free_bytes": free, "total_bytes": total,
                      "budget_bytes": budget, "loader_temp_bytes": loader_temp_bytes(args.hidden),
                      "slack_gb": args.slack_gb}), flush=True)
    cells = [(1, s) for s in (0, 1, 2, 3)] + [(n, s) for n in (2, 4, 8) for s in (1, 2, 3)]
    for n, stage in cells:
        L = max_layers(args.hidden, n, stage, budget)
        pred, psi = arena_bytes(L, args.hidden, n, stage)
        row = {"n_d": n, "stage": stage, "layers": L, "psi": psi, "psi_B": round(psi / 1e9, 2),
               "predicted_arena_bytes": pred}
        try:
            res, _ = instantiate(L, args.hidden, n, stage)
            row.update(res)
            row["fits"] = True
        except torch.OutOfMemoryError as exc:
            row["fits"] = False
            row["error"] = str(exc)[:200]
            gc.collect()
            torch.cuda.empty_cache()
        row["one_layer_more"], row["device_usable_after"] = over_the_top(L + 1, args.hidden, n, stage)
        print(json.dumps(row), flush=True)
    # config 4: 60B (75 x 8192), stage 3, N_d = 8 -- rank 0's arenas on one B200
    res, psi = instantiate(75, 8192, 8, 3)
    res.update({"config": "4: 60B layout (75 x 8192), ZeRO stage 3, N_d = 8, rank 0", "psi": psi, "fits": True})
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mem-gb", type=float, default=180.0)
    ap.add_argument("--hidden", type=int, default=8192)
    ap.add_argument("--device", action="store_true")
    ap.add_argument("--slack-gb", type=float, default=0.25)
    args = ap.parse_args()
    if args.device:
        return device_main(args)
    mem = int(args.mem_gb * 1e9)
    rows = []
    for n in (1, 2, 4, 8):
        for stage in (0, 1, 2, 3):
            L = max_layers(args.hidden, n, stage, mem)
            tot, psi = arena_bytes(L, args.hidden, n, stage) if L else (0, 0)
            rows.append({"n_d": n, "stage": stage, "layers": L, "psi_B": round(psi / 1e9, 2),
                         "arena_GB": round(tot / 1e9, 2)})
            print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
