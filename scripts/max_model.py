"""NEXT-2: a B200 analogue of the paper's Table 2 (left half).

For GPT-style layouts of hidden size 8192 (the 60B/100B family) with L
blocks, find the largest L whose ZeRO arenas -- exactly what zero_buffer_sizes
asks the caller to allocate: model states, the C_B staging pool, the stage-3
layer-gather pool and scratch -- fit one B200 (180 GB, P:38's "memory multiplier"
accounting plus the constant-size buffers of §6.2), per stage and DP degree.
Pure host computation through the C ABI (no GPU).  Activations and the model's
own gradient tensors are not counted (the paper's Table 2 counts model states).

  python scripts/max_model.py [--mem-gb 180] [--hidden 8192]
"""
import argparse
import json
import os
import sys

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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mem-gb", type=float, default=180.0)
    ap.add_argument("--hidden", type=int, default=8192)
    args = ap.parse_args()
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
