"""P_a / P_a+cpu timing on one GPU (NEXT-3 context): partitioned activation
checkpoints of the GPT-2 1.5B block input (batch 8 x seq 1024 x hidden 1600 bf16,
P:824) for 48 layers, with N_m simulated MP ranks sharing the GPU.

Per layer, forward: every MP rank saves its 1/N_m slice; backward, in reverse:
(P_a+cpu: every rank prefetches its slice from host memory,) one rank gathers the
replicated checkpoint.  Reported with CUDA events on the stream: the save and gather
phases, their HBM (or PCIe) bytes and GB/s, and the memory the stores take per rank
against the replicated checkpoints (/ N_m).

  python scripts/pa_bench.py [--n-m 1,2,4,8] [--layers 48]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1910_02054_b200.activation import PaSimGroup, checkpoint_bytes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-m", default="1,2,4,8")
    ap.add_argument("--layers", type=int, default=48)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--hidden", type=int, default=1600)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    numel = args.batch * args.seq * args.hidden
    L = args.layers
    acts = [torch.randn(numel, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
    out = torch.empty(numel, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream()
    for n_m in [int(x) for x in args.n_m.split(",")]:
        for offload in (False, True):
            g = PaSimGroup(n_m, L, numel, "bf16", offload)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            best = None
            for rep in range(args.reps + 1):
                torch.cuda.synchronize()
                ev[0].record(s)
                for l in range(L):
                    g.save(l, acts[l % 4])
                ev[1].record(s)
                for l in reversed(range(L)):
                    g.prefetch(l)
                    g.gather(l, rank=0, out=out)
                ev[2].record(s)
                torch.cuda.synchronize()
                t = (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]))
                if rep and (best is None or sum(t) < sum(best)):
                    best = t
            assert torch.equal(out, acts[0])   # the last gather is layer 0
            sl = g[0].info.slice
            save_bytes = L * n_m * sl * 2 * (1 if offload else 2)      # each rank: read + write its slice
            gather_bytes = L * (numel * 2 * 2 + (n_m * sl * 2 if offload else 0))
            line = {"bench": "pa", "n_m": n_m, "offload": offload, "layers": L, "numel": numel,
                    "save_ms": best[0], "gather_ms": best[1],
                    "save_gbs": save_bytes / (best[0] * 1e-3) / 1e9, "gather_gbs": gather_bytes / (best[1] * 1e-3) / 1e9,
                    "store_bytes_per_rank": g[0].info.host_bytes if offload else g[0].info.device_bytes,
                    "replicated_bytes": checkpoint_bytes(L, args.batch, args.seq, args.hidden, 1),
                    "note": "N_m simulated ranks share one GPU: save/gather bytes are HBM (P_a) or PCIe+HBM (P_a+cpu)"}
            print(json.dumps(line), flush=True)
            g.destroy()


if __name__ == "__main__":
    main()
