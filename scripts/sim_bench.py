"""N_d simulated ranks on one GPU (the PEER kernels over a same-device peer table):
per-kernel HBM efficiency of the pull reduce-scatter and the Adam-fused all-gather,
which on an NVL8 box read / write peers over NVLink instead.  Not a throughput
metric of the method (all ranks share one GPU's HBM); it checks that the PEER
kernels themselves stream at HBM speed.

  python scripts/sim_bench.py [--ranks 4] [--stage 2] [--config gpt2_1.5b]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_1910_02054_b200 import ZeroConfig, ZeroSimGroup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--stage", type=int, default=2)
    ap.add_argument("--config", default="gpt2_1.5b")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    ts = synth.CONFIGS[args.config]()
    nl, ll = [t.numel for t in ts], [t.layer for t in ts]
    dev = torch.device("cuda", 0)
    grp = ZeroSimGroup(nl, ll, args.ranks, args.stage, ZeroConfig.defaults("bf16", timing=True), 64, 1 << 26)
    for i in range(len(ts)):
        m = synth.gpu_masters(ts, 1, dev, only={i})
        for e in grp.ranks:
            e.load_master(m)
    grads = [synth.gpu_grads_flat(ts, 1, r, 0, torch.bfloat16, dev)[1] for r in range(args.ranks)]
    for r, e in enumerate(grp.ranks):
        e.set_grads(grads[r])
    nb = grp[0].info.n_buckets

    layers = sorted({b.layer for b in grp[0].buckets})

    def step():
        if args.stage == 3:   # the forward's layer gathers (k_copy pulls of every rank's shard slice)
            for L in layers:
                for e in grp.ranks:
                    e.gather_params(L)
                    e.release_params(L)
        for k in reversed(range(nb)):
            for e in grp.ranks:
                e.reduce_grads(k)
        for e in grp.ranks:
            e.step()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    for e in grp.ranks:
        e.timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tm = [e.timing() for e in grp.ranks]
    pp = grp[0].info.psi_padded
    N = args.ranks
    # HBM bytes of one simulated step (all ranks on this GPU)
    flat = 4 * pp * N                                   # every rank flattens its Psi'
    rs = N * (N * 2 * pp / N + 2 * pp / N)              # each rank reads N slices, writes its reduced slice
    if args.stage == 3:                                 # own shard's p16 only; + every rank gathers Psi' (read + write)
        adam = N * 28 * pp / N + N * 4 * pp
    else:
        adam = N * 28 * pp / N + (N - 1) * 2 * pp       # K=12 state + G + own p16, plus the other replicas' stores
    print(json.dumps({"bench": "sim_step", "ranks": N, "stage": args.stage, "psi_padded": pp,
                      "ms_per_step": ms, "hbm_bytes_per_step": flat + rs + adam,
                      "effective_TBps": (flat + rs + adam) / (ms * 1e-3) / 1e12,
                      "adam_ms_per_rank": [t.adam_ms / max(t.steps, 1) for t in tm]}), flush=True)
    grp.destroy()


if __name__ == "__main__":
    main()
