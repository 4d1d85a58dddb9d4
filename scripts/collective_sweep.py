"""BASELINE config 5: reduce-scatter / all-gather sweep, 1 MB .. 4 GB, at N = 2/4/8.

  torchrun --nproc-per-node N scripts/collective_sweep.py [--max-mb 4096]

For each message size S (bytes of 16-bit elements, in place):
  * NCCL  reduce_scatter_tensor / all_gather_into_tensor (torch.distributed, the
    library baseline), and
  * the library's own PEER path: one bucket of S bytes through zero_reduce_grads
    (flatten + pull reduce-scatter over CUDA IPC + epilogue) and, separately, the
    fused Adam + all-gather of zero_step on the same one-bucket layout.
busBW = (S / t) * (N - 1) / N (nccl-tests convention) against 900 GB/s per direction;
the per-rank element counts are checked against S (N-1)/N.
One JSON line per (primitive, size) on rank 0.  Needs N >= 2 GPUs (not run in round 1).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N, rank = dist.get_world_size(), dist.get_rank()
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine
    gloo = dist.new_group(backend="gloo")
    size = 1 << 20
    while size <= args.max_mb << 20:
        n = size // 2 // (64 * N) * (64 * N)
        buf = torch.randn(n, device="cuda").to(torch.bfloat16)
        out = torch.empty(n // N, device="cuda", dtype=torch.bfloat16)
        t_rs = timed(lambda: dist.reduce_scatter_tensor(out, buf), args.iters)
        t_ag = timed(lambda: dist.all_gather_into_tensor(buf, out), args.iters)
        # the library's one-bucket PEER path
        eng = ZeroEngine([n], [0], N, rank, 2, ZeroConfig.defaults("bf16", timing=True), "peer", bucket_cap=0)
        eng.link_peers(gloo)
        eng.load_master([torch.zeros(n, device="cuda")])
        grads = [buf]

        def zero_step():
            eng.reduce_grads(0, grads)
            eng.step()
        t_step = timed(zero_step, args.iters)
        tm = eng.timing()
        eng.destroy()
        if rank == 0:
            for name, t in (("nccl_reduce_scatter", t_rs), ("nccl_all_gather", t_ag),
                            ("zero_peer_rs_plus_fused_adam_ag_step", t_step)):
                bus = size / (t * 1e-3) * (N - 1) / N / 1e9
                print(json.dumps({"primitive": name, "bytes": size, "n_gpus": N, "ms": t, "busbw_GBps": bus,
                                  "frac_of_900": bus / 900.0,
                                  "sent_elems_per_rank": (n // N) * (N - 1)}), flush=True)
        size *= 4
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
