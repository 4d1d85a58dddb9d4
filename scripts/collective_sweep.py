"""BASELINE config 5: reduce-scatter / all-gather sweep, 1 MB .. 4 GB, at N = 2/4/8.

  python scripts/collective_sweep.py --gpus N [--max-mb 4096]     # spawns N ranks (torch.distributed.run)
  torchrun --nproc-per-node N scripts/collective_sweep.py [...]    # or under torchrun

For each message size S (bytes of the 16-bit buffer, in place), one JSON line per
primitive on rank 0:
  * NCCL reduce_scatter_tensor / all_gather_into_tensor on the bf16 buffer (the
    library baseline: R16, 16-bit wire) and reduce_scatter_tensor on the fp32 buffer
    (R32's wire, 2S bytes);
  * the library's own PEER path on a one-bucket layout of S bytes: the reduce phase of
    zero_reduce_grads (flatten + pull reduce-scatter over CUDA IPC + epilogue; library
    phase events) and the Adam kernel with the fused all-gather stores of zero_step.
busBW = (S / t) * (N - 1) / N (nccl-tests convention) against 900 GB/s per direction
(nominal NVLink 5) and 770 GB/s (measured peer copy); the elements each rank sent are
read from the library's counters and checked against S (N-1)/N per primitive, i.e. the
2 Psi'(N-1)/N of a ZeRO step.  Time is max over ranks.
ZERO_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 (functional only; NCCL is skipped).
Needs N >= 2 GPUs for numbers; not run yet (the development pool has one GPU per box).
"""
import argparse
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def spawn_if_needed(n):
    if "WORLD_SIZE" in os.environ or n <= 1:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--min-mb", type=int, default=1)
    ap.add_argument("--max-mb", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    spawn_if_needed(args.gpus or 1)
    import torch
    import torch.distributed as dist
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine

    same = os.environ.get("ZERO_BENCH_SAME_DEVICE") == "1"
    local = 0 if same else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if same:
        dist.init_process_group("gloo")
        gloo = dist.group.WORLD
    else:
        dist.init_process_group("nccl", device_id=dev)
        gloo = dist.new_group(backend="gloo")
    N, rank = dist.get_world_size(), dist.get_rank()

    def tmax(v):
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if same else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return tmax(e0.elapsed_time(e1) / args.iters)

    def emit(name, size, ms, sent=None, expect=None, wire_bytes=None):
        if rank != 0:
            return
        b = wire_bytes or size
        bus = b / (ms * 1e-3) * (N - 1) / N / 1e9 if ms else None
        print(json.dumps({"primitive": name, "bytes": size, "wire_bytes": b, "n_gpus": N, "ms": ms, "busbw_GBps": bus,
                          "frac_of_900": bus / 900.0 if bus else None, "frac_of_770": bus / 770.0 if bus else None,
                          "sent_elems_per_rank": sent, "expected_elems": expect,
                          "volume_ok": (sent == expect) if sent is not None else None,
                          "same_device_ranks": same}), flush=True)

    size = args.min_mb << 20
    while size <= args.max_mb << 20:
        n = size // 2 // (64 * N) * (64 * N)
        expect = n // N * (N - 1)
        buf = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
        if not same:
            out = torch.empty(n // N, device=dev, dtype=torch.bfloat16)
            emit("nccl_reduce_scatter_bf16", size, timed(lambda: dist.reduce_scatter_tensor(out, buf)))
            emit("nccl_all_gather_bf16", size, timed(lambda: dist.all_gather_into_tensor(buf, out)))
            b32 = buf.float()
            o32 = torch.empty(n // N, device=dev, dtype=torch.float32)
            emit("nccl_reduce_scatter_fp32 (R32 wire)", size, timed(lambda: dist.reduce_scatter_tensor(o32, b32)),
                 wire_bytes=2 * size)
            del b32, o32, out
        # the library's one-bucket PEER path (stage 2): reduce phase and Adam + fused all-gather
        eng = ZeroEngine([n], [0], N, rank, 2, ZeroConfig.defaults("bf16", timing=True), "peer", bucket_cap=0,
                         device=dev)
        eng.link_peers(gloo)
        eng.load_master([torch.zeros(n, device=dev)])
        grads = [buf]

        def zero_step():
            eng.reduce_grads(0, grads)
            eng.step()
        for _ in range(args.warmup):
            zero_step()
        torch.cuda.synchronize()
        dist.barrier()
        eng.timing()
        c0 = eng.comm_counters()
        timed(zero_step)
        c1 = eng.comm_counters()
        tm = eng.timing()
        steps = max(tm.steps, 1)
        rs_ms, ag_ms = tmax(tm.reduce_ms / steps), tmax(tm.adam_ms / steps)
        k = args.iters + args.warmup
        emit("zero_peer_reduce_phase (flatten + pull RS + epilogue)", size, rs_ms,
             (c1.reduce_scatter - c0.reduce_scatter) // k, expect)
        emit("zero_peer_adam_fused_all_gather", size, ag_ms, (c1.all_gather - c0.all_gather) // k, expect)
        eng.destroy()
        del buf
        size *= 4
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
