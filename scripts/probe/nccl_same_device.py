"""Probe: can several NCCL ranks share one GPU (one process each)?"""
import os, sys
import torch
import torch.multiprocessing as mp


def w(rank, world, port):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
        t = torch.full((1 << 20,), float(rank + 1), device="cuda")
        dist.all_reduce(t)
        out = torch.empty(1 << 18, device="cuda")
        dist.reduce_scatter_tensor(out, t)
        torch.cuda.synchronize()
        print(f"rank {rank}: ok allreduce={t[0].item()} rs={out[0].item()}", flush=True)
        dist.destroy_process_group()
    except Exception as ex:
        print(f"rank {rank}: FAIL {type(ex).__name__}: {str(ex)[:400]}", flush=True)


if __name__ == "__main__":
    for world in (2, 4):
        mp.start_processes(w, args=(world, 29600 + world), nprocs=world, start_method="spawn", join=True)
