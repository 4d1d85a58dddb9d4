"""Multi-process (gloo, world_size 2 and 4, CPU) tests of the N_d > 1 host logic:
every rank computes the same layout with the C library's host functions, the
owned ranges tile [0, Psi') exactly once, counted volumes equal the closed forms,
and the sharded step protocol (flatten -> reduce-scatter in ascending rank ->
global {flag, norm} -> Adam on the shard -> all-gather) run across real processes
reproduces the unpartitioned oracle bit-exactly (SPEC S:388 stage equivalence)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    errs = []
    while not q.empty():
        errs.append(q.get())
    assert all(p.exitcode == 0 for p in procs), errs
    assert not [e for e in errs if e != "ok"], errs


def _entry(rank, world, port, fn, args, q):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        globals()[fn](rank, world, *args)
        dist.barrier()
        dist.destroy_process_group()
        q.put("ok")
    except Exception:
        q.put(traceback.format_exc())
        raise


# ---------------------------------------------------------------------------
def _layout_and_ownership(rank, world):
    import synth
    import paper_1910_02054_b200 as z
    from oracle import planner as P
    ts = synth.gpt2_1p5b()
    nl, ll = [t.numel for t in ts], [t.layer for t in ts]
    e = z.ZeroEngine(nl, ll, world, rank, 2, transport="nccl", nccl_comm=1, bind=False)
    info = e.info
    # identical layout on every rank
    mine = torch.tensor([info.psi_padded, info.n_buckets, info.shard], dtype=torch.int64)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    assert all(torch.equal(a, mine) for a in allv)
    # owned ranges: per bucket slice r -> gather and check they tile [0, Psi')
    own = torch.tensor([[b.base + rank * (b.size // world), b.size // world] for b in e.buckets], dtype=torch.int64)
    allo = [torch.zeros_like(own) for _ in range(world)]
    dist.all_gather(allo, own)
    cover = np.zeros(info.psi_padded // 64, np.int8)    # every range is a multiple of A = 64
    for o in allo:
        for lo, n in o.tolist():
            assert lo % 64 == 0 and n % 64 == 0
            cover[lo // 64:(lo + n) // 64] += 1
    assert np.all(cover == 1)
    # per-rank memory: equal on all ranks and equal to the Fig. 1 formula on Psi'
    m = e.memory()
    tot = m.params16 + m.grads16 + m.optimizer
    assert tot == P.model_state_bytes(info.psi_padded, 12, world, 2)
    # counted volume per rank: RS slices + AG slices == closed form
    rs = sum(b.size // world * (world - 1) for b in e.buckets)
    sent = torch.tensor([2 * rs], dtype=torch.int64)
    assert int(sent) == z.comm_elems_per_rank(info.psi_padded, world, 2)
    dist.all_reduce(sent)
    assert int(sent) == world * P.step_elems_per_rank(info.psi_padded, world, 2)
    e.destroy()


@pytest.mark.parametrize("world", [2, 4])
def test_layout_ownership_across_processes(world):
    _run(world, "_layout_and_ownership")


# ---------------------------------------------------------------------------
def _sharded_protocol(rank, world, stage, dt, mode):
    """The step schedule across processes: each rank keeps only its shard; the
    arithmetic steps are the oracle's (the CUDA kernels are covered on the GPU)."""
    import math
    import synth
    import paper_1910_02054_b200 as z
    from oracle import numerics as nx
    from oracle import step as OS
    ts = synth.mlp_layout((70, 50, 30))
    nl, ll = [t.numel for t in ts], [t.layer for t in ts]
    info, bk, pc = z.plan_layout(nl, ll, world, 8, 1 << 9)
    cfg = OS.AdamConfig.defaults(dt, reduce_mode=mode)
    masters = synth.master_values(ts, 1)

    def flatten(arrs, dtype):
        out = np.zeros(info.psi_padded, dtype)
        for b in bk:
            for p in pc[b.first_piece:b.first_piece + b.n_pieces]:
                out[b.base + p.bucket_off:b.base + p.bucket_off + p.count] = \
                    np.asarray(arrs[p.tensor])[p.tensor_off:p.tensor_off + p.count]
        return out

    own = [(b.base + rank * (b.size // world), b.size // world) for b in bk]
    idx = np.concatenate([np.arange(lo, lo + n) for lo, n in own])
    P32 = flatten(masters, np.float32)[idx]
    M = np.zeros_like(P32)
    V = np.zeros_like(P32)
    ref = OS.init_state(masters, cfg)
    S, good, t, b1t, b2t = cfg.loss_scale, 0, 0, 1.0, 1.0
    for s in range(3):
        mine = OS.grads_from_torch(synth.grads16(ts, 1, rank, s, dt, scale=S))
        flat = flatten(mine, np.uint16)
        # reduce-scatter: gather every rank's buckets, sum slice r in ascending rank (c-2)
        allg = [torch.zeros(info.psi_padded, dtype=torch.int32) for _ in range(world)]   # gloo: no int16
        dist.all_gather(allg, torch.from_numpy(flat.astype(np.int32)))
        G = OS.reduce_grads([a.numpy().astype(np.uint16)[idx] for a in allg], cfg)
        flag = float((~np.isfinite(G)).any())
        inv = np.float32(1.0 / (world * S))
        u = G * inv
        part = torch.tensor([math.fsum((u.astype(np.float64) ** 2).tolist()), flag], dtype=torch.float64)
        parts = [torch.zeros_like(part) for _ in range(world)]
        dist.all_gather(parts, part)
        sumsq = math.fsum(p[0].item() for p in parts)
        overflow = any(p[1].item() for p in parts)
        assert not overflow
        t += 1
        b1t *= float(np.float32(cfg.beta1))
        b2t *= float(np.float32(cfg.beta2))
        step_f = np.float32(float(np.float32(cfg.lr)) / (1 - b1t))
        rsb2_f = np.float32(1 / math.sqrt(1 - b2t))
        P32, M, V = OS.adam_tensor(P32, M, V, u, np.float32(1), step_f, rsb2_f, cfg)
        # all-gather of the updated 16-bit params -> every rank holds the replica
        p16 = nx.to16(P32, dt)
        allp = [torch.zeros(p16.size, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allp, torch.from_numpy(p16.astype(np.int32)))
        replica = np.zeros(info.psi_padded, np.uint16)
        for r in range(world):
            ridx = np.concatenate([np.arange(b.base + r * (b.size // world), b.base + (r + 1) * (b.size // world))
                                   for b in bk])
            replica[ridx] = allp[r].numpy().astype(np.uint16)
        # the unpartitioned oracle on all ranks' gradients
        grads = [OS.grads_from_torch(synth.grads16(ts, 1, r, s, dt, scale=S)) for r in range(world)]
        info_o = OS.step(ref, grads, cfg)
        assert abs(math.sqrt(sumsq) - info_o.grad_norm) <= 1e-15 * info_o.grad_norm
        if cfg.dynamic_loss_scale:
            good += 1
            if good == cfg.scale_window:
                S, good = 2 * S, 0
    assert np.array_equal(P32.view(np.uint32), flatten(ref.p32, np.float32)[idx].view(np.uint32))
    assert np.array_equal(M.view(np.uint32), flatten(ref.m, np.float32)[idx].view(np.uint32))
    assert np.array_equal(replica, flatten(ref.p16, np.uint16))


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dt,mode", [("bf16", "R16"), ("fp16", "R32")])
def test_sharded_protocol_equals_replicated(world, dt, mode):
    _run(world, "_sharded_protocol", 1, dt, mode)


def _max_over_ranks(rank, world):
    import bench
    v = bench.max_over_ranks(float(rank + 1) * 1.5, torch.device("cpu"))
    assert v == world * 1.5


def test_bench_max_over_ranks():
    _run(2, "_max_over_ranks")


def _min_over_ranks(rank, world):
    import bench
    assert bench.min_over_ranks(0 if rank == world - 1 else 1, torch.device("cpu")) == 0
    assert bench.min_over_ranks(1, torch.device("cpu")) == 1


def test_bench_min_over_ranks():
    """bench.py's e2e leg runs only if every rank could allocate its buffers (MIN over ranks)."""
    _run(2, "_min_over_ranks")
