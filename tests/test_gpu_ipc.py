"""Cross-process PEER transport (CUDA IPC peer table + device-side release/acquire
signals), exercised by 2 processes sharing one GPU: the same pull reduce-scatter /
fused all-gather kernels as on an NVL8 box, with the ranks in separate processes
and contexts.  Each rank's shard and replica must equal the replicated-DP oracle
bit-exactly."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, stage, dt, mode, q, distinct=False):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import numpy as np
        import torch.distributed as dist
        import synth
        from harness import bits16, bits32, zcfg_from_oracle
        from oracle import layout as OL
        from oracle import step as OS
        from paper_1910_02054_b200 import ZeroEngine
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank if distinct else 0)   # distinct: one GPU per rank (NVLink)
        ts = synth.mlp_layout((120, 90, 60, 30))
        nl, ll = [t.numel for t in ts], [t.layer for t in ts]
        cfg = OS.AdamConfig.defaults(dt, reduce_mode=mode)
        cap = 1 << 12
        e = ZeroEngine(nl, ll, world, rank, stage, zcfg_from_oracle(cfg), "peer", align=64, bucket_cap=cap)
        e.link_peers()
        masters = synth.master_values(ts, 1)
        e.load_master([torch.from_numpy(a).cuda() for a in masters])
        ost = OS.init_state(masters, cfg)
        lay = OL.make_layout(nl, ll, world, 64, cap)
        for s in range(4):
            scale = ost.S if dt == "fp16" else 1.0
            host = [synth.grads16(ts, 1, r, s, dt, scale=scale) for r in range(world)]
            if s == 2:                       # overflow on rank 1 -> every rank skips the step
                host[1][0] = host[1][0].clone()
                host[1][0][5] = float("inf")
            mine = [g.cuda() for g in host[rank]]
            for k in reversed(range(e.info.n_buckets)):
                e.reduce_grads(k, mine)
            e.step()
            info = e.step_info()
            oinfo = OS.step(ost, [OS.grads_from_torch(h) for h in host], cfg)
            assert info.overflow == int(oinfo.overflow) and info.t == oinfo.t, (s, info.overflow, info.t)
            if not oinfo.overflow:
                assert abs(info.grad_norm - oinfo.grad_norm) <= 1e-12 * oinfo.grad_norm
        # this rank's shard against the oracle
        spans = {}
        for b in lay.buckets:
            for p in b.pieces:
                if p.tensor_off == 0:
                    spans[p.tensor] = b.base + p.bucket_off

        def flat(arrs, dtype):
            out = np.zeros(lay.psi_padded, dtype)
            for t, a in enumerate(arrs):
                out[spans[t]:spans[t] + a.size] = a
            return out

        P32, M, V = e.shard()
        for name, gpu, ref in (("p32", P32, ost.p32), ("m", M, ost.m), ("v", V, ost.v)):
            rf = flat(ref, np.float32)
            if stage == 0:
                want = rf
            else:
                want = np.concatenate([rf[lo:hi] for lo, hi in (lay.owned_range(k, rank)
                                                                for k in range(len(lay.buckets)))])
            assert np.array_equal(bits32(gpu), want.view(np.uint32)), name
        if stage in (0, 1, 2):
            assert np.array_equal(bits16(e.p16_arena()), flat(ost.p16, np.uint16)), "replica"
        else:
            for L in range(max(t.layer for t in ts) + 1):
                views = e.gather_params(L)
                for t, v in views.items():
                    assert np.array_equal(bits16(v), ost.p16[t]), ("gather", L, t)
                e.release_params(L)
        torch.cuda.synchronize()
        dist.barrier()
        e.destroy()
        dist.destroy_process_group()
        q.put("ok")
    except Exception:
        q.put(traceback.format_exc())
        raise


def run_workers(target, world, pre=(), post=(), timeout=300):
    """Start `world` spawned processes target(rank, world, port, *pre, q, *post); return the
    queue messages (asserting none hung and every exit code is 0)."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=target, args=(r, world, port) + tuple(pre) + (q,) + tuple(post))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout)
    hung = [p for p in procs if p.is_alive()]
    for p in hung:
        p.kill()
        p.join(10)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert not hung, f"workers hung: {msgs}"
    assert all(p.exitcode == 0 for p in procs), msgs
    return msgs


@pytest.mark.parametrize("world,stage,dt,mode", [(2, 1, "bf16", "R16"), (2, 2, "fp16", "R16"), (2, 3, "bf16", "R16"),
                                                 (2, 0, "bf16", "R16"), (3, 2, "bf16", "R32"),
                                                 (4, 3, "fp16", "R16"), (8, 2, "bf16", "R16"), (8, 3, "fp16", "R32")])
def test_processes_share_one_gpu(world, stage, dt, mode):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, stage, dt, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    hung = [p for p in procs if p.is_alive()]
    for p in hung:
        p.kill()
        p.join(10)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert not hung, f"workers hung: {msgs}"
    assert all(p.exitcode == 0 for p in procs) and msgs == ["ok"] * world, msgs


def _torch_worker(rank, world, port, stage, q, distinct=False):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import numpy as np
        import torch.distributed as dist
        from harness import bits16
        from oracle import step as OS
        from paper_1910_02054_b200 import ZeroConfig
        from paper_1910_02054_b200.torch_zero import ZeroOptimizer
        from test_gpu_torch_zero import TinyGPTUntied
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank if distinct else 0)
        torch.manual_seed(3)                       # same initial weights on every rank
        model = TinyGPTUntied().cuda().to(torch.bfloat16)
        init = [p.detach().float().cpu().numpy().reshape(-1).copy() for p in model.parameters()]
        opt = ZeroOptimizer(model, stage=stage, config=ZeroConfig.defaults("bf16"), n_d=world, rank=rank,
                            transport="peer", bucket_cap=1 << 14)
        cfg = OS.AdamConfig.defaults("bf16")
        ost = OS.init_state(init, cfg)
        g = torch.Generator(device="cpu").manual_seed(100 + rank)   # each rank its own data
        for step in range(3):
            idx = torch.randint(0, 512, (2, 64), generator=g).cuda()
            loss = torch.nn.functional.cross_entropy(model(idx).float().view(-1, 512), idx.view(-1))
            loss.backward()
            mine = [p.grad.detach().reshape(-1).cpu() for p in opt.params]
            everyone = [None] * world
            dist.all_gather_object(everyone, mine)
            opt.step()
            OS.step(ost, [OS.grads_from_torch(gs) for gs in everyone], cfg)
        torch.cuda.synchronize()
        if stage < 3:
            for t, p in enumerate(opt.params):
                assert np.array_equal(bits16(p.detach().reshape(-1)), ost.p16[t]), opt.names[t]
        else:
            for L in sorted(opt._layer_tensors):
                opt._gather(L)
                for t in opt._layer_tensors[L]:
                    assert np.array_equal(bits16(opt.params[t].detach().reshape(-1)), ost.p16[t]), opt.names[t]
                opt._release(L)
        torch.cuda.synchronize()
        dist.barrier()
        opt.close()
        dist.destroy_process_group()
        q.put("ok")
    except Exception:
        q.put(traceback.format_exc())
        raise


@pytest.mark.parametrize("stage", [2, 3])
def test_torch_training_across_processes(stage):
    """Two processes, one model replica each, ZeroOptimizer over the CUDA-IPC peer
    transport: real autograd hooks drive the cross-process pull reduce-scatter,
    the fused all-gather (stage 2) or the per-layer gathers (stage 3); every rank's
    parameters equal replicated-DP Adam on both ranks' gradients."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_torch_worker, args=(r, 2, port, stage, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    hung = [p for p in procs if p.is_alive()]
    for p in hung:
        p.kill()
        p.join(10)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert not hung, f"workers hung: {msgs}"
    assert all(p.exitcode == 0 for p in procs) and msgs == ["ok", "ok"], msgs


def _handshake_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import time
        import torch.distributed as dist
        import synth
        from paper_1910_02054_b200 import ZeroConfig, ZeroEngine, ZeroError
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ZERO_PEER_TIMEOUT_MS="2000")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        ts = synth.mlp_layout((64, 32))
        e = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], world, rank, 1, ZeroConfig.defaults("bf16"),
                       "peer", align=64, bucket_cap=1 << 12)
        blobs = [None] * world
        dist.all_gather_object(blobs, e.peer_export())
        if rank == 0:
            t0 = time.time()
            try:
                e.peer_open(blobs)
                q.put("opened without its peer")
            except ZeroError as exc:
                dt = time.time() - t0
                q.put("ok" if ("handshake" in str(exc) and dt < 30) else f"wrong error after {dt:.1f}s: {exc}")
        dist.barrier()          # rank 1 never opened its mappings
        if rank == 1:
            q.put("ok")
        e.destroy()
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        import traceback
        q.put(f"rank {rank}: {exc!r}\n{traceback.format_exc()}")


def test_open_without_peer_times_out():
    """zero_peer_open's handshake is bounded: a peer that never links is reported as an
    error within ZERO_PEER_TIMEOUT_MS (bench.py then exits with that error), not a hang."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_handshake_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    hung = [p for p in procs if p.is_alive()]
    for p in hung:
        p.kill()
        p.join(10)
    msgs = []
    while not q.empty():
        msgs.append(q.get())
    assert not hung, f"workers hung: {msgs}"
    assert sorted(msgs) == ["ok", "ok"], msgs


def _gather_overlap_worker(rank, world, port, q, distinct=False):
    """Stage-3 layer gathers over the CUDA-IPC peer table run on the library's gather
    stream (the parameter all-gather is pipelined across the forward/backward):
    while the caller's compute stream is busy with a long kernel, the gather of layer 0
    and the prefetch of layer 1 complete and can be read from a third stream."""
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import numpy as np
        import torch.distributed as dist
        import synth
        from harness import bits16, zcfg_from_oracle
        from oracle import step as OS
        from paper_1910_02054_b200 import ZeroEngine
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank if distinct else 0)
        ts = synth.mlp_layout((512, 256, 256, 128))
        cfg = OS.AdamConfig.defaults("bf16")
        e = ZeroEngine([t.numel for t in ts], [t.layer for t in ts], world, rank, 3, zcfg_from_oracle(cfg), "peer",
                       align=64, bucket_cap=1 << 14)
        e.link_peers()
        masters = synth.master_values(ts, 1)
        e.load_master([torch.from_numpy(a).cuda() for a in masters])
        ost = OS.init_state(masters, cfg)
        torch.cuda.synchronize()
        dist.barrier()                                 # every rank's shard is loaded
        # one untimed gather/release cycle first: the copy kernel's first launch loads its
        # module (lazy loading), which waits for the device; steady state is what is tested
        for L in (0, 1):
            e.gather_params(L)
            e.release_params(L)
        torch.cuda.synchronize()
        dist.barrier()
        side = torch.cuda.Stream()
        caller = torch.cuda.current_stream()
        # rank 0 stalls its compute stream with ~2 s of "layer compute"; the other ranks do not
        # (ranks sharing one GPU time-slice its SMs between their contexts, so only one of them
        # may keep the GPU busy for the concurrency check to mean anything)
        if rank == 0:
            torch.cuda._sleep(int(4e9))
        t0 = time.time()
        v0 = e.gather_params(0)                        # layer 0 was evicted by the warm-up's prefetch of
        t_call = time.time() - t0                      # layer 2: gathered again, on the gather stream
        time.sleep(0.3)
        with torch.cuda.stream(side):
            got0 = {t: bits16(v) for t, v in v0.items()}
        t_read = time.time() - t0
        busy0 = not caller.query()
        v1 = e.gather_params(1)                        # already prefetched: no new gather
        time.sleep(0.1)
        with torch.cuda.stream(side):
            got1 = {t: bits16(v) for t, v in v1.items()}
        busy1 = not caller.query()
        host_s = time.time() - t0
        ok = (busy0 and busy1 and host_s < 1.5) if rank == 0 else True
        if rank != 0:                                  # read the gathers behind the caller's stream
            torch.cuda.synchronize()
            got0 = {t: bits16(v) for t, v in v0.items()}
            got1 = {t: bits16(v) for t, v in v1.items()}
        ok = ok and all(np.array_equal(got0[t], ost.p16[t]) for t in got0)
        ok = ok and all(np.array_equal(got1[t], ost.p16[t]) for t in got1)
        torch.cuda.synchronize()
        e.release_params(0)
        e.release_params(1)
        dist.barrier()
        e.destroy()
        dist.destroy_process_group()
        q.put("ok" if ok else f"rank {rank}: busy {busy0} {busy1} host {host_s:.2f}s (call {t_call:.3f}s, "
              f"read {t_read:.3f}s), "
              f"layer0 {[np.array_equal(got0[t], ost.p16[t]) for t in got0]}, "
              f"layer1 {[np.array_equal(got1[t], ost.p16[t]) for t in got1]}")
    except Exception:
        import traceback
        q.put(traceback.format_exc())
        raise


def test_stage3_gathers_overlap_compute():
    msgs = run_workers(_gather_overlap_worker, 2)
    assert msgs == ["ok", "ok"], msgs


def _soak_worker(rank, world, port, stage, dt, mode, steps, q, distinct=False):
    """Many steps over the CUDA-IPC peer table with NO host synchronization between them (the
    ranks race ahead through the device-side epoch signals), random bucket orders and a few
    injected overflows; the state after the last step must equal the oracle bit for bit."""
    import random
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import numpy as np
        import torch.distributed as dist
        import synth
        from harness import bits16, bits32, zcfg_from_oracle
        from oracle import layout as OL
        from oracle import step as OS
        from paper_1910_02054_b200 import ZeroEngine
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(rank if distinct else 0)
        ts = synth.mlp_layout((120, 90, 60, 30))
        nl, ll = [t.numel for t in ts], [t.layer for t in ts]
        cfg = OS.AdamConfig.defaults(dt, reduce_mode=mode, max_grad_norm=0.05)
        cap = 1 << 11
        e = ZeroEngine(nl, ll, world, rank, stage, zcfg_from_oracle(cfg), "peer", align=64, bucket_cap=cap)
        e.link_peers()
        masters = synth.master_values(ts, 1)
        e.load_master([torch.from_numpy(a).cuda() for a in masters])
        ost = OS.init_state(masters, cfg)
        lay = OL.make_layout(nl, ll, world, 64, cap)
        inject = {steps // 3, (2 * steps) // 3}
        # every step's gradients of every rank, generated up front (the oracle's loss scale path
        # is replayed first so that fp16 gradients are drawn at the scale each step sees)
        host_all = []
        for s in range(steps):
            scale = ost.S if dt == "fp16" else 1.0
            host = [synth.grads16(ts, 1, r, s, dt, scale=scale) for r in range(world)]
            if s in inject:
                host[1][0] = host[1][0].clone()
                host[1][0][3] = float("inf")
            OS.step(ost, [OS.grads_from_torch(h) for h in host], cfg)
            host_all.append(host[rank])
        dev_all = [[g.cuda() for g in h] for h in host_all]
        torch.cuda.synchronize()
        dist.barrier()
        order_rng = random.Random(7)      # the same bucket order on every rank
        layers = sorted({b.layer for b in lay.buckets})
        for s in range(steps):
            order = list(range(e.info.n_buckets))
            order_rng.shuffle(order)
            if stage == 3:                # forward gathers (prefetch) interleaved with the step
                for L in layers:
                    e.gather_params(L)
                    e.release_params(L)
            for k in order:
                e.reduce_grads(k, dev_all[s])
            e.step()
        info = e.step_info()              # the only synchronization
        assert info.t == ost.t, (info.t, ost.t)
        spans = {p.tensor: b.base + p.bucket_off for b in lay.buckets for p in b.pieces if p.tensor_off == 0}

        def flat(arrs, dtype):
            out = np.zeros(lay.psi_padded, dtype)
            for t, a in enumerate(arrs):
                out[spans[t]:spans[t] + a.size] = a
            return out

        P32, M, V = e.shard()
        for name, gpu, ref in (("p32", P32, ost.p32), ("m", M, ost.m), ("v", V, ost.v)):
            rf = flat(ref, np.float32)
            want = rf if stage == 0 else np.concatenate(
                [rf[lo:hi] for lo, hi in (lay.owned_range(k, rank) for k in range(len(lay.buckets)))])
            assert np.array_equal(bits32(gpu), want.view(np.uint32)), name
        if stage in (1, 2):
            assert np.array_equal(bits16(e.p16_arena()), flat(ost.p16, np.uint16)), "replica"
        torch.cuda.synchronize()
        dist.barrier()
        e.destroy()
        dist.destroy_process_group()
        q.put("ok")
    except Exception:
        q.put(traceback.format_exc())
        raise


@pytest.mark.parametrize("world,stage,dt,mode", [(2, 2, "bf16", "R16"), (3, 1, "fp16", "R32"), (4, 3, "bf16", "R16"),
                                                 (2, 0, "fp16", "R16")])
def test_soak_no_host_sync(world, stage, dt, mode):
    msgs = run_workers(_soak_worker, world, pre=(stage, dt, mode, 120), timeout=600)
    assert msgs == ["ok"] * world, msgs


def _scale_worker(rank, world, port, stage, steps, config, q, distinct=False):
    """The c-9 invariant at scale over the product transport: every rank gets the same
    gradients (GPT-2 1.5B layout, first 8 layer groups: 297M parameters, 2^26 buckets), so
    the CUDA-IPC run must reproduce the N_d = 1 run bit for bit (the fp32 sum of N equal
    16-bit values is exact, 1/N is a power of two).  Rank 0 runs the N_d = 1 reference too."""
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import torch.distributed as dist
        import synth
        from paper_1910_02054_b200 import ZeroConfig, ZeroEngine
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = torch.device("cuda", rank if distinct else 0)
        torch.cuda.set_device(dev)
        ts = synth.CONFIGS[config]()
        nl, ll = [t.numel for t in ts], [t.layer for t in ts]
        zc = ZeroConfig.defaults("bf16")
        e = ZeroEngine(nl, ll, world, rank, stage, zc, "peer", align=64, bucket_cap=1 << 26, device=dev)
        e.link_peers()
        one = ZeroEngine(nl, ll, 1, 0, stage, zc, "local", align=64, bucket_cap=1 << 26, device=dev) if rank == 0 else None
        for i in range(len(ts)):
            m = synth.gpu_masters(ts, 1, dev, only={i})
            e.load_master(m)
            if one:
                one.load_master(m)
        grads = [synth.gpu_grads_flat(ts, 1, 0, s, torch.bfloat16, dev)[1] for s in range(min(steps, 2))]
        grads = [grads[s % len(grads)] for s in range(steps)]
        torch.cuda.synchronize()
        dist.barrier()
        for s in range(steps):                     # no host synchronization between steps
            for k in reversed(range(e.info.n_buckets)):
                e.reduce_grads(k, grads[s])
            e.step()
            if one:
                for k in reversed(range(one.info.n_buckets)):
                    one.reduce_grads(k, grads[s])
                one.step()
        info = e.step_info()
        assert info.t == steps and info.overflow == 0
        # gather the ranks' shards (p32) and rank 0's replica to rank 0, compare with N_d = 1
        P32 = e.shard()[0].cpu()
        shards = [None] * world
        dist.all_gather_object(shards, P32)
        replica = e.p16_arena().cpu() if stage in (1, 2) else None
        ok = True
        if rank == 0:
            p1 = one.shard()[0].cpu()
            flat1 = {pc.tensor: b.base + pc.bucket_off for b in one.buckets
                     for pc in one.pieces[b.first_piece:b.first_piece + b.n_pieces] if pc.tensor_off == 0}
            flatn = {pc.tensor: b.base + pc.bucket_off for b in e.buckets
                     for pc in e.pieces[b.first_piece:b.first_piece + b.n_pieces] if pc.tensor_off == 0}
            full = torch.empty(e.info.psi_padded, dtype=torch.float32)
            for b in e.buckets:
                sl = b.size // world
                for r in range(world):
                    full[b.base + r * sl:b.base + (r + 1) * sl] = shards[r][b.shard_off:b.shard_off + sl]
            for t, spec in enumerate(ts):
                a, c = flat1[t], flatn[t]
                ok = ok and torch.equal(p1[a:a + spec.numel].view(torch.int32), full[c:c + spec.numel].view(torch.int32))
                if replica is not None:
                    ok = ok and torch.equal(one.p16_arena().cpu()[a:a + spec.numel].view(torch.int16),
                                            replica[c:c + spec.numel].view(torch.int16))
        torch.cuda.synchronize()
        dist.barrier()
        e.destroy()
        if one:
            one.destroy()
        dist.destroy_process_group()
        q.put("ok" if ok else f"rank {rank}: differs from N_d = 1")
    except Exception:
        q.put(traceback.format_exc())
        raise


@pytest.mark.parametrize("world,stage,config", [
    (4, 2, "gpt2_1.5b_l8"), (2, 1, "gpt2_1.5b_l8"),
    pytest.param(4, 1, "gpt2_1.5b", marks=pytest.mark.skipif(
        os.environ.get("ZERO_SLOW_TESTS") != "1",
        reason="~15 min: 4 processes time-slicing one GPU at full size (ZERO_SLOW_TESTS=1)"))])
def test_ipc_replicated_gradients_at_scale(world, stage, config):
    """(4, 1, gpt2_1.5b) is BASELINE config 2 at full size (Psi = 1,557,611,200, stage 1) over
    the product transport with 4 processes (gated: the ranks time-slice one GPU, ~15 min;
    passed on the GPU box: profiles/r02_pytest_gpu_with_slow.log)."""
    msgs = run_workers(_scale_worker, world, pre=(stage, 3, config), timeout=1200)
    assert msgs == ["ok"] * world, msgs
