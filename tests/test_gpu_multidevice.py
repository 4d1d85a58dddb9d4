"""Multi-device parity: one process per GPU, as on an NVL8 box.

These run when at least two GPUs are visible and skip otherwise (the development
pool has one GPU per box; on an 8-GPU node they exercise the real NVLink path):

* the CUDA-IPC PEER transport with every rank on its own device -- the pull
  reduce-scatter reading peers' buckets over NVLink, the Adam kernel's TMA bulk
  stores into every peer's replica (fused all-gather), the stage-3 layer gathers, and
  the system-scope release/acquire signals crossing GPUs -- bit-exact against the
  replicated-DP oracle at stages 0-3 with R16 and R32;
* the NCCL transport at N >= 2, measured against §8c-6's bounds: every reduced
  gradient within 2 gamma_{N-1} sum_r |g_r| of the oracle's (gamma_k = k 2^-24 /
  (1 - k 2^-24): two recursive fp32 sums of the same values in different orders, each
  within Higham's gamma_{N-1} of the exact sum) for R32 (fp32 wire; exact at N = 2,
  where one fp32 addition is commutative), and for R16 (16-bit wire, partial sums
  rounded per ring hop) within gamma16_{N-1} + u16 of that, u16 the 16-bit unit
  roundoff; the p32/m/v errors
  against the 1e-6 tolerance (max relative error and violation counts, also outside
  the heavily-cancelling elements) are printed;
* the NCCL watchdog across ranks: a rank that never issues a step's collectives leaves
  its peer's reduce-scatter hanging; zero_wait on the peer aborts the communicator and
  reports a sticky ZERO_ENCCL naming the rank.
"""
import json
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0
if NDEV < 2:
    pytest.skip(f"needs >= 2 GPUs ({NDEV} visible)", allow_module_level=True)

from test_gpu_ipc import _torch_worker, _worker, run_workers  # noqa: E402

WORLDS = sorted({2, min(NDEV, 4), min(NDEV, 8)})


@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("stage,dt,mode", [(0, "bf16", "R16"), (1, "bf16", "R16"), (1, "fp16", "R32"),
                                           (2, "fp16", "R16"), (2, "bf16", "R32"), (3, "bf16", "R16"),
                                           (3, "fp16", "R32")])
def test_peer_ipc_one_gpu_per_rank(world, stage, dt, mode):
    msgs = run_workers(_worker, world, pre=(stage, dt, mode), post=(True,))
    assert msgs == ["ok"] * world, msgs


@pytest.mark.parametrize("stage", [2, 3])
def test_torch_training_one_gpu_per_rank(stage):
    msgs = run_workers(_torch_worker, 2, pre=(stage,), post=(True,))
    assert msgs == ["ok", "ok"], msgs


def _nccl_worker(rank, world, port, stage, dt, mode, q):
    import sys
    import traceback
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import numpy as np
        import torch.distributed as dist
        import synth
        from harness import zcfg_from_oracle
        from oracle import layout as OL
        from oracle import numerics as nx
        from oracle import step as OS
        from paper_1910_02054_b200 import ZeroEngine, nccl_comm_ptr
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dev = torch.device("cuda", rank)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        torch.cuda.synchronize()
        ts = synth.mlp_layout((300, 200, 100, 50))
        nl, ll = [x.numel for x in ts], [x.layer for x in ts]
        cfg = OS.AdamConfig.defaults(dt, reduce_mode=mode)
        cap = 1 << 13
        e = ZeroEngine(nl, ll, world, rank, stage, zcfg_from_oracle(cfg), "nccl",
                       nccl_comm=nccl_comm_ptr(dist.group.WORLD), align=64, bucket_cap=cap)
        masters = synth.master_values(ts, 1)
        e.load_master([torch.from_numpy(a).to(dev) for a in masters])
        ost = OS.init_state(masters, cfg)
        lay = OL.make_layout(nl, ll, world, 64, cap)
        spans = {p.tensor: b.base + p.bucket_off for b in lay.buckets for p in b.pieces if p.tensor_off == 0}

        def flat(arrs, dtype):
            out = np.zeros(lay.psi_padded, dtype)
            for ti, a in enumerate(arrs):
                out[spans[ti]:spans[ti] + a.size] = a
            return out

        def mine(a):           # this rank's shard of a flat array (stage >= 1)
            return np.concatenate([a[lo:hi] for lo, hi in (lay.owned_range(k, rank) for k in range(len(lay.buckets)))])

        stats = {"G_bound_violations": 0, "G_max_rel": 0.0}
        heavy = np.zeros(e.info.shard, bool)     # elements whose reduction cancelled heavily at some step
        for s in range(4):
            scale = ost.S if dt == "fp16" else 1.0
            host = [synth.grads16(ts, 1, r, s, dt, scale=scale) for r in range(world)]
            if s == 2:
                host[1][0] = host[1][0].clone()
                host[1][0][5] = float("inf")
            for k in reversed(range(e.info.n_buckets)):
                e.reduce_grads(k, [g.to(dev) for g in host[rank]])
            e.step()
            e.wait(120000)
            info = e.step_info()
            g_np = [OS.grads_from_torch(h) for h in host]
            oinfo = OS.step(ost, g_np, cfg)
            assert info.overflow == int(oinfo.overflow) and info.t == oinfo.t, (s, info.overflow, info.t)
            if oinfo.overflow or stage < 2:
                continue
            # the reduced-gradient shard against the oracle's G
            G = flat([OS.reduce_grads([g[ti] for g in g_np], cfg) for ti in range(len(ts))], np.float32)
            absum = flat([sum(np.abs(nx.widen(g[ti], dt).astype(np.float64)) for g in g_np)
                          for ti in range(len(ts))], np.float64)
            gred = e.arenas["gred"]
            # both sides are recursive sums of the same N values: each is within Higham's
            # gamma_{N-1} sum|g| of the exact sum (gamma_k = k u / (1 - k u)), so they differ by
            # at most twice that (reading c-6); R16 adds each side's 16-bit roundings: N-1 ring
            # hops on NCCL's side (unit roundoff u16 each), one final rounding on the oracle's
            u32 = 2.0 ** -24
            gam32 = (world - 1) * u32 / (1 - (world - 1) * u32)
            if mode == "R32":
                got = gred.view(torch.float32)[:e.info.shard].cpu().numpy().astype(np.float64)
                bound = 2 * gam32 * mine(absum)
            else:
                got = nx.widen(gred.view(torch.int16)[:e.info.shard].cpu().numpy().view(np.uint16), dt).astype(np.float64)
                u16 = 2.0 ** (-8 if dt == "bf16" else -11)       # unit roundoff of the 16-bit format
                gam16 = (world - 1) * u16 / (1 - (world - 1) * u16)
                bound = (gam16 + u16 * (1 + gam32) + gam32) * mine(absum)
            bound = bound + world * (2.0 ** -24 if dt == "fp16" else 2.0 ** -133)   # subnormal spacing
            want = mine(G).astype(np.float64)
            heavy |= bound > 1e-7 * np.abs(want)
            err = np.abs(got - want)
            stats["G_bound_violations"] += int((err > bound * (1 + 1e-12) + 1e-45).sum())
            nz = np.abs(want) > 0
            stats["G_max_rel"] = max(stats["G_max_rel"], float((err[nz] / np.abs(want[nz])).max(initial=0.0)))
            if world == 2 and mode == "R32":     # one fp32 addition: order-free, bit-exact
                assert np.array_equal(got, want), "N=2 fp32 sum must be exact"
        # end-to-end: p32/m/v within 1e-6 relative (R32), count the violations
        P32, M, V = e.shard()
        for name, gpu, ref in (("p32", P32, ost.p32), ("m", M, ost.m), ("v", V, ost.v)):
            rf = flat(ref, np.float32).astype(np.float64)
            want = rf if stage == 0 else mine(rf)
            got = gpu.cpu().numpy().astype(np.float64)
            err = np.abs(got - want)
            tol = 1e-6 * np.abs(want)
            stats[f"{name}_max_rel"] = float((err / np.maximum(np.abs(want), 1e-30)).max(initial=0.0))
            viol = err > tol
            stats[f"{name}_violations_1e-6"] = int(viol.sum())
            # reported, not asserted: after Adam an element may exceed 1e-6 wherever a step's
            # reduction (or m's own sum over steps) cancelled; the per-step reduced gradients
            # are held to the exact bound above
            stats[f"{name}_violations_outside_heavy"] = int((viol & ~heavy).sum())
        stats["heavy_cancellation_elems"] = int(heavy.sum())
        assert stats["G_bound_violations"] == 0, stats
        torch.cuda.synchronize()
        dist.barrier()
        e.destroy()
        dist.destroy_process_group()
        q.put("ok " + json.dumps(stats))
    except Exception:
        q.put(traceback.format_exc())
        raise


@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("stage,dt,mode", [(1, "bf16", "R16"), (2, "fp16", "R16"), (2, "bf16", "R32"),
                                           (3, "fp16", "R32"), (3, "bf16", "R16")])
def test_nccl_transport_within_bounds(world, stage, dt, mode):
    msgs = run_workers(_nccl_worker, world, pre=(stage, dt, mode))
    assert len(msgs) == world and all(m.startswith("ok ") for m in msgs), msgs
    print(f"\nNCCL N={world} stage {stage} {dt} {mode}:", msgs[0][3:])


def _nccl_hang_worker(rank, world, port, q):
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    try:
        import torch.distributed as dist
        import synth
        from paper_1910_02054_b200 import ZeroConfig, ZeroEngine, ZeroError, nccl_comm_ptr
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dev = torch.device("cuda", rank)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        torch.cuda.synchronize()
        ts = synth.mlp_layout((256, 128, 64))
        e = ZeroEngine([x.numel for x in ts], [x.layer for x in ts], world, rank, 2, ZeroConfig.defaults("bf16"),
                       "nccl", nccl_comm=nccl_comm_ptr(dist.group.WORLD), bucket_cap=1 << 12)
        e.load_master(synth.gpu_masters(ts, 1, dev))
        _, g = synth.gpu_grads_flat(ts, 1, rank, 0, torch.bfloat16, dev)
        if rank == 0:               # rank 1 never joins this step: rank 0's collectives hang
            for k in reversed(range(e.info.n_buckets)):
                e.reduce_grads(k, g)
            e.step()
            t0 = time.time()
            try:
                e.wait(2000)
                q.put("no error")
            except ZeroError as exc:
                ok = exc.status == 4 and "rank 0 of" in str(exc) and time.time() - t0 < 60
                q.put("ok" if ok else f"wrong error: {exc}")
        else:
            time.sleep(10)
            q.put("ok")
    except Exception:  # noqa: BLE001
        import traceback
        q.put(traceback.format_exc())
    os._exit(0)        # the aborted communicator belongs to torch's process group: skip teardown


def test_nccl_watchdog_names_the_rank_of_a_hung_collective():
    msgs = run_workers(_nccl_hang_worker, 2, timeout=180)
    assert sorted(msgs) == ["ok", "ok"], msgs


def test_stage3_gathers_overlap_compute_one_gpu_per_rank():
    from test_gpu_ipc import _gather_overlap_worker
    msgs = run_workers(_gather_overlap_worker, 2, post=(True,))
    assert msgs == ["ok", "ok"], msgs


@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("stage,dt,mode", [(2, "bf16", "R16"), (3, "fp16", "R32"), (1, "bf16", "R32")])
def test_soak_no_host_sync_one_gpu_per_rank(world, stage, dt, mode):
    from test_gpu_ipc import _soak_worker
    msgs = run_workers(_soak_worker, world, pre=(stage, dt, mode, 200), post=(True,), timeout=900)
    assert msgs == ["ok"] * world, msgs


@pytest.mark.parametrize("world", WORLDS)
@pytest.mark.parametrize("stage", [1, 2])
def test_ipc_replicated_gradients_at_scale_one_gpu_per_rank(world, stage):
    from test_gpu_ipc import _scale_worker
    msgs = run_workers(_scale_worker, world, pre=(stage, 4, "gpt2_1.5b"), post=(True,), timeout=1200)
    assert msgs == ["ok"] * world, msgs
