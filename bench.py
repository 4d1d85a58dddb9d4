#!/usr/bin/env python
"""bench.py -- ZeRO-DP step throughput on B200 (BASELINE.json metric).

One "step" = one pass of the whole hot path over one
batch of synthetic gradients: for every bucket (in reverse, as backward produces
them) zero_reduce_grads (flatten/cast/scale + reduce-scatter + overflow/norm
epilogue), then zero_step (global decision, fused partitioned Adam + recast into
the all-gather buffer, all-gather).  Inputs are resident in HBM when the timed
region starts; the working set (~25 GB at 1.5B) is >> the 126 MB L2, so no L2
flush is needed between steps (stated in config.l2).

Default (N=1): GPT-2 1.5B layout (Psi = 1,557,611,200), ZeRO stage 1,
bf16 params/grads, fp32 Adam states.  Under torchrun (N>1) every rank runs the
same layout over NCCL (strong scaling: the model is fixed).

  python bench.py [--steps K] [--warmup W] [--config gpt2_1.5b|gpt_7.5b|mlp1m] [--stage S]
  python bench.py --impl reference      # the CPU oracle on a bounded sample (the reference arm)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ZeRO step Gparams/s at 1/2/4/8 B200; % of HBM+NVLink roofline"
NVLINK_GBS = 770.0   # per direction per GPU: the measured peer copy (B200_PROFILING.md); 900 nominal


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt2_1.5b")
    ap.add_argument("--stage", type=int, default=None)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16"])
    ap.add_argument("--cap", type=int, default=1 << 26)
    ap.add_argument("--align", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N>1: peer = CUDA-IPC pull reduce-scatter + Adam-fused all-gather (default); nccl = library collectives")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--graph", action="store_true",
                    help="capture one whole step (all zero_reduce_grads + zero_step) in a CUDA graph and time replays")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-parallel", action="store_true", help="skip the all-cores oracle baseline")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"   # B200_PROFILING.md fallback


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        k = d["kernels"][kernel]
        return k["dram_bytes_per_launch"], k.get("elements")
    except Exception:
        return None, None


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank time over all ranks (identity without torch.distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    if dist.get_backend() == "gloo":
        device = torch.device("cpu")
    t = torch.tensor([value], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, begin: bool):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        win = [s for t, s in self.samples if self.t0 is not None and self.t0 - 0.06 <= t <= (self.t1 or t) + 0.06]
        if not win:
            win = [s for _, s in self.samples]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in win if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in win if s[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({n for s in win for n, v in zip(names, s[2:]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(win)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle, as it stands, on a bounded sample
# ---------------------------------------------------------------------------
def oracle_sample_run(tensors, dtype: str, seed: int, steps: int, warmup: int, budget_s: float):
    """Time oracle.step on a prefix of `tensors` sized to ~budget_s of CPU work.
    Returns (Gparams/s, sample description, elements, seconds)."""
    import numpy as np  # noqa: F401
    import synth
    from oracle import step as OS
    cfg = OS.AdamConfig.defaults(dtype, grad_dtype=dtype)
    # calibrate on ~1M elements
    cal = [synth.TensorSpec("cal", 1 << 20, 0)]
    st = OS.init_state(synth.master_values(cal, seed), cfg)
    g = [OS.grads_from_torch(synth.grads16(cal, seed, 0, 0, dtype))]
    t0 = time.perf_counter()
    OS.step(st, g, cfg)
    rate = (1 << 20) / max(time.perf_counter() - t0, 1e-6)
    want = max(int(rate * budget_s / max(steps + warmup, 1)), 1 << 16)
    sample, n = [], 0
    for t in tensors:
        if n >= want:
            break
        take = min(t.numel, want - n)
        sample.append(synth.TensorSpec(t.name, take, 0, t.role))
        n += take
    st = OS.init_state(synth.master_values(sample, seed), cfg)
    grads = [[OS.grads_from_torch(synth.grads16(sample, seed, 0, s, dtype))] for s in range(min(steps + warmup, 2))]
    for s in range(warmup):
        OS.step(st, grads[s % len(grads)], cfg)
    t0 = time.perf_counter()
    for s in range(steps):
        OS.step(st, grads[s % len(grads)], cfg)
    dt = time.perf_counter() - t0
    desc = (f"first {n} params of the layout in forward order ({len(sample)} tensors), N_d=1, "
            f"{steps} oracle steps (numpy fp32, 1 thread), inputs pre-generated")
    return n * steps / dt / 1e9, desc, n, dt


def _oracle_worker(args):
    tensors, dtype, seed, n_cap, budget_s, barrier = args
    import torch
    torch.set_num_threads(1)
    import synth
    from oracle import step as OS
    cfg = OS.AdamConfig.defaults(dtype, grad_dtype=dtype)
    sample, n = [], 0
    for t in tensors:
        if n >= n_cap:
            break
        take = min(t.numel, n_cap - n)
        sample.append(synth.TensorSpec(t.name, take, 0, t.role))
        n += take
    st = OS.init_state(synth.master_values(sample, seed), cfg)
    grads = [[OS.grads_from_torch(synth.grads16(sample, seed, 0, s, dtype))] for s in range(2)]
    OS.step(st, grads[0], cfg)                   # warm-up
    barrier.wait()
    t0, steps = time.perf_counter(), 0
    while True:
        OS.step(st, grads[steps % 2], cfg)
        steps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return n * steps, time.perf_counter() - t0


def oracle_parallel_run(tensors, dtype: str, seed: int, budget_s: float, procs: int):
    """The same oracle, unchanged, in `procs` forked worker processes (one per host core),
    each stepping its own copy of a prefix sample for ~budget_s.  Elementwise work is
    independent per element, so the aggregate rate is what the oracle reaches on all
    cores.  Returns (Gparams/s, description)."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    n_cap = 1 << 23
    with ctx.Manager() as man:
        barrier = man.Barrier(procs)
        with ctx.Pool(procs) as pool:
            res = pool.map(_oracle_worker, [(tensors, dtype, seed + w, n_cap, budget_s, barrier) for w in range(procs)])
    work = sum(r[0] for r in res)
    dt = max(r[1] for r in res)
    desc = (f"{procs} worker processes (1 thread each), each stepping its own copy of the first {n_cap} params "
            f"of the layout for ~{budget_s:.0f} s (numpy fp32 oracle, unchanged); aggregate = total params x steps / slowest worker")
    return work / dt / 1e9, desc


def run_reference(args, tensors, psi_total):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    budget = min(150.0, 1.2 * (steps + warmup))
    value, desc, n, dt = oracle_sample_run(tensors, args.dtype, args.seed, steps, warmup, budget)
    line = {
        "metric": METRIC, "value": value, "unit": "Gparams/s", "n_gpus": args.gpus, "steps": steps,
        "warmup": warmup, "ms_per_step": dt / steps * 1e3 * psi_total / n, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} layout, ZeRO stage {args.stage}", "psi": psi_total,
                   "param_dtype": args.dtype, "sample_params": n},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "Gparams/s", "cores": 1, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "Gparams/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    import synth
    tensors = synth.CONFIGS[args.config]()
    if args.stage is None:
        args.stage = {"gpt2_1.5b": 1, "gpt_7.5b": 2, "gpt_60b": 3, "mlp1m": 2}.get(args.config, 1)
    psi_total = synth.psi(tensors)
    if args.impl == "reference":
        return run_reference(args, tensors, psi_total)

    import torch
    import torch.distributed as dist
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine, nccl_comm_ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ZERO_BENCH_SAME_DEVICE=1: every rank on cuda:0 (functional check of the N>1 flow on a
    # 1-GPU box; the ranks time-slice the GPU, so its numbers are not throughput)
    same_dev = os.environ.get("ZERO_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
        if args.transport == "nccl":
            raise SystemExit("NCCL cannot place two ranks on one GPU; use --transport peer")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
            warm = torch.ones(1, device=dev)
            dist.all_reduce(warm)
        torch.cuda.synchronize()
    # the graph mode captures on a side stream (capture is not allowed on the legacy stream)
    stream = torch.cuda.Stream(dev) if args.graph else torch.cuda.current_stream(dev)
    torch.cuda.set_stream(stream)
    tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float16

    # phase events cannot be timed inside a captured graph: --graph runs without them
    cfg = ZeroConfig.defaults(args.dtype, timing=not args.graph)
    if args.dtype == "fp16":
        cfg.loss_scale = 1.0        # inputs are generated unscaled; keep S fixed so no step overflows
        cfg.dynamic_loss_scale = False
    transport = "local" if world == 1 else args.transport
    fallback_note = None

    def make_engine(tr):
        comm = nccl_comm_ptr(dist.group.WORLD) if tr == "nccl" else 0
        e = ZeroEngine([t.numel for t in tensors], [t.layer for t in tensors], world, rank, args.stage, cfg,
                       tr, comm, stream, args.align, args.cap, dev)
        if tr == "peer":
            e.link_peers(dist.new_group(backend="gloo"))   # exchange CUDA IPC handles, open the peer table
        return e

    try:
        eng = make_engine(transport)
        ok = 1
    except Exception as exc:  # e.g. CUDA IPC not permitted in this container
        eng, ok, fallback_note = None, 0, f"{transport} transport failed ({exc}); fell back to nccl"
    if world > 1:                                           # every rank must agree on the transport
        flag = torch.tensor([ok], dtype=torch.int32, device=dev if not same_dev else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0 and transport != "nccl" and not same_dev:
            if eng is not None:
                eng.destroy()
            fallback_note = fallback_note or "a peer rank failed to link; fell back to nccl"
            transport = "nccl"
            eng = make_engine("nccl")
    if eng is None:
        raise SystemExit(fallback_note)
    info = eng.info
    nb = info.n_buckets

    # fp32 masters, loaded in chunks of <= 2^29 elements (bounded temporary memory)
    chunk, cur = [], 0
    for i, t in enumerate(tensors):
        chunk.append(i)
        cur += t.numel
        if cur >= (1 << 29) or i == len(tensors) - 1:
            masters = synth.gpu_masters(tensors, args.seed, dev, only=set(chunk))
            eng.load_master(masters)
            torch.cuda.synchronize()
            del masters
            chunk, cur = [], 0
    grad_buf, grads = synth.gpu_grads_flat(tensors, args.seed, rank, 0, tdt, dev)
    eng.set_grads(grads)
    torch.cuda.synchronize()

    layer_ids = sorted({b.layer for b in eng.buckets})
    layer_buckets = {L: [k for k, b in enumerate(eng.buckets) if b.layer == L] for L in layer_ids}

    def one_step():
        if args.stage == 3:
            # SURVEY §8d step-only protocol for P_os+g+p: gather every layer for the
            # forward (prefetching the next), then in reverse for the backward, each layer
            # followed by its buckets' reduce-scatter; release after use
            for L in layer_ids:
                eng.gather_params(L)
                eng.release_params(L)
            for L in reversed(layer_ids):
                eng.gather_params(L)
                for k in reversed(layer_buckets[L]):
                    eng.reduce_grads(k)
                eng.release_params(L)
        else:
            for k in reversed(range(nb)):
                eng.reduce_grads(k)
        eng.step()

    def barrier():
        if world > 1:
            dist.barrier() if same_dev else dist.barrier(device_ids=[local])

    for _ in range(max(args.warmup, 3)):
        one_step()
    torch.cuda.synchronize()
    barrier()
    eng.timing()                           # reset the phase accumulators
    launches0 = eng.timing().kernel_launches
    graph, launches_per_step = None, None
    if args.graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            one_step()
        launches_per_step = eng.timing().kernel_launches - launches0
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
        barrier()
    run_step = graph.replay if graph is not None else one_step

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    clocks.mark(True)
    evs[0].record(stream)
    for i in range(args.steps):
        run_step()
        evs[i + 1].record(stream)      # per-step boundaries (median / p10 / p90)
    torch.cuda.synchronize()
    clocks.mark(False)
    barrier()
    ms = max_over_ranks(evs[0].elapsed_time(evs[-1]) / args.steps, dev)
    per_step = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps))

    def pct(q):
        return per_step[min(len(per_step) - 1, int(q * (len(per_step) - 1) + 0.5))]
    clk = clocks.stop()
    tm = eng.timing()
    gpu_launches = tm.kernel_launches - launches0 if graph is None else launches_per_step * args.steps
    info_rec = eng.step_info()
    assert info_rec.overflow == 0 and info_rec.t >= args.steps, "benchmark steps must not be skipped"

    value = psi_total / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel (fused Adam), measured live with events on its stream
    hbm_peak, peak_kind = peaks()
    S_e = info.psi_padded if args.stage == 0 else info.shard
    g_bytes = 4 if (cfg.reduce_mode == "R32" and world > 1) else 2
    adam_bytes = (24 + g_bytes + 2) * S_e     # p32, m, v read+write, G read, p16 write
    adam_ms = tm.adam_ms / tm.steps if tm.steps else None
    adam_gbs = adam_bytes / (adam_ms * 1e-3) / 1e9 if adam_ms else None
    traffic, t_elems = ncu_traffic("k_adam")
    if traffic is not None and t_elems:
        traffic = traffic * S_e / t_elems   # the capture's bytes per element x this launch's elements
    reduce_ms = tm.reduce_ms / tm.steps if tm.steps else None
    pp = info.psi_padded
    # step roofline: sum over phases of max(HBM bytes / BW_HBM, NVLink bytes / BW_NVL)
    N = world

    def t_roof_at(hbm_gbs):
        hbm = hbm_gbs * 1e9
        t_flat = 4 * pp / hbm
        if N == 1:
            return t_flat + 28 * pp / hbm
        nvl = 2 * pp * (N - 1) / N / (NVLINK_GBS * 1e9)      # one RS or one AG of Psi' 16-bit elements
        if args.stage == 3:                                   # [AG fwd] -> [flatten + RS + AG bwd] -> [Adam]
            return max(2 * pp / hbm, nvl) + max((4 * pp + 2 * pp + 2 * pp / N) / hbm, 2 * nvl) + 28 * pp / N / hbm
        t_rs = max((2 * pp + 2 * pp / N) / hbm, nvl)
        if args.stage == 0:                                   # [flatten] -> [RS] -> [AG of the sums] -> [full Adam]
            return t_flat + t_rs + max(2 * pp / hbm, nvl) + 28 * pp / hbm
        return t_flat + t_rs + max((28 * pp / N + 2 * pp) / hbm, nvl)   # [flatten] -> [RS] -> [Adam || AG]
    t_roof = t_roof_at(hbm_peak)
    line = {
        "metric": METRIC, "value": value, "unit": "Gparams/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "ms_per_step_p10_p50_p90": [pct(0.1), pct(0.5), pct(0.9)] if world == 1 else None,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} layout, ZeRO stage {args.stage}", "psi": psi_total,
                   "psi_padded": pp, "buckets": nb, "bucket_cap_elems": args.cap, "align_elems": args.align,
                   "param_dtype": args.dtype, "adam_state_dtype": "fp32", "reduce_mode": cfg.reduce_mode,
                   "transport": transport, "parallelism": f"zero{args.stage}-dp{world}",
                   "transport_note": fallback_note,
                   "l2": "no flush: >= 25 GB streamed per step vs 126 MB L2"},
        "roofline": {"bound": "hbm", "kernel": "k_adam (fused partitioned Adam + recast)",
                     "achieved": adam_gbs, "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": adam_gbs / hbm_peak if adam_gbs else None, "traffic": traffic,
                     "bytes_per_launch": adam_bytes, "ms_per_launch": adam_ms,
                     "share_of_step": adam_ms / ms if adam_ms else None,
                     "note": None if adam_ms else "--graph: per-kernel events are not recorded inside the graph"},
        "step_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                          "hbm_gbs": hbm_peak, "nvlink_gbs": NVLINK_GBS if N > 1 else None,
                          "frac_at_spec_hbm_8tbs": t_roof_at(8000.0) * 1e3 / ms,
                          "hbm_gbs": hbm_peak, "nvlink_gbs": NVLINK_GBS if N > 1 else None,
                          "reduce_phase_ms": reduce_ms, "flatten_gbs": 4 * pp / (reduce_ms * 1e-3) / 1e9
                          if (N == 1 and reduce_ms) else None},
        "cuda_graph": bool(graph is not None),
        "clocks": clk,
        "gpu_launches": int(gpu_launches),
    }

    # e2e through the public API with HOST buffers: H2D of the step's gradients from
    # pinned memory + the step + D2H of the step record, every step
    if not args.no_e2e:
        # Every step copies that step's gradients H2D from pinned host memory and reads
        # the step record D2H.  The copy of step s+1 (copy stream, second device buffer)
        # overlaps step s; the host reads step s's record before issuing step s+2.
        host = torch.empty(grad_buf.numel(), dtype=grad_buf.dtype, pin_memory=True)
        host.copy_(grad_buf)
        bufs = [grad_buf, torch.empty_like(grad_buf)]
        views = [grads, [bufs[1][o:o + t.numel] for t, o in zip(tensors, synth.tensor_offsets(tensors))]]
        copy_stream = torch.cuda.Stream(dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]
        rec = eng._info_host
        torch.cuda.synchronize()
        # the PCIe bound of this leg: one pinned H2D of the step's gradients, alone
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(copy_stream):
            h0.record(copy_stream)
            bufs[1].copy_(host, non_blocking=True)
            h1.record(copy_stream)
        torch.cuda.synchronize()
        h2d_ms = h0.elapsed_time(h1)
        barrier()
        K = args.e2e_steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(copy_stream)
        with torch.cuda.stream(copy_stream):
            bufs[0].copy_(host, non_blocking=True)
            copied[0].record(copy_stream)
        for s in range(K):
            cur = s % 2
            stream.wait_event(copied[cur])
            eng.set_grads(views[cur])
            for k in reversed(range(nb)):
                eng.reduce_grads(k)
            eng.step()                              # + 32-byte step record D2H into pinned memory
            consumed[cur].record(stream)            # joined: the flattens have read bufs[cur]
            if s + 1 < K:
                nxt = (s + 1) % 2
                copy_stream.wait_event(consumed[nxt])
                with torch.cuda.stream(copy_stream):
                    bufs[nxt].copy_(host, non_blocking=True)
                    copied[nxt].record(copy_stream)
            stream.synchronize()                    # the host reads step s's result
            _ = bytes(rec.numpy()[:32])
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / K, dev)
        e2e_dev_ms = max_over_ranks(e0.elapsed_time(e1) / K, dev)
        eng.set_grads(grads)
        line["e2e"] = {"value": psi_total / (e2e_ms * 1e-3) / 1e9, "unit": "Gparams/s",
                       "h2d_bytes_per_step": int(grad_buf.numel() * grad_buf.element_size()),
                       "d2h_bytes_per_step": 32, "ms_per_step": e2e_ms, "steps": K,
                       "device_ms_per_step": e2e_dev_ms,
                       "h2d_alone_ms": h2d_ms,
                       "h2d_gbs": grad_buf.numel() * grad_buf.element_size() / (h2d_ms * 1e-3) / 1e9,
                       "frac_of_h2d_bound": max(h2d_ms, ms) / e2e_ms,
                       "note": "value from the host wall clock (device_ms_per_step: CUDA events from the first H2D "
                               "to the last step's end); H2D of step s+1 overlaps step s (double-buffered)"}

    if rank == 0 and not args.no_cpu_baseline:
        v, desc, n, dt = oracle_sample_run(tensors, args.dtype, args.seed, 2, 0, args.cpu_budget_s)
        line["cpu_baseline"] = {"value": v, "unit": "Gparams/s", "cores": 1, "kind": "oracle", "sample": desc}
        procs = len(os.sched_getaffinity(0))
        if procs > 1 and not args.no_cpu_parallel:
            try:
                pv, pdesc = oracle_parallel_run(tensors, args.dtype, args.seed, min(args.cpu_budget_s, 10.0), procs)
                line["cpu_baseline_all_cores"] = {"value": pv, "unit": "Gparams/s", "cores": procs, "kind": "oracle",
                                                  "sample": pdesc}
            except Exception as exc:  # a host without fork/shared-memory support
                line["cpu_baseline_all_cores"] = {"value": None, "note": f"not measured: {exc}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
