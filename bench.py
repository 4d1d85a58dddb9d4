#!/usr/bin/env python
"""bench.py -- ZeRO-DP step throughput on B200 (BASELINE.json metric).

One "step" = one pass of the whole hot path over one
batch of synthetic gradients: for every bucket (in reverse, as backward produces
them) zero_reduce_grads (flatten/cast/scale + reduce-scatter + overflow/norm
epilogue), then zero_step (global decision, fused partitioned Adam + recast into
the all-gather buffer, all-gather); at stage 3 the per-layer gathers of the
forward and backward as well.  Inputs are resident in HBM when the timed
region starts.  A working set of >= 25 GB (the GPT layouts) is >> the 126 MB L2, so no
L2 flush is needed between steps; a small one (config 1, ~32 MB) is timed step by step
with L2 flushed before each (stated in config.l2).

Default (N=1): the 7.5B layout of the paper's Fig. 1 (Psi = 7,500,000,000,
120 GB of model states), ZeRO stage 2 (P_os+g), bf16 params/grads with fp32 Adam
states -- the largest BASELINE config that fits one GPU.  The same layout in fp16
with dynamic loss scaling (the paper's precision; reading c-4) is timed
as a second key ("fp16_dynamic").

Multi-GPU (strong scaling: the model is fixed): `--gpus N` under torchrun reads
WORLD_SIZE/RANK/LOCAL_RANK (WORLD_SIZE must equal N); without torchrun, `--gpus N`
spawns the N ranks itself through torch.distributed.run.  ZERO_BENCH_SAME_DEVICE=1
puts every rank on cuda:0 (a functional check of the N>1 flow on a 1-GPU box; the
ranks time-slice one GPU, so its numbers are not throughput).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt_7.5b|gpt2_1.5b|gpt_60b|mlp1m] [--stage S]
  python bench.py --impl reference      # the CPU oracle on a bounded sample (the reference arm)
"""
from __future__ import annotations

import argparse
import gc
import glob
import json
import math
import os
import re
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ZeRO step Gparams/s at 1/2/4/8 B200; % of HBM+NVLink roofline"
NVLINK_GBS = 770.0        # per direction per GPU: the measured peer copy (B200_PROFILING.md)
NVLINK_NOMINAL_GBS = 900.0
L2_BYTES = 126 << 20        # B200 L2
DEFAULT_STAGE = {"gpt2_1.5b": 1, "gpt_7.5b": 2, "gpt_60b": 3, "mlp1m": 2}
# transports with a passing multi-device parity test in this repo's history:
# the CUDA-IPC PEER path is bit-exact across processes (tests/test_gpu_ipc.py); NCCL at
# N > 1 has only the gated tests/test_gpu_multidevice.py, never run on a multi-GPU box
VERIFIED_TRANSPORTS = {"peer"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="ranks (default: WORLD_SIZE, else 1); without torchrun, N > 1 spawns the ranks")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="gpt_7.5b")
    ap.add_argument("--stage", type=int, default=None)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp16"])
    ap.add_argument("--reduce-mode", default="R16", choices=["R16", "R32"])
    ap.add_argument("--cap", type=int, default=1 << 26)
    ap.add_argument("--align", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N>1: peer = CUDA-IPC pull reduce-scatter + Adam-fused all-gather (default); nccl = library collectives")
    ap.add_argument("--allow-unverified", action="store_true",
                    help="run a transport without a passing multi-device parity test (the line says so)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--phase-events", default="auto", choices=["auto", "on", "off"],
                    help="library phase events inside the timed region (auto: on unless the model is < 1e8 "
                         "params, where their host cost is visible; the phase split then comes from a separate "
                         "instrumented pass)")
    ap.add_argument("--graph", action="store_true",
                    help="capture one whole step (all zero_reduce_grads + zero_step) in a CUDA graph and time replays")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--l2-flush", default="auto", choices=["auto", "off"],
                    help="auto: flush L2 before each timed step when the working set fits in it; off: A/B only")
    ap.add_argument("--no-fp16-key", action="store_true", help="skip the fp16 dynamic-loss-scale second run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-parallel", action="store_true", help="skip the all-cores oracle baseline")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    return ap.parse_args()


def world_size(args) -> int:
    """The number of ranks of this run.  Under torchrun WORLD_SIZE rules and must equal
    --gpus when both are given; without torchrun, --gpus N > 1 re-launches this script
    as N ranks (torch.distributed.run on 127.0.0.1) and exits with their status."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if args.gpus is not None and int(ws) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
            raise SystemExit(2)
        return int(ws)
    n = args.gpus or 1
    if n == 1 or args.impl == "reference":
        return n
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


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


def min_over_ranks(value: int, device) -> int:
    """Min of a per-rank integer over all ranks (identity without torch.distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    if dist.get_backend() == "gloo":
        device = torch.device("cpu")
    t = torch.tensor([value], device=device, dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return int(t.item())


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


def run_reference(args, tensors, psi_total, world):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    budget = min(150.0, 1.2 * (steps + warmup))
    value, desc, n, dt = oracle_sample_run(tensors, args.dtype, args.seed, steps, warmup, budget)
    ms_sample = dt / steps * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "Gparams/s", "n_gpus": world, "steps": steps,
        "warmup": warmup,
        # measured: one timed step = the oracle over the bounded sample (sample_params elements)
        "ms_per_step": ms_sample,
        "ms_per_step_kind": "measured per sample step (each step is the oracle over sample_params elements)",
        "ms_per_full_step_extrapolated": ms_sample * psi_total / n,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
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
def nccl_info_summary(log_glob: str, world: int):
    """What NCCL's INFO log says about the communicators of this process (comm size, NVLS)."""
    nr, nvls = [], False
    for p in glob.glob(log_glob):
        try:
            with open(p, errors="replace") as f:
                for line in f:
                    m = re.search(r"\bn[Rr]anks[ =](\d+)", line)
                    if m:
                        nr.append(int(m.group(1)))
                    if "NVLS" in line and "NVLS multicast support is not available" not in line:
                        nvls = True
        except OSError:
            pass
    return {"nranks_seen": sorted(set(nr)), "comm_nranks_ok": bool(nr) and world in nr, "nvls_mentioned": nvls}


def main():
    args = parse()
    world = world_size(args)
    import synth
    tensors = synth.CONFIGS[args.config]()
    if args.stage is None:
        args.stage = DEFAULT_STAGE.get(args.config, 1)
    psi_total = synth.psi(tensors)
    if args.impl == "reference":
        return run_reference(args, tensors, psi_total, world)

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    same_dev = os.environ.get("ZERO_BENCH_SAME_DEVICE") == "1"
    transport = "local" if world == 1 else args.transport
    verified = transport == "local" or transport in VERIFIED_TRANSPORTS
    if not verified and not args.allow_unverified:
        sys.stderr.write(f"bench.py: the {transport} transport has no passing multi-device parity test; "
                         "pass --allow-unverified to time it anyway\n")
        raise SystemExit(3)
    if same_dev and transport == "nccl":
        raise SystemExit("NCCL cannot place two ranks on one GPU; use --transport peer")
    nccl_log = None
    if world > 1 and not same_dev:     # NCCL INFO lines go to a file (never to stdout)
        nccl_log = os.path.join(tempfile.gettempdir(), f"zero_bench_nccl_{os.environ.get('MASTER_PORT', '0')}")
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log + ".%h.%p.log")

    import torch
    import torch.distributed as dist
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine, comm_elems_per_rank, nccl_comm_ptr

    if same_dev:
        local = 0
    elif torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPUs "
                         "(ZERO_BENCH_SAME_DEVICE=1 for a functional run on one GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    gloo = None
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
            gloo = dist.group.WORLD
        else:
            dist.init_process_group("nccl", device_id=dev)
            warm = torch.ones(1, device=dev)
            dist.all_reduce(warm)
            gloo = dist.new_group(backend="gloo")
        torch.cuda.synchronize()
    # the graph mode captures on a side stream (capture is not allowed on the legacy stream)
    stream = torch.cuda.Stream(dev) if args.graph else torch.cuda.current_stream(dev)
    torch.cuda.set_stream(stream)

    def barrier():
        if world > 1:
            dist.barrier() if same_dev else dist.barrier(device_ids=[local])

    def build(dtype):
        """One rank's context for `dtype`: fp32 masters loaded, gradients generated at the
        loss scale S (fp16: dynamic, S0 = 2^16; bf16: static S = 1; reading c-4)."""
        cfg = ZeroConfig.defaults(dtype, timing=not args.graph, reduce_mode=args.reduce_mode)
        comm = nccl_comm_ptr(dist.group.WORLD) if transport == "nccl" else 0
        eng = ZeroEngine([t.numel for t in tensors], [t.layer for t in tensors], world, rank, args.stage, cfg,
                         transport, comm, stream, args.align, args.cap, dev)
        if transport == "peer":
            eng.link_peers(gloo)      # exchange CUDA IPC handles, open the peer table (fails loudly)
        chunk, cur = [], 0           # fp32 masters in chunks of <= 2^29 elements
        for i, t in enumerate(tensors):
            chunk.append(i)
            cur += t.numel
            if cur >= (1 << 29) or i == len(tensors) - 1:
                masters = synth.gpu_masters(tensors, args.seed, dev, only=set(chunk))
                eng.load_master(masters)
                torch.cuda.synchronize()
                del masters
                chunk, cur = [], 0
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
        grad_buf, grads = synth.gpu_grads_flat(tensors, args.seed, rank, 0, tdt, dev, scale=cfg.loss_scale)
        eng.set_grads(grads)
        torch.cuda.synchronize()
        return eng, cfg, grad_buf, grads

    def make_step(eng):
        nb = eng.info.n_buckets
        layer_ids = sorted({b.layer for b in eng.buckets})
        layer_buckets = {L: [k for k, b in enumerate(eng.buckets) if b.layer == L] for L in layer_ids}

        def one_step(evs=None):
            if args.stage == 3:
                # SURVEY §8d step-only protocol for P_os+g+p: gather every layer for the
                # forward (prefetching the next), then in reverse for the backward, each layer
                # followed by its buckets' reduce-scatter; release after use
                if evs:
                    evs[0].record(stream)
                for L in layer_ids:
                    eng.gather_params(L)
                    eng.release_params(L)
                if evs:
                    evs[1].record(stream)
                for L in reversed(layer_ids):
                    eng.gather_params(L)
                    for k in reversed(layer_buckets[L]):
                        eng.reduce_grads(k)
                    eng.release_params(L)
                if evs:
                    evs[2].record(stream)
            else:
                for k in reversed(range(nb)):
                    eng.reduce_grads(k)
            eng.step()
            if evs:
                evs[3].record(stream)
        return one_step

    def timed(eng, steps, sample_clocks=True):
        one_step = make_step(eng)
        for _ in range(max(args.warmup, 3)):
            one_step()
        torch.cuda.synchronize()
        barrier()
        eng.timing()                           # reset the phase accumulators
        launches0 = eng.timing().kernel_launches
        comm0 = eng.comm_counters()
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
        clocks = ClockSampler(local) if sample_clocks else None
        if clocks:
            clocks.start()
            time.sleep(0.3)
        barrier()
        torch.cuda.synchronize()
        comm1 = eng.comm_counters()
        in_region = graph is None and (args.phase_events == "on" or
                                       (args.phase_events == "auto" and psi_total >= 100_000_000))
        if graph is None and not in_region:
            eng.set_timing(False)
        if clocks:
            clocks.mark(True)
        if flush_buf is None:
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            evs[0].record(stream)
            for i in range(steps):
                run_step()
                evs[i + 1].record(stream)      # per-step boundaries (median / p10 / p90)
        else:
            # the working set fits in L2: every timed step starts from a flushed L2 (a write of
            # 2x the L2 size between steps, outside the step's event pair)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)]
            for i in range(steps):
                flush_buf.fill_(i & 0xFF)
                evs[i][0].record(stream)
                run_step()
                evs[i][1].record(stream)
        torch.cuda.synchronize()
        if clocks:
            clocks.mark(False)
        barrier()
        comm2 = eng.comm_counters()
        if flush_buf is None:
            ms = max_over_ranks(evs[0].elapsed_time(evs[-1]) / steps, dev)
            per_step = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(steps))
        else:
            per_step = sorted(a.elapsed_time(b) for a, b in evs)
            ms = max_over_ranks(sum(per_step) / steps, dev)
        clk = clocks.stop() if clocks else None
        tm = eng.timing()
        launches = tm.kernel_launches - launches0 if graph is None else launches_per_step * steps
        phase_events = "in the timed region" if in_region else None
        if graph is None and not in_region:    # the phase split from a separate instrumented pass
            eng.set_timing(True)
            n_instr = min(steps, 20)
            for _ in range(n_instr):
                one_step()
            torch.cuda.synchronize()
            tm = eng.timing()
            phase_events = f"a separate instrumented pass of {n_instr} steps (none in the timed region)"
        phases = None
        if args.stage == 3 and graph is None:
            # one more (untimed) step with events on the caller's stream: with no model compute
            # in the step-only protocol, the forward phase is the exposed gather time
            pe = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            one_step(pe)
            torch.cuda.synchronize()
            phases = {"fwd_gather_phase_ms": pe[0].elapsed_time(pe[1]),
                      "bwd_gather_reduce_phase_ms": pe[1].elapsed_time(pe[2]),
                      "step_phase_ms": pe[2].elapsed_time(pe[3]),
                      "note": "caller-stream events; no model compute in the step-only protocol, so the "
                              "forward phase is all exposed gather time (a real forward hides it, P:476)"}
        rec = eng.step_info()
        if graph is None:
            sent = [(getattr(comm2, f) - getattr(comm1, f)) / steps for f in ("reduce_scatter", "all_gather", "all_reduce")]
        else:   # replays do not pass through the host counters: the captured step's counts
            sent = [getattr(comm1, f) - getattr(comm0, f) for f in ("reduce_scatter", "all_gather", "all_reduce")]
        return {"ms": ms, "per_step": per_step, "tm": tm, "launches": launches, "clocks": clk, "rec": rec,
                "graph": graph is not None, "sent": sent, "phases": phases, "phase_events": phase_events}

    # bytes one step streams (flatten 4 B + Adam 28 B per parameter): below 4x the L2, flush it
    flush_buf = None
    if 32 * psi_total < 4 * L2_BYTES and args.l2_flush == "auto":
        flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    l2_note = (f"no flush: {32 * psi_total / 1e9:.3g} GB streamed per step vs 126 MB L2"
               + (" (--l2-flush off: L2-resident A/B, not a contract number)" if args.l2_flush == "off" else "")
               if flush_buf is None else
               f"flushed before every timed step ({2 * L2_BYTES >> 20} MB write, outside the step's events): "
               f"the {32 * psi_total / 1e6:.3g} MB working set fits in the 126 MB L2")

    eng, cfg, grad_buf, grads = build(args.dtype)
    info = eng.info
    nb = info.n_buckets
    info_buckets = list(eng.buckets)
    res = timed(eng, args.steps)
    rec = res["rec"]
    assert rec.overflow == 0 and rec.t >= args.steps, "benchmark steps must not be skipped"
    ms, tm = res["ms"], res["tm"]
    per_step = res["per_step"]

    def pct(q):
        return per_step[min(len(per_step) - 1, int(q * (len(per_step) - 1) + 0.5))]

    value = psi_total / (ms * 1e-3) / 1e9
    hbm_peak, peak_kind = peaks()
    N = world
    pp = info.psi_padded
    S_e = pp if args.stage == 0 else info.shard
    r32 = cfg.reduce_mode == "R32" and N > 1
    g_bytes = 4 if r32 else 2

    def adam_roofline(tm_):
        """achieved HBM GB/s of the fused Adam, CUDA events on its stream over the timed region"""
        adam_bytes = (24 + g_bytes + 2) * S_e      # p32, m, v read+write, G read, p16 write
        adam_ms = tm_.adam_ms / tm_.steps if tm_.steps else None
        gbs = adam_bytes / (adam_ms * 1e-3) / 1e9 if adam_ms else None
        return adam_bytes, adam_ms, gbs

    adam_bytes, adam_ms, adam_gbs = adam_roofline(tm)
    traffic, t_elems = ncu_traffic("k_adam")
    if traffic is not None and t_elems:
        traffic = traffic * S_e / t_elems   # the capture's bytes per element x this launch's elements
    reduce_ms = tm.reduce_ms / tm.steps if tm.steps else None

    def t_roof_at(hbm_gbs, nvl_gbs=NVLINK_GBS):
        # step roofline: sum over phases of max(HBM bytes / BW_HBM, NVLink bytes / BW_NVL)
        hbm = hbm_gbs * 1e9
        t_flat = 4 * pp / hbm
        adam = (24 + g_bytes + 2) * pp / N
        if N == 1:
            return t_flat + adam / hbm
        nvl = 2 * pp * (N - 1) / N / (nvl_gbs * 1e9)      # one RS or one AG of Psi' 16-bit elements
        nvl_rs = nvl * (2 if (r32 and transport == "nccl") else 1)
        if args.stage == 3:                                   # [AG fwd] -> [flatten + RS + AG bwd] -> [Adam]
            return max(2 * pp / hbm, nvl) + max((4 * pp + 2 * pp + 2 * pp / N) / hbm, nvl_rs + nvl) + adam / hbm
        t_rs = max((2 * pp + 2 * pp / N) / hbm, nvl_rs)
        if args.stage == 0:                                   # [flatten] -> [RS] -> [AG of the sums] -> [full Adam]
            return t_flat + t_rs + max(2 * pp / hbm, nvl) + 28 * pp / hbm
        return t_flat + t_rs + max((adam + 2 * pp) / hbm, nvl)   # [flatten] -> [RS] -> [Adam || AG]
    t_roof = t_roof_at(hbm_peak)

    # counted elements sent per rank per step vs the paper's closed forms
    counted = sum(res["sent"])
    closed = comm_elems_per_rank(pp, N, args.stage)
    comm = {"elems_sent_per_step": {"reduce_scatter": res["sent"][0], "all_gather": res["sent"][1],
                                    "all_reduce": res["sent"][2], "total": counted},
            "closed_form": closed, "closed_form_name": "3 Psi'(N-1)/N" if args.stage == 3 else "2 Psi'(N-1)/N",
            "equal": counted == closed}
    if args.stage == 3 and N > 1:
        # the paper's 3 Psi gathers every layer in the forward and again in the backward;
        # the gather pool still holds the last prefetch_depth + 1 layers of the forward when the
        # backward starts, and those are reused, not gathered again
        sizes = {}
        for b in info_buckets:
            sizes[b.layer] = sizes.get(b.layer, 0) + b.size
        reused = sum(sizes[L] for L in sorted(sizes)[-(cfg.prefetch_depth + 1):])
        expected = closed - reused // N * (N - 1)
        comm.update({"turnaround_reuse_elems": reused, "expected_with_reuse": expected,
                     "equal": counted == expected, "within_closed_form": counted <= closed})
    if N > 1:
        # bus bandwidth in the nccl-tests convention, (S / t) (N-1)/N with S = the 16-bit buffer
        # (2 Psi' bytes); the phases overlap HBM work (the flattens; the Adam of the fused AG)
        S_bytes = 2 * pp
        ag_ms = (tm.ag_ms / tm.steps if tm.steps else None) if transport == "nccl" else adam_ms
        comm["rs_phase_ms"] = reduce_ms
        comm["rs_busbw_gbs"] = S_bytes / (reduce_ms * 1e-3) / 1e9 * (N - 1) / N if reduce_ms else None
        comm["ag_phase_ms"] = ag_ms
        comm["ag_busbw_gbs"] = S_bytes / (ag_ms * 1e-3) / 1e9 * (N - 1) / N if ag_ms else None
        comm["ag_phase_kind"] = "nccl all-gather group" if transport == "nccl" else "fused into the Adam kernel's bulk stores"
        comm["busbw_ref_gbs"] = {"nominal": NVLINK_NOMINAL_GBS, "measured_peer_copy": NVLINK_GBS}
        for k in ("rs", "ag"):
            v = comm.get(f"{k}_busbw_gbs")
            comm[f"{k}_frac_of_nominal"] = v / NVLINK_NOMINAL_GBS if v else None

    line = {
        "metric": METRIC, "value": value, "unit": "Gparams/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "ms_per_step_p10_p50_p90": [pct(0.1), pct(0.5), pct(0.9)],
        "higher_is_better": True, "scaling": "strong",
        # dtype = the arithmetic type the path computes in (fp32 Adam / fp32 sums); the
        # parameter and gradient storage type is config.param_dtype
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} layout, ZeRO stage {args.stage}", "psi": psi_total,
                   "psi_padded": pp, "buckets": nb, "bucket_cap_elems": args.cap, "align_elems": args.align,
                   "param_dtype": args.dtype, "loss_scale": "dynamic, S0 = 2^16" if args.dtype == "fp16" else "static 1",
                   "adam_state_dtype": "fp32", "reduce_mode": cfg.reduce_mode,
                   "transport": transport, "transport_verified": verified, "parallelism": f"zero{args.stage}-dp{world}",
                   "same_device_ranks": bool(same_dev and world > 1),
                   "l2": l2_note},
        "roofline": {"bound": "hbm", "kernel": "k_adam (fused partitioned Adam + recast)",
                     "achieved": adam_gbs, "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": adam_gbs / hbm_peak if adam_gbs else None, "traffic": traffic,
                     "bytes_per_launch": adam_bytes, "ms_per_launch": adam_ms,
                     "share_of_step": adam_ms / ms if adam_ms else None,
                     "events": res["phase_events"],
                     "note": None if adam_ms else "--graph: per-kernel events are not recorded inside the graph"},
        "step_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                          "hbm_gbs": hbm_peak, "nvlink_gbs": NVLINK_GBS if N > 1 else None,
                          "frac_at_spec_hbm_8tbs": t_roof_at(8000.0, NVLINK_NOMINAL_GBS) * 1e3 / ms,
                          "reduce_phase_ms": reduce_ms, "flatten_gbs": 4 * pp / (reduce_ms * 1e-3) / 1e9
                          if (N == 1 and reduce_ms) else None},
        "comm": comm,
        "stage3_phases": res["phases"],
        "cuda_graph": res["graph"],
        "clocks": res["clocks"],
        "gpu_launches": int(res["launches"]),
    }
    if nccl_log:
        line["nccl_info"] = nccl_info_summary(nccl_log + ".*.log", world)

    # e2e through the public API with HOST buffers: H2D of the step's gradients from
    # pinned memory + the step + D2H of the step record, every step
    if not args.no_e2e:
        # the buffers first, then every rank agrees: a rank that cannot pin its host copy
        # (e.g. host memory exhausted by N ranks) must not leave the others inside a step
        try:
            host = torch.empty(grad_buf.numel(), dtype=grad_buf.dtype, pin_memory=True)
            spare = torch.empty_like(grad_buf)
            ok, why = 1, None
        except RuntimeError as exc:
            host = spare = None
            ok, why = 0, str(exc)
        if min_over_ranks(ok, dev) == 1:
            line["e2e"] = run_e2e(args, eng, make_step(eng), grad_buf, grads, host, spare, tensors, stream, dev,
                                  psi_total, ms, barrier)
        else:
            line["e2e"] = {"value": None, "unit": "Gparams/s", "note": f"not measured: {why or 'a peer rank could not allocate its buffers'}"}
        del host, spare

    # the same layout in fp16 with dynamic loss scaling (the paper's precision)
    if args.dtype == "bf16" and not args.no_fp16_key and not args.graph:
        eng.destroy()
        del eng, grad_buf, grads
        gc.collect()
        torch.cuda.empty_cache()
        e16, c16, gb16, g16 = build("fp16")
        r16 = timed(e16, args.steps, sample_clocks=False)
        _, a16_ms, a16_gbs = adam_roofline(r16["tm"])
        line["fp16_dynamic"] = {
            "value": psi_total / (r16["ms"] * 1e-3) / 1e9, "unit": "Gparams/s", "ms_per_step": r16["ms"],
            "loss_scale": "dynamic (S0 = 2^16, x2 per 1000 good steps, x1/2 on overflow)",
            "loss_scale_last": r16["rec"].loss_scale, "overflow_last": r16["rec"].overflow, "t_last": r16["rec"].t,
            "step_roofline_frac": t_roof * 1e3 / r16["ms"],
            "adam_gbs": a16_gbs, "adam_frac": a16_gbs / hbm_peak if a16_gbs else None,
            "gpu_launches": int(r16["launches"])}
        assert r16["rec"].overflow == 0 and r16["rec"].loss_scale == 2.0 ** 16, "fp16 run overflowed"
        e16.destroy()
        del e16, gb16, g16

    if rank == 0 and not args.no_cpu_baseline:
        v, desc, n, dt = oracle_sample_run(tensors, args.dtype, args.seed, 2, 0, args.cpu_budget_s)
        line["cpu_baseline"] = {"value": v, "unit": "Gparams/s", "cores": 1, "kind": "oracle", "sample": desc}
        procs = len(os.sched_getaffinity(0))
        if procs > 1 and not args.no_cpu_parallel and world == 1:
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


def run_e2e(args, eng, one_step, grad_buf, grads, host, spare, tensors, stream, dev, psi_total, ms, barrier):
    """Every step copies that step's gradients H2D from pinned host memory and reads the
    step record D2H.  The copy of step s+1 (copy stream, second device buffer) overlaps
    step s; the host reads step s's record before issuing step s+2."""
    import torch
    import synth
    host.copy_(grad_buf)
    bufs = [grad_buf, spare]
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
        one_step()                              # the whole step; its 32-byte record lands in pinned memory
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
    del bufs
    nbytes = int(grad_buf.numel() * grad_buf.element_size())
    return {"value": psi_total / (e2e_ms * 1e-3) / 1e9, "unit": "Gparams/s",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 32, "ms_per_step": e2e_ms, "steps": K,
            "device_ms_per_step": e2e_dev_ms, "h2d_alone_ms": h2d_ms,
            "h2d_gbs": nbytes / (h2d_ms * 1e-3) / 1e9,
            "frac_of_h2d_bound": max(h2d_ms, ms) / e2e_ms,
            "note": "value from the host wall clock (device_ms_per_step: CUDA events from the first H2D "
                    "to the last step's end); H2D of step s+1 overlaps step s (double-buffered)"}


if __name__ == "__main__":
    main()
