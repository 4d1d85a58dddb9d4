"""The NCCL transport's host path on one GPU: a 1-rank NCCL communicator borrowed
from torch keeps every collective call of the NCCL schedule (in-place reduce-
scatter / all-reduce per bucket on the library's comm stream, the C_B staging pool
with its events, the 16-byte decision all-gather, the per-bucket parameter
all-gather, stage 3's grouped layer gathers with prefetch and release events).
With one rank every collective is an identity, so the result must equal the
replicated-DP oracle bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run  # noqa: E402


@pytest.fixture(scope="module")
def comm():
    import torch.distributed as dist
    from paper_1910_02054_b200 import nccl_comm_ptr
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = torch.ones(1, device="cuda")
    dist.all_reduce(t)
    torch.cuda.synchronize()
    yield nccl_comm_ptr(dist.group.WORLD)
    torch.cuda.synchronize()
    dist.destroy_process_group()


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
@pytest.mark.parametrize("stage", [0, 1, 2, 3])
def test_nccl_one_rank_matches_oracle(comm, dt, stage):
    ts = synth.mlp_layout((300, 200, 100, 50))
    n_layers = max(t.layer for t in ts) + 1
    p = Pair(Run(ts, 1, stage, OS.AdamConfig.defaults(dt), cap=1 << 13,
                 inject=(2,), transport="nccl", nccl_comm=comm))
    e = p.engines[0]
    for s in range(5):
        oi, gi = p.step()
        p.compare_info(oi, gi)
        assert oi.overflow == (s == 2)
        if stage == 3:       # NCCL grouped layer gathers with prefetch, every step
            for order in (range(n_layers), reversed(range(n_layers))):
                for L in order:
                    views = e.gather_params(L)
                    for t, v in views.items():
                        assert np.array_equal(v.cpu().view(torch.int16).numpy().view(np.uint16), p.ost.p16[t])
                    e.release_params(L)
    p.compare()
    c = e.comm_counters()
    assert c.steps == 5
    p.destroy()
