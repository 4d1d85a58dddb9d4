"""P_a / P_a+cpu on the GPU through the C ABI (zero_pa_*), against oracle/activation.py:
the re-materialized checkpoint must equal the saved one bit for bit (the oracle's
gather of the oracle's partitions), for every MP degree, ragged sizes, both dtypes,
device and host (P_a+cpu) stores, the layer order of a backward pass, and the
torch recompute path (gradients bit-equal to torch.utils.checkpoint)."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import activation as OA

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1910_02054_b200.activation import PaContext, PaSimGroup, partitioned_checkpoint  # noqa: E402
from paper_1910_02054_b200.zero import ZeroError  # noqa: E402


def _payload(numel, seed, dtype):
    """Seeded 16-bit patterns (any bits, including NaN/inf encodings: the path is a copy)."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 1 << 16, size=numel, dtype=np.uint16)
    t = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16 if dtype == "bf16" else torch.float16)
    return bits, t


def _bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("offload", [False, True])
@pytest.mark.parametrize("n_m", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("numel", [1, 7, 8 * 24 + 5, 100_003])
def test_round_trip_matches_oracle(n_m, numel, offload):
    dt = "bf16" if numel % 2 else "fp16"
    g = PaSimGroup(n_m, 1, numel, dt, offload)
    bits, act = _payload(numel, numel * 10 + n_m, dt)
    g.save(0, act)
    g.prefetch(0)
    expect = OA.gather([OA.partition(bits, n_m, r) for r in range(n_m)], numel)
    assert np.array_equal(expect, bits)
    for r in range(n_m):   # every MP rank re-materializes the same replicated copy
        out = g.gather(0, rank=r)
        torch.cuda.synchronize()
        assert np.array_equal(_bits(out), expect), r
    info = g[0].info
    assert info.padded == OA.padded_elems(numel, n_m) and info.slice * n_m == info.padded
    for r in range(n_m):
        c = g[r].counters()
        lo, hi = OA.slice_bounds(numel, n_m, r)
        mine = max(0, min(hi, numel) - lo)
        assert c.saved_elems == mine
        assert c.gathered_elems == numel - mine
        if offload:
            assert c.d2h_bytes == 2 * mine and c.h2d_bytes == 2 * info.slice
        else:
            assert c.d2h_bytes == 0 and c.h2d_bytes == 0
    g.destroy()


@pytest.mark.parametrize("offload", [False, True])
def test_backward_layer_order(offload):
    """Forward saves layers 0..L-1; backward prefetches/gathers L-1..0."""
    L, numel, n_m = 6, 3 * 1024 + 40, 4
    g = PaSimGroup(n_m, L, numel, "bf16", offload)
    acts = [_payload(numel, 100 + l, "bf16") for l in range(L)]
    for l in range(L):
        g.save(l, acts[l][1])
    for l in reversed(range(L)):
        g.prefetch(l)
        out = g.gather(l, rank=l % n_m)
        torch.cuda.synchronize()
        assert np.array_equal(_bits(out), acts[l][0]), l
    g.destroy()


def test_call_order_errors():
    g = PaSimGroup(2, 2, 64, "bf16", offload=True)
    with pytest.raises(ZeroError, match="ESTATE"):
        g[0].prefetch(0)                      # never saved
    _, act = _payload(64, 1, "bf16")
    g.save(0, act)
    g[0].prefetch(0)
    with pytest.raises(ZeroError, match="ESTATE"):
        g.gather(0)                           # rank 1 has not prefetched
    g[1].prefetch(0)
    g.gather(0)
    with pytest.raises(ZeroError, match="EINVAL"):
        g[0].save(2, act)                     # layer out of range
    g.destroy()
    h = PaSimGroup(2, 1, 64, "bf16", offload=False)
    h[0].save(0, act)
    with pytest.raises(ZeroError, match="ESTATE"):
        h.gather(0)                           # rank 1 has not saved
    h.destroy()


def test_gpt2_checkpoint_shape_full_size():
    """GPT-2 1.5B block input (batch 8 x seq 1024 x hidden 1600) at N_m = 4:
    every element of every layer round-trips (compared on the device)."""
    numel, L, n_m = 8 * 1024 * 1600, 4, 4
    for offload in (False, True):
        g = PaSimGroup(n_m, L, numel, "bf16", offload)
        gen = torch.Generator(device="cuda").manual_seed(7)
        acts = [torch.randint(-32768, 32767, (numel,), generator=gen, device="cuda", dtype=torch.int16)
                .view(torch.bfloat16) for _ in range(L)]
        for l in range(L):
            g.save(l, acts[l])
        for l in reversed(range(L)):
            g.prefetch(l)
            out = g.gather(l, rank=3)
            assert torch.equal(out.view(torch.int16), acts[l].view(torch.int16)), (offload, l)
        assert g[0].info.device_bytes == (numel // n_m * 2 if offload else L * numel // n_m * 2)
        g.destroy()


class _Block(torch.nn.Module):
    def __init__(self, h):
        super().__init__()
        self.ln = torch.nn.LayerNorm(h)
        self.fc = torch.nn.Linear(h, 4 * h)
        self.fc2 = torch.nn.Linear(4 * h, h)

    def forward(self, x):
        return x + self.fc2(torch.nn.functional.gelu(self.fc(self.ln(x))))


@pytest.mark.parametrize("n_m,offload", [(1, False), (2, False), (4, True), (3, False)])
def test_torch_recompute_matches_checkpoint(n_m, offload):
    """Gradients through partitioned checkpoints equal torch.utils.checkpoint's
    (use_reentrant=True) bit for bit: the recompute sees the identical input."""
    torch.manual_seed(0)
    h, b, s, L = 64, 2, 24, 3
    blocks = torch.nn.ModuleList([_Block(h) for _ in range(L)]).cuda().to(torch.bfloat16)
    x0 = torch.randn(b, s, h, device="cuda", dtype=torch.bfloat16)

    def run(use_pa):
        for p in blocks.parameters():
            p.grad = None
        x = x0.clone().requires_grad_(True)
        y = x
        pa = PaSimGroup(n_m, L, b * s * h, "bf16", offload) if use_pa else None
        for i, blk in enumerate(blocks):
            if use_pa:
                y = partitioned_checkpoint(blk, y, pa, i)
            else:
                y = torch.utils.checkpoint.checkpoint(blk, y, use_reentrant=True)
        y.float().square().sum().backward()
        grads = [x.grad.clone()] + [p.grad.clone() for p in blocks.parameters()]
        if pa is not None:
            pa.destroy()
        return y.detach(), grads

    y_ref, g_ref = run(False)
    y_pa, g_pa = run(True)
    assert torch.equal(y_ref, y_pa)
    for a, b_ in zip(g_ref, g_pa):
        assert torch.equal(a, b_)


@pytest.fixture(scope="module")
def comm():
    import torch.distributed as dist
    from paper_1910_02054_b200 import nccl_comm_ptr
    if not dist.is_initialized():
        sck = socket.socket()
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
        sck.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = torch.ones(1, device="cuda")
    dist.all_reduce(t)
    torch.cuda.synchronize()
    yield nccl_comm_ptr(dist.group.WORLD)
    torch.cuda.synchronize()
    dist.destroy_process_group()


@pytest.mark.parametrize("offload", [False, True])
def test_nccl_one_rank(comm, offload):
    """The NCCL transport's schedule (staging, in-place all-gather, copy out) on a
    1-rank communicator: an identity, so bit-exact."""
    numel, L = 5000 + 3, 3
    pa = PaContext(1, 0, L, numel, "fp16", offload, "nccl", comm)
    acts = [_payload(numel, 40 + l, "fp16") for l in range(L)]
    for l in range(L):
        pa.save(l, acts[l][1])
    for l in reversed(range(L)):
        pa.prefetch(l)
        out = pa.gather(l)
        torch.cuda.synchronize()
        assert np.array_equal(_bits(out), acts[l][0])
    pa.destroy()
