"""Exhaustive pin of the CUDA recast (reading c-5; SURVEY c-9 "all 2^32 fp32
patterns"): every fp32 bit pattern is loaded as an fp32 master through
zero_load_master, whose kernel writes the 16-bit parameter with the same
cvt.rn routine the fused Adam uses; the 2^32 results must equal the oracle's
conversion bit for bit (NaN inputs: the output must be a NaN)."""
import os

import numpy as np
import pytest
import torch

from oracle import numerics as nx

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)
if os.environ.get("ZERO_SLOW_TESTS") != "1":   # ~6 min (the oracle converts 2 x 2^32 values)
    pytest.skip("exhaustive cast pin: set ZERO_SLOW_TESTS=1 (run log in profiles/r01_exhaustive_cast.txt)",
                allow_module_level=True)


@pytest.mark.parametrize("dt", ["bf16", "fp16"])
def test_all_fp32_patterns(dt):
    from paper_1910_02054_b200 import ZeroConfig, ZeroEngine
    torch.cuda.empty_cache()
    n = 1 << 32
    eng = ZeroEngine([n], [0], 1, 0, 1, ZeroConfig.defaults(dt), "local", align=64, bucket_cap=1 << 26)
    pats = torch.arange(-(1 << 31), 1 << 31, dtype=torch.int32, device="cuda").view(torch.float32)
    eng.load_master([pats])
    torch.cuda.synchronize()
    del pats
    out = eng.p16_arena()          # flat replica; the single tensor starts at 0
    ch = 1 << 28
    for start in range(0, n, ch):
        # patterns in the same order as the GPU tensor: int32 -2^31 .. 2^31-1 as bits
        bits = (np.arange(start, start + ch, dtype=np.int64) - (1 << 31)).astype(np.int32).view(np.uint32)
        x = bits.view(np.float32)
        want = nx.to16(x, dt)
        got = out[start:start + ch].cpu().view(torch.int16).numpy().view(np.uint16)
        nan = np.isnan(x)
        assert np.array_equal(got[~nan], want[~nan]), f"chunk {start}"
        assert np.all(np.isnan(nx.widen(got[nan], dt)))
    eng.destroy()
    del out
    torch.cuda.empty_cache()
