"""Pins for oracle/numerics.py (reading c-5): SPEC examples, the round-trip bound
and exhaustive agreement with torch's CPU conversions (an independent library)."""
import numpy as np
import pytest
import torch

from oracle import numerics as nx


def _torch16(x32: np.ndarray, dtype) -> np.ndarray:
    return torch.from_numpy(x32).to(dtype).view(torch.int16).numpy().view(np.uint16)


def _tie_patterns(dt: str) -> np.ndarray:
    """fp32 values exactly halfway between consecutive 16-bit values, and the
    fp32 neighbours of each halfway point (every rounding decision boundary)."""
    h = np.arange(0, 0x7C00 if dt == "fp16" else 0x7F80, dtype=np.uint32)
    lo = nx.widen(h.astype(np.uint16), dt).astype(np.float64)
    hi = nx.widen((h + 1).astype(np.uint16), dt).astype(np.float64)
    if dt == "fp16":
        hi[-1] = 65536.0  # next value above 65504 if the exponent continued
    else:
        hi[-1] = float(np.float64(2.0) ** 128)
    mid = ((lo + hi) / 2).astype(np.float32)   # exact: halfway points fit fp32
    bits = mid.view(np.uint32)
    cand = np.concatenate([bits, bits - 1, bits + 1])
    cand = cand[(cand.view(np.float32) >= 0) & np.isfinite(cand.view(np.float32))]
    allp = np.concatenate([cand, cand | np.uint32(0x80000000)])
    return allp.view(np.float32)


def test_spec_examples_fp16():
    # 0 -> 0x0000, 1.0 -> 0x3C00, 65520 -> +inf (0x7C00)
    out = nx.f32_to_f16_bits(np.array([0.0, 1.0, 65520.0, 65519.0, -65520.0], np.float32))
    assert list(out) == [0x0000, 0x3C00, 0x7C00, 0x7BFF, 0xFC00]
    assert nx.f16_bits_to_f32(np.array([0x3C00, 0x0000], np.uint16)).tolist() == [1.0, 0.0]


def test_roundtrip_bound_fp16():
    # S:69 bound |f16(x) - x| <= 2^-10 |x| + 6e-8 (sampled inside the finite fp16 range)
    rng = np.random.default_rng(0)
    x = rng.uniform(-6.0e4, 6.0e4, 10000).astype(np.float32)
    x = np.concatenate([x, rng.uniform(-1e-4, 1e-4, 10000).astype(np.float32)])
    back = nx.f16_bits_to_f32(nx.f32_to_f16_bits(x)).astype(np.float64)
    assert np.all(np.abs(back - x) <= 2.0 ** -10 * np.abs(x.astype(np.float64)) + 6e-8)


@pytest.mark.parametrize("dt,tdt", [("fp16", torch.float16), ("bf16", torch.bfloat16)])
def test_widen_exact_all_patterns(dt, tdt):
    h = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
    w = nx.widen(h, dt)
    ref = torch.from_numpy(h.view(np.int16)).view(tdt).to(torch.float32).numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(w), nan)
    assert np.array_equal(w[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    # narrowing a widened value is the identity (widening is exact)
    assert np.array_equal(nx.to16(w[~nan], dt), h[~nan])


@pytest.mark.parametrize("dt,tdt", [("fp16", torch.float16), ("bf16", torch.bfloat16)])
def test_narrow_matches_torch_ties_and_random(dt, tdt):
    x = _tie_patterns(dt)
    rng = np.random.default_rng(1)
    rnd = rng.integers(0, 1 << 32, size=4_000_000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    specials = np.array([np.inf, -np.inf, 0.0, -0.0, np.nan, 3.4028235e38, -3.4028235e38,
                         1e-45, -1e-45, 5.96e-8, 2.98e-8, 65504.0, 65519.99, 65520.0], np.float32)
    x = np.concatenate([x, rnd, specials])
    mine = nx.to16(x, dt)
    ref = _torch16(x, tdt)
    nan = np.isnan(x)
    assert np.array_equal(mine[~nan], ref[~nan])
    assert np.all(np.isnan(nx.widen(mine[nan], dt)))


def test_ulp_distance():
    a = np.array([0x3C00, 0x0001, 0x8001, 0x7BFF], np.uint16)
    b = np.array([0x3C01, 0x8001, 0x0001, 0x7C00], np.uint16)
    assert list(nx.ulp16_distance(a, b)) == [1, 2, 2, 1]
