"""16-bit number formats used by mixed-precision training (oracle, test infrastructure).

P:264-266 (§3.1 "Mixed-Precision Training"): parameters and gradients are held in
16-bit, the optimizer keeps fp32 copies.  The paper uses fp16; bf16 is the B200
default (reading R-dtype).  Reading c-5: conversions
fp32 -> 16-bit are IEEE round-to-nearest-even; overflow goes to +-inf;
subnormals per IEEE; NaN stays NaN (payload/sign of a NaN is not compared).

Implementation:
* fp16: numpy's float32 -> float16 cast (a library primitive; IEEE RTNE).
* bf16: written out from the definition of RTNE on the top 16 bits of the
  fp32 pattern:  (bits + 0x7FFF + ((bits >> 16) & 1)) >> 16, NaN -> quiet NaN.
* widening 16 -> 32 is exact for both formats.

Pins (tests/test_oracle_numerics.py): SPEC examples 0 -> 0x0000, 1.0 -> 0x3C00,
65520 -> 0x7C00; the round-trip bound |f16(x)-x| <= 2^-10|x| + 6e-8
(S:69); exhaustive agreement with torch's CPU conversions (an independent
library routine) over all 2^16 patterns and >= 4M fp32 patterns incl. every
rounding tie; widening exactness for all 2^16 patterns.
"""
from __future__ import annotations

import numpy as np

FP16 = "fp16"
BF16 = "bf16"


def f32_to_f16_bits(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        return x.astype(np.float16).view(np.uint16)


def f16_bits_to_f32(h) -> np.ndarray:
    return np.asarray(h, dtype=np.uint16).view(np.float16).astype(np.float32)


def f32_to_bf16_bits(x) -> np.ndarray:
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16))
    out = rounded.astype(np.uint16)  # carry into the exponent is the correct overflow to inf
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    if nan.any():
        out = np.where(nan, ((b >> np.uint64(16)).astype(np.uint16) | np.uint16(0x0040)), out)
    return out.astype(np.uint16)


def bf16_bits_to_f32(h) -> np.ndarray:
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def to16(x, dtype: str) -> np.ndarray:
    """RTNE16(x): fp32 array -> 16-bit patterns (uint16)."""
    if dtype == FP16:
        return f32_to_f16_bits(x)
    if dtype == BF16:
        return f32_to_bf16_bits(x)
    raise ValueError(dtype)


def widen(h, dtype: str) -> np.ndarray:
    """16-bit patterns -> exact fp32 values."""
    if dtype == FP16:
        return f16_bits_to_f32(h)
    if dtype == BF16:
        return bf16_bits_to_f32(h)
    raise ValueError(dtype)


def ulp16_distance(a, b) -> np.ndarray:
    """Distance in units of last place between 16-bit patterns (sign-magnitude
    mapped to ordered integers), used for the "1 ulp" tolerance (c-6)."""
    def ordered(h):
        h = np.asarray(h, dtype=np.uint16).astype(np.int32)
        return np.where(h & 0x8000, -(h & 0x7FFF), h)
    return np.abs(ordered(a) - ordered(b))
