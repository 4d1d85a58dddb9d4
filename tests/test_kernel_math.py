"""CPU check of the integer arithmetic the flatten epilogue uses to form b^2 from a
16-bit pattern b (csrc/kernels.cu, epi_elem<.., 2>): rebiasing the exponent field into
an fp64 bit pattern gives the exact value of every normal fp16 / bf16 number, and
2r - min_normal the exact value of every subnormal and of zero -- checked against
numpy's / torch's own widening over all 2^15 non-negative patterns of each format."""
import numpy as np
import torch


def _rebias(x, shift, bias_delta):
    hi = (x.astype(np.uint64) << np.uint64(shift)) + np.uint64(bias_delta << 20)
    return (hi << np.uint64(32)).view(np.float64)


def test_fp16_rebias_exact():
    x = np.arange(0x7C00, dtype=np.uint64)                 # every finite non-negative fp16
    r = _rebias(x, 10, 1008)
    d = np.where(x < 0x400, 2.0 * r - 2.0 ** -14, r)
    want = x.astype(np.uint16).view(np.float16).astype(np.float64)
    assert np.array_equal(d, want)


def test_bf16_rebias_exact():
    x = np.arange(0x7F80, dtype=np.uint64)                 # every finite non-negative bf16
    r = _rebias(x, 13, 896)
    d = np.where(x < 0x80, 2.0 * r - 2.0 ** -126, r)
    want = torch.from_numpy(x.astype(np.int16)).view(torch.bfloat16).double().numpy()
    assert np.array_equal(d, want)
