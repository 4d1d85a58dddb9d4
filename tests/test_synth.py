"""The shared seeded input generator (synth/): known splitmix64 outputs, range,
determinism and the paper layouts' parameter counts."""
import numpy as np

import synth


def test_splitmix64_reference_values():
    # splitmix64 with state 0: first outputs of the reference generator (Vigna)
    assert synth.splitmix64_scalar(0) == 0xE220A8397B1DCDAF
    assert synth.splitmix64_scalar(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4
    v = synth._splitmix64_vec(np.array([0, 0x9E3779B97F4A7C15], np.uint64))
    assert v.tolist() == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]


def test_uniform_range_and_determinism():
    k = synth.stream_key(1, synth.KIND_GRAD, 3, 2)
    a = synth.uniform_pm1(k, 100, 100000)
    b = synth.uniform_pm1(k, 100, 100000)
    assert np.array_equal(a, b) and a.dtype == np.float32
    assert a.min() >= -1.0 and a.max() < 1.0
    assert abs(float(a.mean())) < 0.01
    # sub-ranges are consistent (counter-based: element i depends only on i)
    assert np.array_equal(synth.uniform_pm1(k, 150, 10), a[50:60])
    assert not np.array_equal(synth.uniform_pm1(synth.stream_key(7, 1, 3, 2), 100, 100), a[:100])
    # exact 24-bit grid
    assert np.all((a * 2 ** 23) == np.round(a * 2 ** 23))


def test_layout_counts():
    assert synth.psi(synth.mlp_layout()) == 1_000_000
    assert synth.psi(synth.gpt2_1p5b()) == 1_557_611_200
    assert synth.psi(synth.gpt_7p5b()) == 7_500_000_000
    assert synth.psi(synth.gpt_60b()) == 60_826_075_136
    assert len(synth.gpt2_1p5b()) == 580 and len(synth.gpt_60b()) == 904
