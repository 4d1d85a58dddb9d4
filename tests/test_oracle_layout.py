"""Pins for oracle/layout.py (reading c-7; P:357 equal partitions, P:366 buckets,
P:420-422 constant-size buffers): SPEC make_layout examples, SURVEY's config-1
table, and brute-force structural properties on random layouts."""
import random

import numpy as np
import pytest

import synth
from oracle import layout as L


def _owned(lay, r):
    return [lay.owned_range(k, r) for k in range(len(lay.buckets))]


@pytest.mark.parametrize("psi,n,padded,ranges", [
    (10, 4, 12, [(0, 3), (3, 6), (6, 9), (9, 12)]),
    (8, 1, 8, [(0, 8)]),
    (7, 2, 8, [(0, 4), (4, 8)]),
])
def test_spec_make_layout(psi, n, padded, ranges):
    lay = L.make_layout([psi], [0], n, 1, 0)            # one bucket, A = 1
    assert lay.psi_padded == padded
    assert [_owned(lay, r)[0] for r in range(n)] == ranges


def test_config1_table(golden):
    g = golden("layout_config1.json")
    ts = synth.mlp_layout()
    lay = L.make_layout([t.numel for t in ts], [t.layer for t in ts], g["n_d"], g["align"], g["cap"])
    assert lay.psi == g["psi"] and lay.psi_padded == g["psi_padded"] and lay.shard == g["shard"]
    got = [[b.layer, b.base, b.size, [[p.tensor, p.tensor_off, p.bucket_off, p.count] for p in b.pieces]]
           for b in lay.buckets]
    assert got == g["buckets"]


def _check_properties(numels, layers, n, a, cb, groups=None):
    lay = L.make_layout(numels, layers, n, a, cb, groups)
    Q = n * a
    psi = sum(numels)
    cover = np.zeros(lay.psi_padded, np.int32)
    seen = [0] * len(numels)
    prev_end = {}
    for k, b in enumerate(lay.buckets):
        assert b.size % Q == 0 and b.size > 0
        if cb:
            assert b.size <= cb // Q * Q
        assert all(layers[p.tensor] == b.layer for p in b.pieces)       # never spans layers
        if groups is not None:                                            # R-MP1: never mixes groups
            assert all(groups[p.tensor] == b.group for p in b.pieces)
        for p in b.pieces:
            assert p.bucket_off % a == 0                                  # A-aligned starts
            assert p.bucket_off + p.count <= b.size
            flat = b.base + p.bucket_off
            cover[flat:flat + p.count] += 1
            assert p.tensor_off == seen[p.tensor]                         # tensor order kept
            if p.tensor in prev_end:                                      # split tensors contiguous
                assert prev_end[p.tensor] == flat
            prev_end[p.tensor] = flat + p.count
            seen[p.tensor] += p.count
    assert seen == list(numels)                                           # every element placed once
    assert cover.max(initial=0) <= 1 and int(cover.sum()) == psi
    assert lay.psi_padded == sum(b.size for b in lay.buckets)
    # equal partitions: each rank owns exactly Psi'/N and the ranges tile [0, Psi')
    own = np.zeros(lay.psi_padded, np.int32)
    for r in range(n):
        tot = 0
        for lo, hi in _owned(lay, r):
            own[lo:hi] += 1
            tot += hi - lo
        assert tot == lay.psi_padded // n
    assert np.all(own == 1)
    # shard offsets are the prefix sums of B_k / N
    acc = 0
    for b in lay.buckets:
        assert b.shard_off == acc
        acc += b.size // n
    # bases are increasing and contiguous
    for k in range(1, len(lay.buckets)):
        assert lay.buckets[k].base == lay.buckets[k - 1].base + lay.buckets[k - 1].size
    return lay


def test_random_layout_properties():
    rnd = random.Random(1234)
    for _ in range(1500):
        nt = rnd.randint(1, 12)
        numels = [rnd.choice([0, 1, 2, 3, 7, 63, 64, 65, 100, 257, 1000, 4096]) if rnd.random() < 0.5
                  else rnd.randint(1, 3000) for _ in range(nt)]
        if sum(numels) == 0:
            numels[0] = 5
        layers, L_ = [], 0
        for _t in range(nt):
            if rnd.random() < 0.3:
                L_ += 1
            layers.append(L_)
        n = rnd.choice([1, 2, 3, 4, 8])
        a = rnd.choice([1, 2, 4, 64])
        Q = n * a
        cb = rnd.choice([0, Q, 7 * Q, rnd.randint(Q, 40 * Q), 100000])
        _check_properties(numels, layers, n, a, cb)


def test_cap_below_q_rejected():
    with pytest.raises(ValueError):
        L.make_layout([100], [0], 4, 64, 255)


def test_paper_layouts_counts():
    # SURVEY §8 table (computed with the same rule at A = 64): tensors, Psi', buckets, shard
    cases = [("gpt2_1.5b", 8, 580, 1557621248, 51, 194702656),
             ("gpt_7.5b", 8, 724, 7500023296, 123, 937502912),
             ("gpt_60b", 8, 904, 60826075136, 983, 7603259392)]
    for name, n, nt, pp, nb, shard in cases:
        ts = synth.CONFIGS[name]()
        lay = L.make_layout([t.numel for t in ts], [t.layer for t in ts], n, 64, 1 << 26)
        assert (len(ts), lay.psi_padded, len(lay.buckets), lay.shard) == (nt, pp, nb, shard)


def test_mp_groups_split_like_layers():
    """Reading R-MP1: a change of MP group (replicated vs partitioned tensor) closes a
    bucket exactly as a layer change does, so the grouped layout equals the plain
    layout of the same tensors with every maximal same-(layer, group) run given its
    own layer id; all-zero groups change nothing."""
    rnd = random.Random(99)
    for _ in range(800):
        nt = rnd.randint(1, 14)
        numels = [rnd.choice([0, 1, 5, 64, 65, 300]) if rnd.random() < 0.4 else rnd.randint(1, 2000)
                  for _ in range(nt)]
        if sum(numels) == 0:
            numels[0] = 3
        layers, L_ = [], 0
        for _t in range(nt):
            if rnd.random() < 0.25:
                L_ += 1
            layers.append(L_)
        groups = [rnd.randint(0, 1) for _ in range(nt)]
        n = rnd.choice([1, 2, 4, 8])
        a = rnd.choice([1, 8, 64])
        Q = n * a
        cb = rnd.choice([0, Q, 5 * Q, rnd.randint(Q, 30 * Q)])
        lay = _check_properties(numels, layers, n, a, cb, groups)
        # relabel: a new pseudo-layer at every (layer, group) change among non-empty tensors
        pseudo, cur, key = [], -1, None
        for t in range(nt):
            k = (layers[t], groups[t])
            if numels[t] > 0 and k != key:
                cur, key = cur + 1, k
            pseudo.append(max(cur, 0))
        ref = L.make_layout(numels, pseudo, n, a, cb)
        assert [(b.base, b.size, [(p.tensor, p.tensor_off, p.bucket_off, p.count) for p in b.pieces])
                for b in lay.buckets] == [(b.base, b.size, [(p.tensor, p.tensor_off, p.bucket_off, p.count)
                                                            for p in b.pieces]) for b in ref.buckets]
        plain = L.make_layout(numels, layers, n, a, cb)
        zero = L.make_layout(numels, layers, n, a, cb, [0] * nt)
        assert [(b.base, b.size, b.layer) for b in plain.buckets] == [(b.base, b.size, b.layer) for b in zero.buckets]
