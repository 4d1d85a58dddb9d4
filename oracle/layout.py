"""Partition / bucket layout (oracle, test infrastructure).

What it computes: where every element of every tensor lives in the padded flat
index space [0, Psi'), which gradient bucket it is reduced in, and which rank
owns it.

Paper: P:357 (§5.1) "we group the optimizer states into N_d equal partitions,
such that the i-th data parallel process only updates the optimizer states
corresponding to the i-th partition"; P:366 (§5.2) "we bucketize all the
gradients corresponding to a particular partition, and perform reduction on the
entire bucket at once"; P:420-422 (§6.2) constant-size fused buffer C_B;
P:306 parameters of a layer are needed together (buckets never span layers).
The concrete rule is reading c-7:

  Q = N*A, cap = floor(C_B/Q)*Q (C_B = 0 means unlimited; require C_B >= Q)
  walk tensors in forward order; a new bucket starts at every layer change and
  whenever the next A-aligned start has no room; a tensor that does not fit is
  split at cap; each bucket is padded to a multiple of Q; rank r owns the r-th
  1/N slice of every bucket.
  ZeRO x MP (reading R-MP1): an optional per-tensor group (1 = the
  tensor is replicated across the model-parallel group, 0 = MP-partitioned) also
  starts a new bucket when it changes, so no bucket mixes the two (a bucket's
  gradient-norm contribution is then either counted on every MP rank or only on
  MP rank 0).  With no groups the layout is unchanged.

Pins (tests/test_oracle_layout.py): SPEC make_layout examples (S:347-349:
(10,4) -> 12 with ranges [0,3),[3,6),[6,9),[9,12); (8,1) -> [0,8); (7,2) -> 8) as
the one-bucket A=1 case; brute-force properties on 10^3+ random cases (equal
partitions, every element placed exactly once, B_k = 0 mod Q, A-aligned starts,
split tensors contiguous, buckets inside one layer); SURVEY's config-1 table.
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence, Tuple


@dataclasses.dataclass
class Piece:
    tensor: int       # tensor index (forward order)
    tensor_off: int   # first element of the tensor covered by this piece
    bucket_off: int   # position inside the bucket
    count: int


@dataclasses.dataclass
class Bucket:
    layer: int
    group: int = 0    # R-MP1: 1 = MP-replicated tensors
    base: int = 0     # global flat offset
    size: int = 0     # B_k (padded, multiple of N*A)
    used: int = 0
    pieces: List[Piece] = dataclasses.field(default_factory=list)
    shard_off: int = 0  # local offset of this bucket's slice in every rank's shard


@dataclasses.dataclass
class Layout:
    n_d: int
    align: int
    cap: int
    buckets: List[Bucket]
    psi: int          # true parameter count
    psi_padded: int   # Psi'

    @property
    def shard(self) -> int:
        return self.psi_padded // self.n_d

    def owned_range(self, k: int, r: int) -> Tuple[int, int]:
        b = self.buckets[k]
        s = b.size // self.n_d
        return b.base + r * s, b.base + (r + 1) * s

    def tensor_flat_offsets(self, n_tensors: int) -> List[List[Tuple[int, int, int]]]:
        """per tensor: list of (tensor_off, flat_off, count)."""
        out: List[List[Tuple[int, int, int]]] = [[] for _ in range(n_tensors)]
        for b in self.buckets:
            for p in b.pieces:
                out[p.tensor].append((p.tensor_off, b.base + p.bucket_off, p.count))
        return out


def _align_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


def make_layout(numels: Sequence[int], layers: Sequence[int], n_d: int, align: int,
                bucket_cap: int, groups: Sequence[int] = None) -> Layout:
    if n_d < 1 or align < 1 or (align & (align - 1)) != 0:
        raise ValueError("n_d >= 1 and align a power of two required")
    Q = n_d * align
    if bucket_cap == 0:
        cap = None
    else:
        if bucket_cap < Q:
            raise ValueError("bucket_cap < N*A")
        cap = bucket_cap // Q * Q
    if any(layers[i] > layers[i + 1] for i in range(len(layers) - 1)):
        raise ValueError("layers must be non-decreasing")

    buckets: List[Bucket] = []
    cur = Bucket(layer=layers[0] if layers else 0)

    def close(b: Bucket):
        if b.used > 0:
            buckets.append(b)

    for t, (n, L) in enumerate(zip(numels, layers)):
        if n == 0:
            continue
        G = groups[t] if groups is not None else 0
        if cur.used > 0 and (L != cur.layer or G != cur.group):
            close(cur)
            cur = Bucket(layer=L, group=G)
        if cur.used == 0:
            cur.layer, cur.group = L, G
        rem, toff = n, 0
        while rem > 0:
            start = _align_up(cur.used, align)
            room = (cap - start) if cap is not None else rem
            if room <= 0:
                close(cur)
                cur = Bucket(layer=L, group=G)
                continue
            take = min(rem, room)
            cur.pieces.append(Piece(t, toff, start, take))
            cur.used = start + take
            rem -= take
            toff += take
            if rem > 0:
                close(cur)
                cur = Bucket(layer=L, group=G)
    close(cur)

    base = 0
    shard_off = 0
    for b in buckets:
        b.size = _align_up(b.used, Q)
        b.base = base
        b.shard_off = shard_off
        base += b.size
        shard_off += b.size // n_d
    return Layout(n_d=n_d, align=align, cap=cap or 0, buckets=buckets,
                  psi=sum(numels), psi_padded=base)
