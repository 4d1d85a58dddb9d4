"""P_a / P_a+cpu: partitioned activation checkpoints (oracle, test infrastructure).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module;
it shares no code with the CUDA path.

What the paper fixes (§6.1 "P_a: Partitioned Activation Checkpointing",
P:406-419, and §8 "Communication Analysis of ZeRO-R"):
  * "once the forward propagation for a layer of a model is computed, the input
    activations are partitioned across all the model parallel process, until it is
    needed again during the backprogation. At this point, ZeRO uses an all-gather
    operation to re-materialize a replicated copy of the activations";
  * it "works in conjunction with activation checkpointing ... storing partitioned
    activation checkpoints only instead of replicated copies";
  * P_a+cpu offloads the partitioned checkpoints to host memory;
  * memory: the activation footprint shrinks "by a factor proportional to the MP
    degree";
  * communication: Megatron moves 12 x seq x hidden per transformer block (two
    all-reduces forward, two in the recompute, two backward; an all-reduce is
    2 x message) and P_a adds one all-gather of seq x hidden per block, "less than
    10%"; P_a+cpu adds 2x data movement to and from CPU memory.

What it computes is therefore the identity on the checkpointed activation: the
all-gather of the N_m partitions is, element for element, the activation that was
saved (the partition only changes where the bytes live).  The oracle writes that out:
`partition` takes MP rank r's slice, `gather` concatenates the slices in rank order.

Partition shape (reading R-Pa1): the paper does not say how the
checkpoint is split.  Here the n = b*s*h elements of one checkpoint are padded to
n' = a multiple of N_m * 8 and rank r keeps the contiguous slice [r*n'/N_m,
(r+1)*n'/N_m) (8-element, i.e. 16-byte, granules for 16-bit data); padding is zero.

Pins (tests/test_oracle_activation.py): brute force over small sizes and every
N_m in 1..9 (each element in exactly one slice, in order; gather(partition(x)) == x
bitwise), the memory ratio N_m exactly, the 100B example of P:419 (reading R-Pa2),
and the 1/12 communication ratio of P:492.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

GRANULE = 8  # elements per 16-byte granule of 16-bit data (reading R-Pa1)


def padded_elems(n: int, n_m: int) -> int:
    """n rounded up to a multiple of N_m * 8 (reading R-Pa1)."""
    q = n_m * GRANULE
    return (n + q - 1) // q * q


def slice_bounds(n: int, n_m: int, r: int) -> tuple[int, int]:
    """[lo, hi) of MP rank r's slice in the padded index space."""
    s = padded_elems(n, n_m) // n_m
    return r * s, (r + 1) * s


def partition(x: np.ndarray, n_m: int, r: int) -> np.ndarray:
    """MP rank r's partition of the checkpoint x, zero-padded."""
    n = x.size
    lo, hi = slice_bounds(n, n_m, r)
    out = np.zeros(hi - lo, dtype=x.dtype)
    take = max(0, min(hi, n) - lo)
    out[:take] = x.reshape(-1)[lo:lo + take]
    return out


def gather(slices: list[np.ndarray], n: int) -> np.ndarray:
    """The all-gather that re-materializes the replicated checkpoint:
    the slices in rank order, cut back to the checkpoint's n elements."""
    return np.concatenate(slices)[:n]


def checkpoint_bytes(layers: int, batch: int, seq: int, hidden: int, n_m: int, elem_bytes: int = 2,
                     partitioned: bool = True) -> Fraction:
    """Per-GPU bytes of one checkpointed activation (the block input, b x s x h) per
    transformer layer; with P_a each MP rank keeps 1/N_m of it."""
    full = Fraction(layers * batch * seq * hidden * elem_bytes)
    return full / n_m if partitioned else full


def megatron_block_comm(seq: int, hidden: int, batch: int = 1) -> int:
    """Megatron-LM with activation checkpointing, per transformer block: 2 all-reduces
    forward + 2 in the recompute + 2 backward, each 2 x (b*s*h)."""
    return 6 * 2 * batch * seq * hidden


def pa_block_comm(seq: int, hidden: int, batch: int = 1) -> int:
    """P_a's extra all-gather of the block-input checkpoint before the recompute:
    message_size = b*s*h."""
    return batch * seq * hidden


def pa_cpu_extra_transfer(seq: int, hidden: int, batch: int = 1, n_m: int = 1) -> Fraction:
    """P_a+cpu: each MP rank's partition goes to host memory and back, 2 x its
    1/N_m share of the checkpoint per block ("2x added data movement")."""
    return Fraction(2 * batch * seq * hidden, n_m)
