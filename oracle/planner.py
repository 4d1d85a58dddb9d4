"""Analytic model-state memory and communication volume (oracle, test infrastructure).

Memory (Fig. 1 caption, §3.1, §5.1, §5.2, §5.3):
  K = 12 for mixed-precision Adam;
  baseline DP        (2 + 2 + K) Psi
  P_os   (stage 1)   (2 + 2) Psi + K Psi / N_d          ("4Psi + K Psi/N_d")
  P_os+g (stage 2)   2 Psi + (2 + K) Psi / N_d          ("2Psi + 14Psi/N_d")
  P_os+g+p (stage 3) (2 + 2 + K) Psi / N_d              ("16Psi/N_d")
Max model size (Table 2): the largest Psi whose model states fit the
device memory M when additionally divided by the MP degree N_m.
Communication (§7): per-rank elements sent per step; the paper's
2Psi / 2Psi / 3Psi are the N -> infinity limits of the exact ring counts
(reading c-8 #12):  RS sends len (N-1)/N, AG sends chunk (N-1).

All arithmetic is exact (Python ints / Fractions); GB = 10^9 bytes.

Pins (tests/test_oracle_planner.py): all 54 printed Table 1 values
under the printing reading c-8 #13, the Fig. 1 example (P:38, P:360, P:370,
P:397), §3.1's 24 GB / 3 GB, §1's 16 TB / "16GB", the 20
Table 2 values (reading c-8 #14), SPEC's desk-scale bytes,
SPEC's volume examples and the 1.5x ratio.
"""
from __future__ import annotations

from fractions import Fraction

GB = 10 ** 9
STAGE_DP, STAGE_OS, STAGE_OSG, STAGE_OSGP = 0, 1, 2, 3


def model_state_bytes(psi: int, K: int, n_d: int, stage: int) -> Fraction:
    """Per-device model-state bytes (exact)."""
    psi = Fraction(psi)
    if stage == STAGE_DP:
        return (2 + 2 + K) * psi
    if stage == STAGE_OS:
        return 4 * psi + K * psi / n_d
    if stage == STAGE_OSG:
        return 2 * psi + (2 + K) * psi / n_d
    if stage == STAGE_OSGP:
        return (2 + 2 + K) * psi / n_d
    raise ValueError(stage)


def model_state_breakdown(psi: int, K: int, n_d: int, stage: int) -> dict:
    """bytes per category {params16, grads16, optimizer} (exact Fractions)."""
    psi = Fraction(psi)
    p16 = 2 * psi / n_d if stage >= STAGE_OSGP else 2 * psi
    g16 = 2 * psi / n_d if stage >= STAGE_OSG else 2 * psi
    opt = K * psi / n_d if stage >= STAGE_OS else K * psi
    return {"params16": p16, "grads16": g16, "optimizer": opt}


def bytes_per_param(K: int, n_d: int, stage: int) -> Fraction:
    return model_state_bytes(1, K, n_d, stage)


def max_model_size(stage: int, n_d: int, n_m: int, device_bytes: int, K: int = 12) -> Fraction:
    """Table 2 left half: Psi_max = device_bytes * N_m / bytes_per_param."""
    return Fraction(device_bytes) * n_m / bytes_per_param(K, n_d, stage)


# ---- communication volume -------------------------------------------------

def rs_sent(length: int, n: int) -> Fraction:
    """reduce-scatter: elements sent per rank (ring/pipelined)."""
    return Fraction(length * (n - 1), n)


def ag_sent(chunk: int, n: int) -> int:
    """all-gather: elements sent per rank."""
    return chunk * (n - 1)


def ar_sent(length: int, n: int) -> Fraction:
    """all-reduce = reduce-scatter + all-gather."""
    return rs_sent(length, n) + ag_sent(Fraction(length, n), n)


def step_elems_per_rank(psi_padded: int, n_d: int, stage: int) -> Fraction:
    """Elements each rank sends in one step.

    stages 0/1/2: RS Psi'(N-1)/N + AG Psi'(N-1)/N
    stage 3:      RS + AG forward + AG backward = 3Psi'(N-1)/N"""
    one = Fraction(psi_padded * (n_d - 1), n_d)
    if stage in (STAGE_DP, STAGE_OS, STAGE_OSG):
        return 2 * one
    if stage == STAGE_OSGP:
        return 3 * one
    raise ValueError(stage)


def paper_volume(psi: int, stage: int) -> int:
    """The paper's asymptotic per-step volume: 2 Psi (DP, P_os, P_os+g), 3 Psi (P_os+g+p)."""
    return 3 * psi if stage == STAGE_OSGP else 2 * psi


def temp_buffer_bytes(psi: int, fused_fp32: bool = True, cb_limit=None) -> int:
    """§3.2 / §6.2: a Psi-sized fused fp32 buffer is 4 Psi bytes;
    C_B caps it at a constant."""
    full = 4 * psi if fused_fp32 else 2 * psi
    return full if cb_limit is None else min(full, cb_limit)
