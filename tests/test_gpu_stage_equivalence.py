"""SPEC acceptance criteria 6 and 11 on the GPU, through the C ABI:

 6. stage equivalence -- for N in {1, 2, 4, 8}, the 2-8-8-1 MLP, 50 steps, seeds {1, 7}:
    the fp32 masters and 16-bit parameters of P_os, P_os+g and P_os+g+p are bitwise
    equal to the replicated-DP baseline (stage 0) after EVERY step, and to the oracle
    at the end;
 11. C_B bound -- bucketed reduction with capacities {N*A (the smallest), 7*N*A, unlimited}
    gives identical results, and each run's counted volume is the closed form of its
    own padded Psi'.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import planner as P
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run, bits32  # noqa: E402


def _state(p):
    p32, _ = p.gpu_tensors("p32")
    p16, _ = p.gpu_tensors("p16", 0)
    return [bits32(a) for a in p32], [a.copy() for a in p16]


@pytest.mark.parametrize("seed", [1, 7])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_stage_equivalence_every_step(seed, n):
    ts = synth.mlp_layout((2, 8, 8, 1))
    cfg = OS.AdamConfig.defaults("fp16")
    runs = [Pair(Run(ts, n, stage, cfg, align=1, cap=0, seed=seed)) for stage in range(4)]
    for s in range(50):
        for p in runs:
            oinfo, ginfos = p.step()
            p.compare_info(oinfo, ginfos)
        base32, base16 = _state(runs[0])
        for stage, p in enumerate(runs[1:], 1):
            g32, g16 = _state(p)
            for t in range(len(ts)):
                assert np.array_equal(g32[t], base32[t]), (seed, n, stage, s, "p32", t)
                assert np.array_equal(g16[t], base16[t]), (seed, n, stage, s, "p16", t)
    for p in runs:
        p.compare()          # and every stage equals the oracle after 50 steps
        p.destroy()


@pytest.mark.parametrize("n,stage", [(2, 1), (4, 2), (8, 3), (4, 0)])
def test_bucket_capacity_does_not_change_results(n, stage):
    ts = synth.mlp_layout((60, 40, 20))
    cfg = OS.AdamConfig.defaults("bf16")
    A = 8
    results = []
    for cap in (n * A, 7 * n * A, 0):
        p = Pair(Run(ts, n, stage, cfg, align=A, cap=cap, seed=3))
        for _s in range(4):
            p.step()
        p.compare()
        g32, g16 = _state(p)
        results.append((g32, g16))
        pp = p.lay.psi_padded
        c = p.engines[0].comm_counters()
        sent = c.reduce_scatter + c.all_gather + c.all_reduce
        if stage < 3:          # 2 Psi'(N-1)/N per step on this run's own padded Psi'
            assert sent == 4 * P.step_elems_per_rank(pp, n, stage)
        else:                  # no layer gathers in this protocol: the reduce-scatter third
            assert c.reduce_scatter == 4 * P.rs_sent(pp, n)
        p.destroy()
    for g32, g16 in results[1:]:
        for t in range(len(ts)):
            assert np.array_equal(g32[t], results[0][0][t]) and np.array_equal(g16[t], results[0][1][t])
