"""Checkpoint / resharding through zero_export_state / zero_import_state: the state
in tensor coordinates is independent of N_d, stage and C_B, so a run can be saved
on 4 simulated ranks at stage 2 and resumed on 2 ranks at stage 3 (or on 1 rank) --
against the oracle that simply continues (partitions are a placement)."""
import numpy as np
import pytest
import torch

import synth
from oracle import step as OS

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from harness import Pair, Run  # noqa: E402


@pytest.mark.parametrize("src,dst", [((4, 2, "R16"), (2, 3, "R16")), ((1, 1, "R16"), (4, 2, "R32")),
                                     ((4, 0, "R16"), (1, 2, "R16"))])
def test_save_reshard_resume(src, dst):
    from paper_1910_02054_b200 import consolidate_states
    ts = synth.mlp_layout((300, 200, 100))
    n0, st0, m0 = src
    n1, st1, m1 = dst
    a = Pair(Run(ts, n0, st0, OS.AdamConfig.defaults("fp16", scale_window=2, reduce_mode=m0), cap=1 << 13))
    for _ in range(3):
        a.step()
    state = consolidate_states([e.export_state() for e in a.engines])
    # the consolidated state equals the oracle's, in tensor coordinates, bitwise
    for k, ref in (("master", a.ost.p32), ("m", a.ost.m), ("v", a.ost.v)):
        for t, r in enumerate(ref):
            assert np.array_equal(state[k][t].cpu().numpy().view(np.uint32), r.view(np.uint32)), (k, t)
    assert state["scalars"]["t"] == a.ost.t and state["scalars"]["loss_scale"] == a.ost.S
    assert state["scalars"]["good_steps"] == a.ost.good
    # resume on another N_d / stage / reduce mode: the Pair's oracle continues from a's
    b = Pair(Run(ts, n1, st1, OS.AdamConfig.defaults("fp16", scale_window=2, reduce_mode=m1), cap=1 << 12))
    for e in b.engines:
        e.import_state(state)
    b.ost = a.ost
    b.step_no = a.step_no
    for _ in range(3):
        oi, gi = b.step()
        b.compare_info(oi, gi)
    b.compare()
    a.destroy()
    b.destroy()
