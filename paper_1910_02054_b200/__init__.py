"""B200-native ZeRO-DP hot path (arXiv 1910.02054): C-ABI library + thin binding.

The partitioned mixed-precision Adam step (stages P_os, P_os+g, P_os+g+p) runs in
hand-written sm_100a kernels behind include/zero_b200.h; see DESIGN.md.
"""
from .zero import (ZeroConfig, ZeroEngine, ZeroError, ZeroSimGroup, comm_elems_per_rank,  # noqa: F401
                   consolidate_states, model_state_bytes, nccl_comm_ptr, plan_layout)

__all__ = ["ZeroConfig", "ZeroEngine", "ZeroError", "ZeroSimGroup", "plan_layout", "model_state_bytes",
           "comm_elems_per_rank", "nccl_comm_ptr", "consolidate_states"]
