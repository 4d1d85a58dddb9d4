"""B200-native ZeRO-DP hot path (arXiv 1910.02054): C-ABI library + thin binding.

The partitioned mixed-precision Adam step (stages P_os, P_os+g, P_os+g+p) runs in
hand-written sm_100a kernels behind include/zero_b200.h; see DESIGN.md.

The names below are resolved on first use, which loads libzero_b200.so and raises
ImportError if it has not been built (there is no CPU fallback); importing the
package alone does not load it, so `python -m paper_1910_02054_b200._build` works
in a fresh checkout.
"""
__all__ = ["ZeroConfig", "ZeroEngine", "ZeroError", "ZeroSimGroup", "plan_layout", "model_state_bytes",
           "comm_elems_per_rank", "nccl_comm_ptr", "consolidate_states"]


def __getattr__(name):
    if name in __all__:
        from . import zero
        return getattr(zero, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
