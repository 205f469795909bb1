"""paper_1911_08907_b200 -- B200-native APS (Auto-Precision Scaling, arXiv
1911.08907) gradient synchronisation: libaps.so (sm_100a CUDA + NCCL) and its
thin ctypes binding.  See include/aps.h for the C ABI and DESIGN.md."""
from .aps import (ApsContext, ApsError, debug_cast, debug_cast_sr, debug_decode, debug_ring_reduce, layout, layout_mixed, load,
                  nccl_comm_destroy, nccl_comm_init, nccl_unique_id, ring_step, round_off_error, sim_allreduce,
                  sim_connect, sim_layer_scales)

from .ddp import ApsHookState, aps_hook

__all__ = ["ApsHookState", "aps_hook", "ApsContext", "ApsError", "debug_cast", "debug_decode", "debug_ring_reduce", "layout", "layout_mixed", "load",
           "nccl_comm_destroy", "nccl_comm_init", "nccl_unique_id", "ring_step", "sim_allreduce",
           "sim_layer_scales", "sim_connect", "round_off_error", "debug_cast_sr"]
