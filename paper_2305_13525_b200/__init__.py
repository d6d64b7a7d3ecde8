"""B200-native MoE layer (arXiv 2305.13525 hot path): top-1 gating with capacity,
dispatch, expert-parallel all-to-all with Duplicate Token Dropping, tcgen05
expert FFN, weighted combine — behind the C ABI of include/moe.h; the paper's
tiled optimizer step for the expert parameters behind include/moe_optim.h.

The CUDA library (libmoe.so) is loaded lazily by `binding.lib()`; there is no
CPU fallback.
"""
from .binding import (MOE_F_AUX_LOSS, MOE_F_RANDOM_PRIORITY, MOE_F_CAC, MOE_F_CHECKPOINT, MOE_F_FORCED_ROUTING, MOE_F_NCCL_EXCHANGE, MOE_F_NVLS, MOE_F_STATS, MOE_F_TIMING, MoEConfig, MoEError, MoEFunction,  # noqa: F401
                      MOE_TILE_PARAMS_PAPER, MoELayer, lib, moe_adamw_plan, moe_adamw_step, moe_gemm_bf16,
                      moe_get_unique_id, moe_plan_bytes, moe_plan_collectives, moe_plan_layout,
                      EmuGroup, MoEComm, moe_comm_plan_bytes)
