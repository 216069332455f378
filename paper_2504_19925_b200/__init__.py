"""B200-native decoupled-MoE expert step (arXiv 2504.19925).

The hot path -- plan, dispatch, reduce, Adam, re-place -- lives in the C-ABI library
``libmoedc.so`` (include/moe_dc.h; CUDA kernels for sm_100a under csrc/).  This package is
its thin Python binding: ``api`` mirrors the C names, ``layer.DecoupledExpertLayer`` drives
one MoE layer's iteration.  There is no CPU fallback: importing ``api`` without the built
library raises.
"""
from .api import (AdamConfig, DispatchBuffers, MoeContext, MoeError, Plan,  # noqa: F401
                  MOE_OPT_DEDUP, MOE_OPT_HOST_STATE, MOE_OPT_LAZY_REPLICATE, MOE_PLAN_KEEP, MOE_PLAN_MINMAX, MOE_PLAN_SCHEDULED, MOE_PLAN_PAPER_ALG1,
                  MOE_PLAN_STATIC, moe_dispatch, moe_place, moe_plan, moe_slot_capacity, moe_step,
                  moe_update, synth_grads, synth_master, TokenExchange, MOE_TOK_GATE,
                  moe_token_dispatch, moe_token_combine)
from .layer import DecoupledExpertLayer  # noqa: F401
