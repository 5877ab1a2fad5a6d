"""B200-native (sm_100a) EPS-MoE layer: the expert-parallel MoE FFN layer in
prefill with the paper's expert pipeline scheduler (arXiv 2410.12247).

The compute path is libepsmoe.so (include/epsmoe.h); this package only marshals
arguments.  It never imports oracle/ and has no CPU fallback.
"""
from .abi import (MOE_GEMM_AUTO, MOE_GEMM_DENSE, MOE_GEMM_GROUPED, EpsMoeError, lib, make_config,  # noqa: F401
                  make_plan, moe_cost_model_t, moe_plan_t, plan_compute)
from .layer import HostAllgather, LocalGroup, MoELayer, gemm_grouped  # noqa: F401
