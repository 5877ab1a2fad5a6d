"""ctypes mirror of include/epsmoe.h (argument marshalling only).

Every step of the layer runs in libepsmoe.so; this module only converts
Python / torch arguments to the C ABI.  Loading fails loudly when the library
is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EPSMOE_LIB: another build of the same library (dev A/B of two kernel versions on one box)
LIB_PATH = os.environ.get("EPSMOE_LIB") or os.path.join(_HERE, "libepsmoe.so")

MOE_MAX_EXPERTS = 256
MOE_MAX_TOPK = 8
MOE_MAX_CHUNKS = 64
MOE_COST_POINTS = 12
MOE_COMM_POINTS = 4

MOE_GEMM_AUTO, MOE_GEMM_GROUPED, MOE_GEMM_DENSE = 0, 1, 2
STAGES = ["router", "route", "shared", "gateup", "down", "combine", "dispatch_a2a", "combine_a2a", "total",
          "exposed_a2a"]
STATUS = {0: "MOE_OK", 1: "MOE_ERR_INVALID", 2: "MOE_ERR_UNSUPPORTED", 3: "MOE_ERR_CAPACITY",
          4: "MOE_ERR_CUDA", 5: "MOE_ERR_NCCL", 6: "MOE_ERR_MISMATCH"}


class moe_config_t(C.Structure):
    _fields_ = [("num_experts", C.c_int32), ("top_k", C.c_int32), ("hidden", C.c_int32),
                ("ffn", C.c_int32), ("num_shared", C.c_int32), ("shared_ffn", C.c_int32),
                ("ep", C.c_int32), ("rank", C.c_int32), ("max_tokens", C.c_int64),
                ("norm_topk", C.c_int32), ("routed_scale", C.c_float), ("dispatch_fp8", C.c_int32),
                ("local_reduce", C.c_int32), ("route_groups", C.c_int32), ("route_topk_groups", C.c_int32),
                ("a2a_p2p", C.c_int32)]


class moe_weights_t(C.Structure):
    _fields_ = [("w_router", C.c_void_p), ("w_gate", C.c_void_p), ("w_up", C.c_void_p),
                ("w_down", C.c_void_p), ("ws_gate", C.c_void_p), ("ws_up", C.c_void_p),
                ("ws_down", C.c_void_p), ("router_bias", C.c_void_p)]


class moe_plan_t(C.Structure):
    _fields_ = [("num_chunks", C.c_int32), ("token_slices", C.c_int32), ("gemm_kind", C.c_int32),
                ("sm_gemm", C.c_int32), ("comm_ctas", C.c_int32),
                ("group_begin", C.c_int32 * (MOE_MAX_CHUNKS + 1)),
                ("expert_kind", C.c_uint8 * MOE_MAX_EXPERTS),
                ("pred_comm_ms", C.c_float), ("pred_comp_ms", C.c_float), ("pred_k_ms", C.c_float),
                ("pred_b_ms", C.c_float), ("pred_gain_ms", C.c_float), ("tile_m", C.c_int32)]

    def as_dict(self):
        n = self.num_chunks
        return dict(num_chunks=n, token_slices=self.token_slices, gemm_kind=self.gemm_kind,
                    sm_gemm=self.sm_gemm, comm_ctas=self.comm_ctas,
                    group_begin=list(self.group_begin[:n // max(1, self.token_slices) + 1]),
                    pred_comm_ms=self.pred_comm_ms, pred_comp_ms=self.pred_comp_ms,
                    pred_k_ms=self.pred_k_ms, pred_b_ms=self.pred_b_ms, pred_gain_ms=self.pred_gain_ms,
                    tile_m=self.tile_m)


class moe_cost_model_t(C.Structure):
    _fields_ = [("n_points", C.c_int32), ("m_points", C.c_float * MOE_COST_POINTS),
                ("gemm_ms", (C.c_float * MOE_COST_POINTS) * 2), ("a2a_fixed_ms", C.c_float),
                ("a2a_gbps", C.c_float), ("k_ms", C.c_float), ("b_ms", C.c_float),
                ("num_sms", C.c_int32), ("n_comm", C.c_int32), ("comm_ctas", C.c_int32 * MOE_COMM_POINTS),
                ("a2a_gbps_at", C.c_float * MOE_COMM_POINTS), ("gemm_scale_at", C.c_float * MOE_COMM_POINTS)]


class moe_debug_t(C.Structure):
    _fields_ = [("override_routing", C.c_int32), ("logits", C.c_void_p), ("topk_idx", C.c_void_p),
                ("topk_w", C.c_void_p), ("pos", C.c_void_p), ("hist", C.c_void_p),
                ("seg_start", C.c_void_p), ("shared_out", C.c_void_p),
                ("global_hist_host", C.c_void_p), ("plan_used", C.POINTER(moe_plan_t)),
                ("lr_pos", C.c_void_p), ("lr_hist", C.c_void_p), ("chunk_rows_host", C.c_void_p),
                ("combine_in", C.c_void_p), ("gemm_resident", C.c_void_p)]


_SIGS = {
    "moe_layer_workspace_bytes": (C.c_size_t, [C.POINTER(moe_config_t)]),
    "moe_get_unique_id": (C.c_int, [C.c_void_p]),
    "moe_layer_create": (C.c_int, [C.POINTER(moe_config_t), C.POINTER(moe_weights_t), C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "moe_layer_destroy": (C.c_int, [C.c_void_p]),
    "moe_layer_create_hostcoll": (C.c_int, [C.POINTER(moe_config_t), C.POINTER(moe_weights_t), C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "moe_local_group_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "moe_local_group_destroy": (C.c_int, [C.c_void_p]),
    "moe_layer_create_local": (C.c_int, [C.POINTER(moe_config_t), C.POINTER(moe_weights_t), C.c_void_p,
                                         C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "moe_plan_compute": (C.c_int, [C.POINTER(moe_config_t), C.POINTER(moe_cost_model_t), C.c_int64,
                                   C.c_void_p, C.POINTER(moe_plan_t)]),
    "moe_plan_pipeline": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(moe_plan_t)]),
    "moe_exchange_layout": (C.c_int, [C.POINTER(moe_config_t), C.POINTER(moe_plan_t), C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]),
    "moe_layer_calibrate": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(moe_cost_model_t)]),
    "moe_layer_set_cost_model": (C.c_int, [C.c_void_p, C.POINTER(moe_cost_model_t)]),
    "moe_layer_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(moe_plan_t),
                                    C.c_void_p, C.POINTER(moe_debug_t)]),
    "moe_layer_forward_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                         C.POINTER(moe_plan_t), C.c_void_p]),
    "moe_layer_forward_host_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                               C.POINTER(moe_plan_t), C.c_void_p]),
    "moe_layer_host_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "moe_layer_last_launches": (C.c_int32, [C.c_void_p]),
    "moe_layer_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "moe_layer_set_comm_only": (C.c_int, [C.c_void_p, C.c_int32]),
    "moe_layer_stage_ms": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_int32)]),
    "moe_last_error": (C.c_char_p, []),
    "moe_gemm_grouped": (C.c_int, [C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p,
                                   C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
}

_LIB = None


def lib():
    """Load libepsmoe.so (RTLD_GLOBAL so NCCL resolves to torch's copy)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


# int allgather(void* ctx, const void* send, void* recv, size_t bytes)
HOST_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class EpsMoeError(RuntimeError):
    pass


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().moe_last_error().decode(errors="replace")
        raise EpsMoeError(f"{what}: {STATUS.get(status, status)}: {msg}")


def make_config(E, k, H, F, S=0, Fs=0, ep=1, rank=0, max_tokens=1, norm_topk=0, routed_scale=1.0,
                dispatch_fp8=0, local_reduce=0, route_groups=0, route_topk_groups=0, a2a_p2p=0):
    return moe_config_t(E, k, H, F, S, Fs, ep, rank, max_tokens, norm_topk, routed_scale, dispatch_fp8,
                        local_reduce, route_groups, route_topk_groups, a2a_p2p)


def plan_compute(cfg: moe_config_t, global_tokens: int, global_hist=None, cost: moe_cost_model_t | None = None):
    """Host-only expert pipeline scheduler (no GPU needed).  global_hist: numpy int32 [ep, E] or None."""
    import numpy as np
    plan = moe_plan_t()
    hp = None
    if global_hist is not None:
        gh = np.ascontiguousarray(global_hist, dtype=np.int32)
        hp = gh.ctypes.data_as(C.c_void_p)
    check(lib().moe_plan_compute(C.byref(cfg), C.byref(cost) if cost is not None else None,
                                 int(global_tokens), hp, C.byref(plan)), "moe_plan_compute")
    return plan


def exchange_layout(cfg: moe_config_t, plan: moe_plan_t, global_hist):
    """Host-only all2all layout of rank cfg.rank (see moe_exchange_layout)."""
    import numpy as np
    E, D = cfg.num_experts, cfg.ep
    gh = np.ascontiguousarray(global_hist, dtype=np.int32)
    send_off = np.zeros(E + 1, np.int64)
    recv_off = np.zeros((E // D) * D + 1, np.int64)
    cs = np.zeros((plan.num_chunks, D), np.int64)
    cr = np.zeros((plan.num_chunks, D), np.int64)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    check(lib().moe_exchange_layout(C.byref(cfg), C.byref(plan), p(gh), p(send_off), p(recv_off), p(cs), p(cr)),
          "moe_exchange_layout")
    return send_off, recv_off, cs, cr


def make_plan(num_chunks=1, gemm_kind=MOE_GEMM_GROUPED, sm_gemm=0, comm_ctas=0, tile_m=0, token_slices=1):
    """num_chunks = PN = expert groups x token_slices (chunk c = group c // S, slice c % S)."""
    p = moe_plan_t()
    p.tile_m = tile_m
    p.num_chunks = num_chunks
    p.token_slices = token_slices
    p.gemm_kind = gemm_kind
    p.sm_gemm = sm_gemm
    p.comm_ctas = comm_ctas
    return p
