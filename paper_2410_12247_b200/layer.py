"""MoELayer: the Python face of the C ABI (torch only for memory / streams).

One call of ``forward`` runs Algorithm 1 entirely in
libepsmoe.so: router GEMM, topKGating, split, (all2all dispatch,) expert
SwiGLU GEMMs on tcgen05, (all2all combine,) weighted LocalReduce.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import abi


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class LocalGroup:
    """In-process EP group (moe_local_group_create): `ep` MoELayer ranks on one
    GPU, each forward driven from its own host thread (tests only)."""

    def __init__(self, ep: int):
        self.ep = ep
        h = C.c_void_p()
        abi.check(abi.lib().moe_local_group_create(ep, C.byref(h)), "moe_local_group_create")
        self.handle = h

    def __del__(self):
        try:
            abi.lib().moe_local_group_destroy(self.handle)
        except Exception:
            pass


class HostAllgather:
    """The blocking host allgather moe_layer_create_hostcoll needs, over a
    torch.distributed process group (e.g. gloo): rank r's `bytes` bytes land at
    recv + r * bytes on every rank.  Argument marshalling only: the C library
    decides what to exchange (counts, cudaIpc handles)."""

    def __init__(self, group=None):
        self.group = group
        self.fn = abi.HOST_ALLGATHER_FN(self._call)   # keep the C callback alive

    def _call(self, ctx, send, recv, nbytes):
        try:
            import torch.distributed as dist
            ws = dist.get_world_size(self.group)
            src = torch.empty(nbytes, dtype=torch.uint8)
            C.memmove(src.data_ptr(), send, nbytes)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(ws)]
            dist.all_gather(outs, src, group=self.group)
            for r, t in enumerate(outs):
                C.memmove(recv + r * nbytes, t.data_ptr(), nbytes)
            return 0
        except Exception:  # reported to the library as a failed collective (MOE_ERR_MISMATCH)
            return 1


class MoELayer:
    """weights: dict of DEVICE tensors (bf16): w_router [E,H], w_gate / w_up
    [E_loc,F,H], w_down [E_loc,H,F], optional ws_gate / ws_up [S*Fs,H],
    ws_down [H,S*Fs], router_bias fp32 [E]."""

    def __init__(self, E, k, H, F, weights, S=0, Fs=0, ep=1, rank=0, max_tokens=1, norm_topk=0,
                 routed_scale=1.0, dispatch_fp8: bool = False, local_reduce: bool = False,
                 route_groups: int = 0, route_topk_groups: int = 0, a2a_p2p: int = 0,
                 uid_dispatch: bytes | None = None, uid_combine: bytes | None = None,
                 device=None, local_group: "LocalGroup | None" = None,
                 host_allgather: "HostAllgather | None" = None):
        self.lib = abi.lib()
        self.cfg = abi.make_config(E, k, H, F, S, Fs, ep, rank, max_tokens, norm_topk, routed_scale,
                                   1 if dispatch_fp8 else 0, 1 if local_reduce else 0, route_groups,
                                   route_topk_groups, int(a2a_p2p))
        self.E, self.k, self.H, self.F, self.S, self.Fs, self.ep, self.rank = E, k, H, F, S, Fs, ep, rank
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nbytes = self.lib.moe_layer_workspace_bytes(C.byref(self.cfg))
        if nbytes == 0:
            abi.check(1, "moe_layer_workspace_bytes")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.weights = weights  # keep alive
        w = abi.moe_weights_t(*[_ptr(weights.get(n)) for n in
                                ("w_router", "w_gate", "w_up", "w_down", "ws_gate", "ws_up", "ws_down",
                                 "router_bias")])
        h = C.c_void_p()
        ud = C.create_string_buffer(uid_dispatch, 128) if uid_dispatch is not None else None
        uc = C.create_string_buffer(uid_combine, 128) if uid_combine is not None else None
        with torch.cuda.device(self.device):
            if host_allgather is not None:
                self.host_allgather = host_allgather  # keep the callback alive
                abi.check(self.lib.moe_layer_create_hostcoll(C.byref(self.cfg), C.byref(w), host_allgather.fn, None,
                                                             C.c_void_p(self.workspace.data_ptr()), nbytes,
                                                             C.byref(h)),
                          "moe_layer_create_hostcoll")
            elif local_group is not None:
                self.local_group = local_group  # keep alive
                abi.check(self.lib.moe_layer_create_local(C.byref(self.cfg), C.byref(w), local_group.handle,
                                                          C.c_void_p(self.workspace.data_ptr()), nbytes, C.byref(h)),
                          "moe_layer_create_local")
            else:
                abi.check(self.lib.moe_layer_create(C.byref(self.cfg), C.byref(w), ud, uc,
                                                    C.c_void_p(self.workspace.data_ptr()), nbytes, C.byref(h)),
                          "moe_layer_create")
        self.handle = h

    # ------------------------------------------------------------------
    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        abi.check(abi.lib().moe_get_unique_id(buf), "moe_get_unique_id")
        return buf.raw

    def plan(self, global_tokens: int, global_hist=None) -> abi.moe_plan_t:
        import numpy as np
        p = abi.moe_plan_t()
        hp = None
        if global_hist is not None:
            gh = np.ascontiguousarray(global_hist, dtype=np.int32)
            hp = gh.ctypes.data_as(C.c_void_p)
        abi.check(self.lib.moe_plan_pipeline(self.handle, int(global_tokens), hp, C.byref(p)), "moe_plan_pipeline")
        return p

    def calibrate(self, stream=None) -> abi.moe_cost_model_t:
        m = abi.moe_cost_model_t()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        abi.check(self.lib.moe_layer_calibrate(self.handle, C.c_void_p(st.cuda_stream), C.byref(m)),
                  "moe_layer_calibrate")
        return m

    def set_cost_model(self, m: abi.moe_cost_model_t) -> None:
        abi.check(self.lib.moe_layer_set_cost_model(self.handle, C.byref(m)), "moe_layer_set_cost_model")

    def forward(self, x: torch.Tensor, y: torch.Tensor | None = None, plan: abi.moe_plan_t | None = None,
                stream=None, debug: abi.moe_debug_t | None = None) -> torch.Tensor:
        assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous() and x.shape[1] == self.H
        T = x.shape[0]
        if y is None:
            y = torch.empty_like(x)
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        abi.check(self.lib.moe_layer_forward(self.handle, C.c_void_p(x.data_ptr()), T, C.c_void_p(y.data_ptr()),
                                             C.byref(plan) if plan is not None else None,
                                             C.c_void_p(st.cuda_stream),
                                             C.byref(debug) if debug is not None else None),
                  "moe_layer_forward")
        return y

    def forward_host(self, x_host: torch.Tensor, y_host: torch.Tensor, plan=None, stream=None) -> torch.Tensor:
        """End-to-end call on HOST (pinned) bf16 buffers: H2D, layer, D2H, synchronised."""
        T = x_host.shape[0]
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        abi.check(self.lib.moe_layer_forward_host(self.handle, C.c_void_p(x_host.data_ptr()), T,
                                                  C.c_void_p(y_host.data_ptr()),
                                                  C.byref(plan) if plan is not None else None,
                                                  C.c_void_p(st.cuda_stream)),
                  "moe_layer_forward_host")
        return y_host

    def forward_host_async(self, x_host: torch.Tensor, y_host: torch.Tensor, plan=None, stream=None) -> None:
        """forward_host without the final wait: consecutive calls overlap their copies with the
        previous call's compute; x_host / y_host stay owned by the layer until host_sync()."""
        T = x_host.shape[0]
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        abi.check(self.lib.moe_layer_forward_host_async(self.handle, C.c_void_p(x_host.data_ptr()), T,
                                                        C.c_void_p(y_host.data_ptr()),
                                                        C.byref(plan) if plan is not None else None,
                                                        C.c_void_p(st.cuda_stream)),
                  "moe_layer_forward_host_async")

    def host_sync(self, stream=None) -> None:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        abi.check(self.lib.moe_layer_host_sync(self.handle, C.c_void_p(st.cuda_stream)), "moe_layer_host_sync")

    def set_comm_only(self, on: bool = True) -> None:
        """ep > 1 measurement hook: later forwards skip ComputeMoE and the shared
        experts (y undefined), so the chunked all2all is timed alone."""
        abi.check(self.lib.moe_layer_set_comm_only(self.handle, 1 if on else 0), "moe_layer_set_comm_only")

    def set_profiling(self, on: bool = True) -> None:
        abi.check(self.lib.moe_layer_set_profiling(self.handle, 1 if on else 0), "moe_layer_set_profiling")

    def stage_ms(self) -> dict:
        """Per-stage device ms of the last forward (events on the launching streams)."""
        ms = (C.c_float * len(abi.STAGES))()
        cnt = (C.c_int32 * len(abi.STAGES))()
        abi.check(self.lib.moe_layer_stage_ms(self.handle, ms, cnt), "moe_layer_stage_ms")
        return {n: (float(ms[i]), int(cnt[i])) for i, n in enumerate(abi.STAGES)}

    def last_launches(self) -> int:
        return int(self.lib.moe_layer_last_launches(self.handle))

    def debug_buffers(self, T: int, override=None, combine_in: bool = False):
        """Allocate a moe_debug_t with device outputs; override=(idx, w) tensors
        switches routing to explicit (fig:eps_overview fixture); combine_in also
        captures the expert outputs the weighted unpermute reads ([T*k, H])."""
        dev = self.device
        bufs = dict(
            logits=torch.empty(T, self.E, dtype=torch.float32, device=dev),
            topk_idx=torch.empty(T, self.k, dtype=torch.int32, device=dev),
            topk_w=torch.empty(T, self.k, dtype=torch.float32, device=dev),
            pos=torch.empty(T, self.k, dtype=torch.int32, device=dev),
            hist=torch.empty(self.E, dtype=torch.int32, device=dev),
            seg_start=torch.empty(self.E + 1, dtype=torch.int32, device=dev),
            shared_out=torch.empty(T, self.H, dtype=torch.bfloat16, device=dev) if self.S else None,
            lr_pos=torch.full((T, self.k), -7, dtype=torch.int32, device=dev) if self.cfg.local_reduce else None,
            lr_hist=torch.full((256,), -7, dtype=torch.int32, device=dev) if self.cfg.local_reduce else None,
            combine_in=torch.empty(T * self.k, self.H, dtype=torch.bfloat16, device=dev)
            if combine_in and not self.cfg.local_reduce else None,
            gemm_resident=torch.zeros(2, dtype=torch.int32, device=dev),
        )
        if override is not None:
            bufs["topk_idx"] = override[0].to(dev, torch.int32).contiguous()
            bufs["topk_w"] = override[1].to(dev, torch.float32).contiguous()
        import numpy as np
        ghist = np.zeros((self.ep, self.E), dtype=np.int32)
        plan_used = abi.moe_plan_t()
        chunk_rows = np.full((2, abi.MOE_MAX_CHUNKS, self.ep), -1, dtype=np.int64)
        d = abi.moe_debug_t(1 if override is not None else 0,
                            *[_ptr(bufs[n]) for n in ("logits", "topk_idx", "topk_w", "pos", "hist",
                                                       "seg_start", "shared_out")],
                            ghist.ctypes.data_as(C.c_void_p), C.pointer(plan_used),
                            _ptr(bufs["lr_pos"]), _ptr(bufs["lr_hist"]), chunk_rows.ctypes.data_as(C.c_void_p),
                            _ptr(bufs["combine_in"]), _ptr(bufs["gemm_resident"]))
        bufs["chunk_rows"] = chunk_rows
        bufs["global_hist"] = ghist
        bufs["plan_used"] = plan_used
        bufs["_struct"] = d
        return d, bufs

    def close(self) -> None:
        if getattr(self, "handle", None):
            abi.check(self.lib.moe_layer_destroy(self.handle), "moe_layer_destroy")
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gemm_grouped(epi, A, B0, B1, n, out, row_start, row_count, b_group_rows, bias=None, num_ctas=148,
                 tile_m=128, stream=None):
    """Test / calibration hook: one launch of the layer's tcgen05 GEMM family."""
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    abi.check(abi.lib().moe_gemm_grouped(int(epi), _ptr(A), A.shape[0], _ptr(B0), _ptr(B1), B0.shape[0],
                                         int(b_group_rows), A.shape[1], int(n), _ptr(out), out.shape[1],
                                         _ptr(bias), row_start.numel(), _ptr(row_start), _ptr(row_count),
                                         int(num_ctas), int(tile_m), C.c_void_p(st.cuda_stream)),
              "moe_gemm_grouped")
    return out
