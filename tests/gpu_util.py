"""Helpers for the GPU tests: move gen/ inputs to the device, build a layer,
compare against the oracle with the north-star tolerances."""
import numpy as np
import torch

from paper_2410_12247_b200 import MoELayer


def dev_bf16(bits: np.ndarray, device="cuda") -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16))
    return t.to(device).view(torch.bfloat16)


def to_f32(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


def layer_from_inputs(inp, k, norm_topk, max_tokens=None, ep=1, rank=0, experts=None, **kw):
    w = dict(w_router=dev_bf16(inp.w_router), w_gate=dev_bf16(inp.w_gate), w_up=dev_bf16(inp.w_up),
             w_down=dev_bf16(inp.w_down))
    if inp.S:
        w.update(ws_gate=dev_bf16(inp.ws_gate), ws_up=dev_bf16(inp.ws_up), ws_down=dev_bf16(inp.ws_down))
    if inp.router_bias is not None:
        w["router_bias"] = torch.from_numpy(inp.router_bias).cuda()
    return MoELayer(inp.E, k, inp.H, inp.F, w, S=inp.S, Fs=inp.Fs, ep=ep, rank=rank,
                    max_tokens=max_tokens or inp.T, norm_topk=norm_topk, **kw)


def assert_close(y, ref, what=""):
    """North-star tolerance (BASELINE.json): max|err| <= 1e-2 max|ref| and
    normwise mean relative error sum|err| / sum|ref| <= 2e-3 (R5)."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(y - ref)
    mx = err.max() / max(np.abs(ref).max(), 1e-30)
    mean = err.sum() / max(np.abs(ref).sum(), 1e-30)
    assert mx <= 1e-2 and mean <= 2e-3, f"{what}: max {mx:.3e} mean {mean:.3e}"
    return mx, mean
