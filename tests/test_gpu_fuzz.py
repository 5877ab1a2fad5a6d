"""Randomised small configurations (seeded): shapes at the validation limits
(H multiple of 64, F multiple of 128, E up to 256, k up to 8, T ragged incl. 1),
norm / raw gating, shared experts on/off, skew bias, FP8 dispatch, LocalReduce,
device-limited routing, EP 1/2/4 with both all2all planes.  y vs the oracle
(north-star tolerance) on the exact-logit grid, so routing is exact."""
import threading

import numpy as np
import pytest
import torch

import oracle
from gen import Inputs, router_skew_bias
from paper_2410_12247_b200 import MOE_GEMM_GROUPED, LocalGroup, MoELayer, make_plan

from .gpu_util import assert_close, dev_bf16

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    D = int(rng.choice([1, 1, 2, 4]))
    E = int(D * rng.choice([1, 2, 3, 4, 8, 16]))
    E = min(E, 256)
    k = int(rng.integers(1, min(8, E) + 1))
    H = int(64 * rng.integers(1, 7))
    F = int(128 * rng.integers(1, 4))
    S = int(rng.integers(0, 3))
    T = int(rng.choice([1, 17, 255, 700, 1333]))
    opts = dict(norm=int(rng.integers(0, 2)), fp8=bool(rng.random() < 0.25 and H % 128 == 0),
                lr=bool(rng.random() < 0.25), p2p=bool(D > 1 and rng.random() < 0.5),
                skew=float(rng.choice([0.0, 0.0, 1.0])))
    if E >= 4 and rng.random() < 0.3:
        G = int(rng.choice([g for g in (2, 4) if E % g == 0]))
        M = int(rng.integers(1, G))
        if k <= M * (E // G):
            opts.update(route_groups=G, route_topk_groups=M)
    return D, E, k, H, F, S, T, opts


@pytest.mark.parametrize("seed", list(range(40)))
def test_fuzz_layer_vs_oracle(seed):
    D, E, k, H, F, S, T, o = _case(1000 + seed)
    inp = Inputs(E=E, k=k, H=H, F=F, S=min(S, 1), Fs=128 * S if S else 0, T=T, seed=seed, grid=True)
    bias = router_skew_bias(E, o["skew"]) if o["skew"] else None
    E_loc = E // D
    rg = dict(route_groups=o.get("route_groups", 0), route_topk_groups=o.get("route_topk_groups", 0))
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=o["norm"],
                           ws_gate_bits=inp.ws_gate if inp.S else None, ws_up_bits=inp.ws_up if inp.S else None,
                           ws_down_bits=inp.ws_down if inp.S else None, router_bias=bias, D=D, N=1,
                           dispatch_fp8=o["fp8"], local_reduce=o["lr"], **rg)
    start = oracle.token_shards(T, D)
    group = LocalGroup(D) if D > 1 else None
    layers, xs = [], []
    for r in range(D):
        w = dict(w_router=dev_bf16(inp.w_router), w_gate=dev_bf16(inp.w_gate[r * E_loc:(r + 1) * E_loc]),
                 w_up=dev_bf16(inp.w_up[r * E_loc:(r + 1) * E_loc]),
                 w_down=dev_bf16(inp.w_down[r * E_loc:(r + 1) * E_loc]))
        if inp.S:
            w.update(ws_gate=dev_bf16(inp.ws_gate), ws_up=dev_bf16(inp.ws_up), ws_down=dev_bf16(inp.ws_down))
        if bias is not None:
            w["router_bias"] = torch.from_numpy(bias).cuda()
        T_loc = int(start[r + 1] - start[r])
        layers.append(MoELayer(E, k, H, F, w, S=inp.S, Fs=inp.Fs, ep=D, rank=r,
                               max_tokens=max(int(np.diff(start).max()), 1),
                               norm_topk=o["norm"], dispatch_fp8=o["fp8"], local_reduce=o["lr"], local_group=group,
                               a2a_p2p=o["p2p"], **rg))
        xs.append(dev_bf16(inp.x[start[r]:start[r + 1]]) if T_loc else
                  torch.empty(0, H, dtype=torch.bfloat16, device="cuda"))
    ys, errs = [None] * D, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                # one chunk: LocalReduce's sum grouping depends on N (R16); the oracle uses N = 1
                ys[r] = layers[r].forward(xs[r], plan=make_plan(1, MOE_GEMM_GROUPED), stream=s)
                s.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(D)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, (errs, D, E, k, H, F, S, T, o)
    y = torch.cat(ys).float().cpu().numpy()
    assert_close(y, ref["y"], f"seed {seed}: D{D} E{E} k{k} H{H} F{F} S{S} T{T} {o}")
    for L in layers:
        L.close()


@pytest.mark.parametrize("seed", list(range(30)))
def test_fuzz_plans_vs_oracle(seed):
    """Random explicit plans on random configurations: expert-group chunk
    counts, token slices (ep > 1, not with LocalReduce), GEMM kind, tile rows;
    y vs the oracle simulating the same (D, N, slices)."""
    D, E, k, H, F, S, T, o = _case(5000 + seed)
    rng = np.random.default_rng(9000 + seed)
    E_loc = E // D
    NG = int(rng.integers(1, E_loc + 1))
    SL = int(rng.integers(1, 4)) if (D > 1 and not o["lr"] and NG * 3 <= 64) else 1
    kind = int(rng.choice([1, 2]))
    tile_m = int(rng.choice([0, 128, 256]))
    inp = Inputs(E=E, k=k, H=H, F=F, S=min(S, 1), Fs=128 * S if S else 0, T=T, seed=seed + 77, grid=True)
    bias = router_skew_bias(E, o["skew"]) if o["skew"] else None
    rg = dict(route_groups=o.get("route_groups", 0), route_topk_groups=o.get("route_topk_groups", 0))
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=o["norm"],
                           ws_gate_bits=inp.ws_gate if inp.S else None, ws_up_bits=inp.ws_up if inp.S else None,
                           ws_down_bits=inp.ws_down if inp.S else None, router_bias=bias, D=D, N=NG,
                           token_slices=SL, dispatch_fp8=o["fp8"], local_reduce=o["lr"], **rg)
    start = oracle.token_shards(T, D)
    T_max = max(int(np.diff(start).max()), 1)
    group = LocalGroup(D) if D > 1 else None
    layers, xs = [], []
    for r in range(D):
        w = dict(w_router=dev_bf16(inp.w_router), w_gate=dev_bf16(inp.w_gate[r * E_loc:(r + 1) * E_loc]),
                 w_up=dev_bf16(inp.w_up[r * E_loc:(r + 1) * E_loc]),
                 w_down=dev_bf16(inp.w_down[r * E_loc:(r + 1) * E_loc]))
        if inp.S:
            w.update(ws_gate=dev_bf16(inp.ws_gate), ws_up=dev_bf16(inp.ws_up), ws_down=dev_bf16(inp.ws_down))
        if bias is not None:
            w["router_bias"] = torch.from_numpy(bias).cuda()
        layers.append(MoELayer(E, k, H, F, w, S=inp.S, Fs=inp.Fs, ep=D, rank=r, max_tokens=T_max,
                               norm_topk=o["norm"], dispatch_fp8=o["fp8"], local_reduce=o["lr"], local_group=group,
                               a2a_p2p=o["p2p"], **rg))
        T_loc = int(start[r + 1] - start[r])
        xs.append(dev_bf16(inp.x[start[r]:start[r + 1]]) if T_loc else
                  torch.empty(0, H, dtype=torch.bfloat16, device="cuda"))
    ys, errs = [None] * D, []
    plan = make_plan(NG * SL, kind, tile_m=tile_m, token_slices=SL)

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ys[r] = layers[r].forward(xs[r], plan=plan, stream=s)
                s.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(D)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    desc = f"seed {seed}: D{D} E{E} k{k} H{H} F{F} S{S} T{T} NG{NG} SL{SL} kind{kind} tile{tile_m} {o}"
    assert not errs, (errs, desc)
    assert_close(torch.cat(ys).float().cpu().numpy(), ref["y"], desc)
    for L in layers:
        L.close()


@pytest.mark.parametrize("p2p", [False, True])
def test_worst_case_concentration(p2p):
    """Every token of every rank routes to the same k experts on one rank (the
    capacity bound D * max_tokens * min(k, E_loc) is met exactly there)."""
    D, E, k, H, F, T = 4, 16, 4, 128, 128, 803
    inp = Inputs(E=E, k=k, H=H, F=F, T=T, seed=3, grid=True)
    bias = np.full(E, -1000.0, np.float32)
    bias[4:8] = 0.0                                   # experts 4..7 = all of rank 1's experts
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=1,
                           router_bias=bias, D=D)
    assert (np.sort(ref["idx"], axis=1) == np.arange(4, 8)).all()
    start = oracle.token_shards(T, D)
    T_max = int(np.diff(start).max())
    group = LocalGroup(D)
    layers, xs = [], []
    for r in range(D):
        w = dict(w_router=dev_bf16(inp.w_router), w_gate=dev_bf16(inp.w_gate[r * 4:(r + 1) * 4]),
                 w_up=dev_bf16(inp.w_up[r * 4:(r + 1) * 4]), w_down=dev_bf16(inp.w_down[r * 4:(r + 1) * 4]),
                 router_bias=torch.from_numpy(bias).cuda())
        layers.append(MoELayer(E, k, H, F, w, ep=D, rank=r, max_tokens=T_max, norm_topk=1, local_group=group,
                               a2a_p2p=p2p))
        xs.append(dev_bf16(inp.x[start[r]:start[r + 1]]))
    ys, errs = [None] * D, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ys[r] = layers[r].forward(xs[r], stream=s)
                s.synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(D)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    assert_close(torch.cat(ys).float().cpu().numpy(), ref["y"], f"concentrated p2p={p2p}")
    for L in layers:
        L.close()
