"""Parity at BASELINE.json's full sizes (EP = 1 on one B200), in the launch
configuration bench.py times (planner-chosen plan, default tiles):

  * exact-logit grid inputs (x, W_r on {-8..8}/8, /64): logits, top-k indices,
    histogram, segment offsets and the permutation are checked on ALL tokens,
    bit-exact, against the oracle (numpy fp64 routing + dispatch_layout);
  * both distributions: routing stage-wise on ALL tokens (the oracle's top-k of
    the GPU's fp32 logits, bit-exact), the combine stage-wise on 4096 tokens
    (oracle.combine of the GPU's o / s / w, bit-exact), and y on >= 256 tokens
    that together touch every expert vs oracle.moe_tokens (y_t depends only on
    x_t and the weights), north-star tolerance.

Inputs come from gen/ (the device twin of the numpy generator, bit-identical:
test_gpu_parity.test_device_generator_matches_numpy; re-spot-checked here)."""
import numpy as np
import pytest
import torch

import oracle
from gen import (CONFIGS, MODE_GRID, MODE_UNIF, TID_WDOWN, TID_WGATE, TID_WR, TID_WS_DOWN, TID_WS_GATE,
                 TID_WS_UP, TID_WUP, TID_X, device_fill_bf16, fill_bf16, unif_scale)
from paper_2410_12247_b200 import MoELayer

from .gpu_util import assert_close

pytestmark = pytest.mark.gpu
SEED = 20241016


def _gen(shape, tid, base, mode, param):
    t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    device_fill_bf16(t.data_ptr(), t.numel(), SEED, tid, base, mode, float(param))
    return t


def _bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _spot_check(t, tid, base, mode, param):
    n = min(4096, t.numel())
    ref = fill_bf16(n, SEED, tid, base, mode, param)
    assert np.array_equal(_bits(t.reshape(-1)[:n]), ref)


@pytest.mark.parametrize("name", ["dsv2", "mixtral", "dsv2_lite"])
def test_full_size_parity(name):
    c = CONFIGS[name]
    E, k, H, F, S, Fs, T, norm = c["E"], c["k"], c["H"], c["F"], c["S"], c["Fs"], c["T"], c["norm_topk"]
    sH, sF = unif_scale(H), unif_scale(F)
    w = dict(w_gate=_gen((E, F, H), TID_WGATE, 0, MODE_UNIF, sH), w_up=_gen((E, F, H), TID_WUP, 0, MODE_UNIF, sH),
             w_down=_gen((E, H, F), TID_WDOWN, 0, MODE_UNIF, sF))
    _spot_check(w["w_gate"], TID_WGATE, 0, MODE_UNIF, sH)
    SF = S * Fs
    if SF:
        w.update(ws_gate=_gen((SF, H), TID_WS_GATE, 0, MODE_UNIF, sH), ws_up=_gen((SF, H), TID_WS_UP, 0, MODE_UNIF, sH),
                 ws_down=_gen((H, SF), TID_WS_DOWN, 0, MODE_UNIF, unif_scale(SF)))
    host_w = {}

    def expert_weights(e):
        if e not in host_w:
            host_w[e] = (_bits(w["w_gate"][e]), _bits(w["w_up"][e]), _bits(w["w_down"][e]))
        return host_w[e]
    shared = (_bits(w["ws_gate"]), _bits(w["ws_up"]), _bits(w["ws_down"])) if SF else None

    for dist in ("grid", "unif"):
        if dist == "grid":
            w["w_router"] = _gen((E, H), TID_WR, 0, MODE_GRID, 64.0)
            x = _gen((T, H), TID_X, 0, MODE_GRID, 8.0)
            _spot_check(x, TID_X, 0, MODE_GRID, 8.0)
        else:
            w["w_router"] = _gen((E, H), TID_WR, 0, MODE_UNIF, sH)
            x = _gen((T, H), TID_X, 0, MODE_UNIF, unif_scale(1))
        layer = MoELayer(E, k, H, F, w, S=S, Fs=Fs, max_tokens=T, norm_topk=norm)
        d, b = layer.debug_buffers(T, combine_in=True)
        y = layer.forward(x, debug=d)
        torch.cuda.synchronize()
        x_bits, wr_bits = _bits(x), _bits(w["w_router"])
        idx_gpu = b["topk_idx"].cpu().numpy()
        # stage-wise routing on ALL tokens: the oracle's top-k of the GPU's own fp32
        # logits == the GPU's indices bit for bit, weights within 1e-5
        gl = b["logits"].cpu().numpy()
        st_idx, st_w = oracle.topk_gating(gl, k, norm)
        assert np.array_equal(idx_gpu, st_idx), dist
        assert np.allclose(b["topk_w"].cpu().numpy(), st_w, rtol=1e-5, atol=0), dist
        # stage-wise combine on a 4096-token sample: y == oracle.combine(s, o[pos], w) bit for bit
        cs = np.unique(np.linspace(0, T - 1, 4096).astype(np.int64))
        pos_s = b["pos"][torch.from_numpy(cs).cuda()]
        o_s = b["combine_in"][pos_s.reshape(-1).long()].float().cpu().numpy().reshape(len(cs), k, H)
        s_s = b["shared_out"][torch.from_numpy(cs).cuda()].float().cpu().numpy() if SF else \
            np.zeros((len(cs), H), np.float32)
        y_st = oracle.combine(s_s, o_s, b["topk_w"].cpu().numpy()[cs])
        assert np.array_equal(y[torch.from_numpy(cs).cuda()].float().cpu().numpy(), y_st), dist
        del b["combine_in"]
        if dist == "grid":
            # routing + permutation on ALL tokens (grid => fp32 logits exact)
            ref_logits = oracle.router_logits(x_bits, wr_bits)
            assert np.array_equal(b["logits"].cpu().numpy(), ref_logits)
            ref_idx, ref_w = oracle.topk_gating(ref_logits, k, norm)
            assert np.array_equal(idx_gpu, ref_idx)
            assert np.allclose(b["topk_w"].cpu().numpy(), ref_w, rtol=1e-5, atol=0)
            lay = oracle.dispatch_layout(ref_idx, E, 1)
            assert np.array_equal(b["hist"].cpu().numpy(), lay["hist"][0])
            assert np.array_equal(b["seg_start"].cpu().numpy(), lay["send_start"][0])
            assert np.array_equal(b["pos"].cpu().numpy(), lay["pos"][0])
        # y vs the oracle's plain definition on >= 256 tokens that together touch
        # every expert (greedy cover over an even spread, then filled up)
        spread = np.unique(np.linspace(0, T - 1, 8192).astype(np.int64))
        chosen, seen = [], set()
        for t in spread:
            if not set(idx_gpu[t].tolist()) <= seen:
                chosen.append(int(t))
                seen |= set(idx_gpu[t].tolist())
        assert len(seen) == E
        fill = [int(t) for t in np.unique(np.linspace(0, T - 1, 256).astype(np.int64))]
        sample = np.array(sorted(set(chosen) | set(fill)))
        assert len(sample) >= 256
        ref = oracle.moe_tokens(x_bits[sample], wr_bits, expert_weights, k, norm, shared=shared)
        same = (ref["idx"] == idx_gpu[sample]).all(axis=1)
        # grid: exact logits, identical routing; uniform: the fp32 order may flip a
        # near-tie (the stage-wise check above covers those tokens' routing)
        assert same.mean() >= (1.0 if dist == "grid" else 0.97), (dist, same.mean())
        assert len(set(idx_gpu[sample][same].reshape(-1).tolist())) == E
        assert_close(y[sample].float().cpu().numpy()[same], ref["y"][same], f"{name}/{dist}")
        layer.close()
        del x, y, layer
        torch.cuda.empty_cache()


@pytest.mark.parametrize("name,skew,fp8", [("dsv2", 0.0, False), ("mixtral", 0.0, False), ("dsv2", 1.0, True)])
def test_full_size_ep8_on_one_gpu(name, skew, fp8):
    """BASELINE's EP = 8 configuration at full size, the eight ranks as eight
    layers on one B200 (in-process group), planner-chosen plan (Mixtral: one
    expert per rank, so token slices), both all2all data planes: y == the EP = 1
    layer's y, bit for bit, on every token.  Also under skewed (Zipf-like)
    routing with the FP8 dispatch payload (R15: EP = D == EP = 1 holds in FP8)."""
    from gen import router_skew_bias
    import threading

    from paper_2410_12247_b200 import LocalGroup
    c = CONFIGS[name]
    E, k, H, F, S, Fs, T, norm = c["E"], c["k"], c["H"], c["F"], c["S"], c["Fs"], c["T"], c["norm_topk"]
    D, E_loc = 8, c["E"] // 8
    sH, sF = unif_scale(H), unif_scale(F)
    w = dict(w_router=_gen((E, H), TID_WR, 0, MODE_UNIF, sH), w_gate=_gen((E, F, H), TID_WGATE, 0, MODE_UNIF, sH),
             w_up=_gen((E, F, H), TID_WUP, 0, MODE_UNIF, sH), w_down=_gen((E, H, F), TID_WDOWN, 0, MODE_UNIF, sF))
    SF = S * Fs
    if SF:
        w.update(ws_gate=_gen((SF, H), TID_WS_GATE, 0, MODE_UNIF, sH), ws_up=_gen((SF, H), TID_WS_UP, 0, MODE_UNIF, sH),
                 ws_down=_gen((H, SF), TID_WS_DOWN, 0, MODE_UNIF, unif_scale(SF)))
    x = _gen((T, H), TID_X, 0, MODE_UNIF, unif_scale(1))
    if skew:
        w["router_bias"] = torch.from_numpy(router_skew_bias(E, skew, SEED)).cuda()
    ref_layer = MoELayer(E, k, H, F, w, S=S, Fs=Fs, max_tokens=T, norm_topk=norm, dispatch_fp8=fp8)
    y1 = ref_layer.forward(x)
    torch.cuda.synchronize()
    y1 = y1.cpu()
    ref_layer.close()
    del ref_layer
    start = oracle.token_shards(T, D)
    for p2p in (0, 1, 2):   # NCCL-path layout (in-process transport), put kernels, copy engines
        group = LocalGroup(D)
        layers = []
        for r in range(D):
            wr = {n: t for n, t in w.items() if n not in ("w_gate", "w_up", "w_down")}
            for n in ("w_gate", "w_up", "w_down"):
                wr[n] = w[n][r * E_loc:(r + 1) * E_loc]
            layers.append(MoELayer(E, k, H, F, wr, S=S, Fs=Fs, ep=D, rank=r, max_tokens=int(np.diff(start).max()),
                                   norm_topk=norm, local_group=group, a2a_p2p=p2p, dispatch_fp8=fp8))
        ys, plans, errs = [None] * D, [None] * D, []

        def worker(r):
            try:
                torch.cuda.set_device(0)
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    d, b = layers[r].debug_buffers(int(start[r + 1] - start[r]))
                    ys[r] = layers[r].forward(x[start[r]:start[r + 1]], stream=s, debug=d)
                    s.synchronize()
                    plans[r] = b["plan_used"].as_dict()
            except Exception as e:  # pragma: no cover
                errs.append(repr(e))

        th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(D)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        assert not errs, errs
        assert all(p == plans[0] for p in plans)          # every rank ran the same plan
        print(f"{name} skew={skew} fp8={fp8} EP8 p2p={p2p} plan: chunks={plans[0]['num_chunks']} slices={plans[0]['token_slices']} "
              f"groups={plans[0]['group_begin']}")
        y = torch.cat([v.cpu() for v in ys])
        assert torch.equal(y, y1), f"{name} skew={skew} fp8={fp8} EP8 p2p={p2p} plan={plans[0]}"
        for L in layers:
            L.close()
        del layers, ys
        torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["dsv2_decode", "mixtral_decode"])
def test_decode_configs_graph_replay_vs_oracle(name):
    """The decode-regime bench lines (256 tokens, DSv2 / Mixtral dims) in the
    launch configuration bench.py times them: one forward captured in a CUDA
    graph with the host-planned plan, replayed.  The replay's y equals an eager
    forward's y bit for bit; routing stage-wise on all tokens (the oracle's
    top-k of the GPU's fp32 logits); y on ALL 256 tokens vs oracle.moe_tokens
    within the north-star tolerance."""
    c = CONFIGS[name]
    E, k, H, F, S, Fs, T, norm = c["E"], c["k"], c["H"], c["F"], c["S"], c["Fs"], c["T"], c["norm_topk"]
    sH, sF = unif_scale(H), unif_scale(F)
    w = dict(w_router=_gen((E, H), TID_WR, 0, MODE_UNIF, sH), w_gate=_gen((E, F, H), TID_WGATE, 0, MODE_UNIF, sH),
             w_up=_gen((E, F, H), TID_WUP, 0, MODE_UNIF, sH), w_down=_gen((E, H, F), TID_WDOWN, 0, MODE_UNIF, sF))
    SF = S * Fs
    if SF:
        w.update(ws_gate=_gen((SF, H), TID_WS_GATE, 0, MODE_UNIF, sH), ws_up=_gen((SF, H), TID_WS_UP, 0, MODE_UNIF, sH),
                 ws_down=_gen((H, SF), TID_WS_DOWN, 0, MODE_UNIF, unif_scale(SF)))
    x = _gen((T, H), TID_X, 0, MODE_UNIF, unif_scale(1))
    _spot_check(x, TID_X, 0, MODE_UNIF, unif_scale(1))
    layer = MoELayer(E, k, H, F, w, S=S, Fs=Fs, max_tokens=T, norm_topk=norm)
    plan = layer.plan(T)
    y = torch.empty_like(x)
    layer.forward(x, y, plan=plan)          # warm-up, as bench.py does before capturing
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        layer.forward(x, y, plan=plan)
    y.zero_()
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    y_graph = y.clone()
    d, b = layer.debug_buffers(T)
    y_eager = layer.forward(x, plan=plan, debug=d)
    torch.cuda.synchronize()
    assert torch.equal(y_graph, y_eager)
    idx_gpu = b["topk_idx"].cpu().numpy()
    st_idx, st_w = oracle.topk_gating(b["logits"].cpu().numpy(), k, norm)
    assert np.array_equal(idx_gpu, st_idx)
    assert np.allclose(b["topk_w"].cpu().numpy(), st_w, rtol=1e-5, atol=0)
    shared = (_bits(w["ws_gate"]), _bits(w["ws_up"]), _bits(w["ws_down"])) if SF else None
    cache = {}

    def expert_weights(e):
        if e not in cache:
            cache.clear()
            cache[e] = (_bits(w["w_gate"][e]), _bits(w["w_up"][e]), _bits(w["w_down"][e]))
        return cache[e]
    ref = oracle.moe_tokens(_bits(x), _bits(w["w_router"]), expert_weights, k, norm, shared=shared)
    same = (ref["idx"] == idx_gpu).all(axis=1)
    assert same.mean() >= 0.97, same.mean()
    assert_close(y_graph.float().cpu().numpy()[same], ref["y"][same], name)
    layer.close()
