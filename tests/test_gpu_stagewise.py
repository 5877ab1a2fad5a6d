"""Stage-wise parity (SURVEY §8(c) "What pins each part"): each stage of the
CUDA path is fed to the oracle's implementation of the NEXT stage, so results
that must be unique are compared bit for bit even where an earlier stage's
floating point (fp32 accumulation order of the router GEMM) makes the
end-to-end comparison tolerance-only.

  * routing: oracle.topk_gating applied to the GPU's own fp32 logits must equal
    the GPU's indices bit for bit and its weights within 1e-5 (R5), on the
    uniform (full-mantissa) distribution, where logits are not exact;
  * combine: oracle.combine on the GPU's (o, s, w, pos) must equal the GPU's y
    bit for bit (R4: the same fp32 fmaf chain in slot order), for the default
    kernel, both fused EP = 1 variants and the EP > 1 combine buffer;
  * NaN inputs (R18), the DENSE fused-combine launch order, and the SM-partition
    probe (NEXT-1)."""
import threading

import numpy as np
import pytest
import torch

import oracle
from gen import Inputs
from paper_2410_12247_b200 import MOE_GEMM_DENSE, MOE_GEMM_GROUPED, LocalGroup, MoELayer, make_plan

from .gpu_util import assert_close, dev_bf16, layer_from_inputs, to_f32

pytestmark = pytest.mark.gpu


def _bf16_bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def stagewise_combine_ref(bufs, T, k, s_bits=None):
    """oracle.combine on the GPU's stage inputs: o rows at the send rows
    (combine_in[pos[t][j]]), s (bf16) or zeros, the GPU's w."""
    o = oracle.bf16_bits_to_f64(_bf16_bits(bufs["combine_in"])).astype(np.float32)
    pos = bufs["pos"].cpu().numpy()
    w = bufs["topk_w"].cpu().numpy()
    H = o.shape[1]
    o_slots = o[pos.reshape(-1)].reshape(T, k, H)
    s = oracle.bf16_bits_to_f64(s_bits).astype(np.float32) if s_bits is not None else np.zeros((T, H), np.float32)
    return oracle.combine(s, o_slots, w)


def stagewise_routing_check(logits, idx, w, k, norm, **rg):
    ref_idx, ref_w = oracle.topk_gating(logits, k, norm, **rg)
    assert np.array_equal(idx, ref_idx)
    assert np.allclose(w, ref_w, rtol=1e-5, atol=0)


CASES = {
    "mid_shared": (dict(E=16, k=4, H=512, F=384, S=1, Fs=256), 4, 0),
    "e160_k6": (dict(E=160, k=6, H=256, F=128, S=2, Fs=128), 6, 0),
    "mixtral_like": (dict(E=8, k=2, H=512, F=256), 2, 1),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("T", [333, 9000])
def test_stagewise_routing_uniform(name, T):
    """Full-mantissa inputs: the GPU's logits differ from the oracle's in the
    last fp32 bits (accumulation order), so routing is checked stage-wise on
    ALL tokens, bit-exact; y within tolerance where the routing agrees."""
    kw, k, norm = CASES[name]
    inp = Inputs(seed=101, T=T, **kw)
    L = layer_from_inputs(inp, k, norm)
    d, b = L.debug_buffers(T)
    L.forward(dev_bf16(inp.x), debug=d)
    torch.cuda.synchronize()
    stagewise_routing_check(b["logits"].cpu().numpy(), b["topk_idx"].cpu().numpy(), b["topk_w"].cpu().numpy(),
                            k, norm)
    L.close()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("fuse", ["0", "1", "2"])
def test_stagewise_combine_ep1(name, fuse, monkeypatch):
    """EP = 1: y == oracle.combine(s, o[pos], w) bit for bit, for the combine
    kernel (fuse 0), the shared DownGemm with the combine in its epilogue
    (EPI_COMBINE, fuse 1) and the token-piece overlap (fuse 2).  The fused
    variants never materialise s, so s comes from an unfused forward of the
    same layer (the shared GEMMs are the same launches)."""
    kw, k, norm = CASES[name]
    T = 9000                                   # >= 8192: the side-stream and 4-piece paths
    inp = Inputs(seed=202, T=T, **kw)
    x = dev_bf16(inp.x)
    monkeypatch.setenv("EPSMOE_FUSE_COMBINE", fuse)
    L = layer_from_inputs(inp, k, norm)
    s_bits = None
    if inp.S:
        d0, b0 = L.debug_buffers(T)            # shared_out requested: unfused path
        L.forward(x, debug=d0)
        torch.cuda.synchronize()
        s_bits = _bf16_bits(b0["shared_out"])
    d, b = L.debug_buffers(T, combine_in=True)
    d.shared_out = None                        # keep the fused path
    y = L.forward(x, debug=d)
    torch.cuda.synchronize()
    ref = stagewise_combine_ref(b, T, k, s_bits)
    assert np.array_equal(_bf16_bits(y), oracle.bf16_value_to_bits(ref))
    L.close()


def _ep_run(inp, k, norm, D, plan, p2p, combine_in=True):
    E = inp.E
    E_loc = E // D
    start = oracle.token_shards(inp.T, D)
    group = LocalGroup(D)
    layers = []
    for r in range(D):
        w = dict(w_router=dev_bf16(inp.w_router), w_gate=dev_bf16(inp.w_gate[r * E_loc:(r + 1) * E_loc]),
                 w_up=dev_bf16(inp.w_up[r * E_loc:(r + 1) * E_loc]),
                 w_down=dev_bf16(inp.w_down[r * E_loc:(r + 1) * E_loc]))
        if inp.S:
            w.update(ws_gate=dev_bf16(inp.ws_gate), ws_up=dev_bf16(inp.ws_up), ws_down=dev_bf16(inp.ws_down))
        layers.append(MoELayer(E, k, inp.H, inp.F, w, S=inp.S, Fs=inp.Fs, ep=D, rank=r,
                               max_tokens=int(np.diff(start).max()), norm_topk=norm, local_group=group, a2a_p2p=p2p))
    ys, bufs, errs = [None] * D, [None] * D, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                T_loc = int(start[r + 1] - start[r])
                d, b = layers[r].debug_buffers(T_loc, combine_in=combine_in)
                ys[r] = layers[r].forward(dev_bf16(inp.x[start[r]:start[r + 1]]), plan=plan, stream=s, debug=d)
                s.synchronize()
                bufs[r] = b
        except Exception as e:  # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(D)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=180)
    assert not errs, errs
    for L in layers:
        L.close()
    return ys, bufs, start


@pytest.mark.parametrize("p2p", [0, 1, 2])
@pytest.mark.parametrize("D,N", [(2, 3), (4, 2)])
def test_stagewise_combine_and_routing_ep(D, N, p2p):
    """EP > 1: on every rank, routing stage-wise vs its logits and y ==
    oracle.combine(s, comb[pos], w) bit for bit, where comb is the combine
    buffer the all2all (NCCL-path layout, put kernels with the fused DownGemm
    scatter, or copy engines) filled."""
    kw, k, norm = CASES["mid_shared"]
    inp = Inputs(seed=303 + D, T=1501, **kw)
    ys, bufs, start = _ep_run(inp, k, norm, D, make_plan(N, MOE_GEMM_GROUPED), p2p)
    for r in range(D):
        b = bufs[r]
        T_loc = int(start[r + 1] - start[r])
        stagewise_routing_check(b["logits"].cpu().numpy(), b["topk_idx"].cpu().numpy(), b["topk_w"].cpu().numpy(),
                                k, norm)
        ref = stagewise_combine_ref(b, T_loc, k, _bf16_bits(b["shared_out"]))
        assert np.array_equal(_bf16_bits(ys[r]), oracle.bf16_value_to_bits(ref)), r


@pytest.mark.parametrize("p2p", [1, 2])
def test_dense_chunks_with_fused_combine_flags(p2p, monkeypatch):
    """a chunk of several DENSE experts runs as one DownGemm
    launch per expert; with the fused peer-memory combine only the LAST launch
    may raise the chunk's flags.  N < E_loc so chunks hold several experts; y ==
    EP = 1 bit for bit, over repeated forwards (stale rows would differ)."""
    monkeypatch.setenv("EPSMOE_P2P_FUSE", "1")
    inp = Inputs(E=16, k=4, H=256, F=256, S=1, Fs=128, T=997, seed=404, grid=True)
    plan = make_plan(2, MOE_GEMM_DENSE)          # E_loc = 4 (D = 4): 2 experts per chunk
    ys, bufs, start = _ep_run(inp, 4, 0, 4, plan, p2p, combine_in=False)
    L1 = layer_from_inputs(inp, 4, 0)
    y1 = L1.forward(dev_bf16(inp.x), plan=make_plan(1, MOE_GEMM_DENSE))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([y.cpu() for y in ys]), y1.cpu())
    L1.close()


def test_nan_token_and_nan_logit_r18():
    """a token whose x holds a NaN gets all-NaN logits,
    selects experts 0..k-1 with NaN weights and a NaN y row, with no fault; the
    other tokens' y are bit-identical to the run without it.  A NaN router bias
    (a NaN logit of one expert) is never selected (oracle R18)."""
    kw, k, norm = CASES["mid_shared"]
    T = 700
    inp = Inputs(seed=505, T=T, **kw)
    L = layer_from_inputs(inp, k, norm)
    x = dev_bf16(inp.x)
    y_ref = L.forward(x).clone()
    xn = x.clone()
    xn[123, 7] = float("nan")
    d, b = L.debug_buffers(T)
    y = L.forward(xn, debug=d)
    torch.cuda.synchronize()
    idx = b["topk_idx"].cpu().numpy()
    assert idx[123].tolist() == list(range(k))
    assert torch.isnan(b["topk_w"][123]).all() and torch.isnan(y[123].float()).all()
    keep = torch.ones(T, dtype=torch.bool)
    keep[123] = False
    assert torch.equal(y[keep.cuda()], y_ref[keep.cuda()])
    assert (idx >= 0).all() and (idx < inp.E).all()
    L.close()
    # one expert's logit NaN for every token (router bias): never selected
    bias = np.zeros(inp.E, np.float32)
    bias[3] = np.nan
    inp.router_bias = bias
    L = layer_from_inputs(inp, k, norm)
    d, b = L.debug_buffers(T)
    L.forward(x, debug=d)
    torch.cuda.synchronize()
    idx = b["topk_idx"].cpu().numpy()
    assert not (idx == 3).any()
    stagewise_routing_check(b["logits"].cpu().numpy(), idx, b["topk_w"].cpu().numpy(), k, norm)
    L.close()


def test_sm_partition_probe_ep1():
    """NEXT-1: with a plan's GEMM grid below the SM count, no more than sm_gemm
    persistent GEMM CTAs of the forward are ever resident together (shared
    experts, chunked routed GEMMs): the kernels count themselves in
    moe_debug_t.gemm_resident.  With all SMs, the count reaches the SM count."""
    kw, k, norm = CASES["e160_k6"]
    inp = Inputs(seed=606, T=20000, **kw)
    L = layer_from_inputs(inp, k, norm)
    x = dev_bf16(inp.x)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for sm in (100, 132, nsm):
        d, b = L.debug_buffers(inp.T)
        L.forward(x, plan=make_plan(4, MOE_GEMM_GROUPED, sm_gemm=sm), debug=d)
        torch.cuda.synchronize()
        cur, mx = b["gemm_resident"].cpu().tolist()
        assert cur == 0 and 0 < mx <= sm, (sm, mx)
        assert b["plan_used"].sm_gemm == sm
    L.close()


def test_sm_partition_from_the_cost_model_ep2():
    """NEXT-1 at EP = 2 (in-process group, put-kernel plane): the plan the
    forward runs takes (sm_gemm, comm_ctas) from the installed cost model - a
    model where SMs are precious gives 4 CTAs per communicator, one where the
    all2all dominates gives 16 - identical on both ranks, and the probe shows
    no more than sm_gemm GEMM CTAs resident (shared experts and chunk GEMMs
    serialised on one stream)."""
    from paper_2410_12247_b200 import abi
    D, k, norm = 2, 4, 0
    inp = Inputs(E=16, k=4, H=512, F=384, S=1, Fs=256, T=6000, seed=707, grid=True)
    E_loc = 8
    start = oracle.token_shards(inp.T, D)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count

    def model(scales, rates, gemm):
        c = abi.moe_cost_model_t()
        c.n_points = 2
        c.m_points[0], c.m_points[1] = 100.0, 10000.0
        for kind in (0, 1):
            c.gemm_ms[kind][0], c.gemm_ms[kind][1] = gemm * 0.01, gemm
        c.a2a_fixed_ms, c.k_ms, c.b_ms = 0.01, 0.02, 0.0
        c.num_sms, c.n_comm = nsm, 4
        for i, (cc, s, r) in enumerate(zip((4, 8, 12, 16), scales, rates)):
            c.comm_ctas[i], c.gemm_scale_at[i], c.a2a_gbps_at[i] = cc, s, r
        c.a2a_gbps = max(rates)
        return c
    models = {4: model((1.06, 1.12, 1.19, 1.27), (700, 700, 700, 700), 1.0),
              16: model((1.03, 1.06, 1.09, 1.12), (1, 2, 4, 8), 0.05)}
    group = LocalGroup(D)
    layers = []
    for r in range(D):
        w = dict(w_router=dev_bf16(inp.w_router), w_gate=dev_bf16(inp.w_gate[r * E_loc:(r + 1) * E_loc]),
                 w_up=dev_bf16(inp.w_up[r * E_loc:(r + 1) * E_loc]),
                 w_down=dev_bf16(inp.w_down[r * E_loc:(r + 1) * E_loc]),
                 ws_gate=dev_bf16(inp.ws_gate), ws_up=dev_bf16(inp.ws_up), ws_down=dev_bf16(inp.ws_down))
        layers.append(MoELayer(16, k, 512, 384, w, S=1, Fs=256, ep=D, rank=r, max_tokens=3000, norm_topk=norm,
                               local_group=group, a2a_p2p=1))
    L1 = layer_from_inputs(inp, k, norm)
    y1 = L1.forward(dev_bf16(inp.x), plan=make_plan(1, MOE_GEMM_GROUPED)).cpu()
    L1.close()
    for want, m in models.items():
        out, errs = [None] * D, []

        def worker(r):
            try:
                torch.cuda.set_device(0)
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    layers[r].set_cost_model(m)
                    d, b = layers[r].debug_buffers(int(start[r + 1] - start[r]))
                    y = layers[r].forward(dev_bf16(inp.x[start[r]:start[r + 1]]), stream=s, debug=d)
                    s.synchronize()
                    out[r] = (y.cpu(), b["plan_used"].as_dict(), b["gemm_resident"].cpu().tolist())
            except Exception as e:  # pragma: no cover
                errs.append(repr(e))

        th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(D)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=180)
        assert not errs, errs
        plans = [o[1] for o in out]
        assert all(p == plans[0] for p in plans)
        assert plans[0]["comm_ctas"] == want and plans[0]["sm_gemm"] == nsm - 2 * want, plans[0]
        for y, p, (cur, mx) in out:
            assert cur == 0 and 0 < mx <= p["sm_gemm"], (p, mx)
        # GROUPED vs AUTO kinds and chunking never change a bit (R6, tile-shape neutrality)
        assert torch.equal(torch.cat([o[0] for o in out]), y1)
    for L in layers:
        L.close()
