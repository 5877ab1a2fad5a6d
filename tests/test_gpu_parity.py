"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Integer artefacts bit-exact; outputs within the north-star
tolerance (max|err| <= 1e-2 max|ref|, mean rel <= 2e-3)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from gen import MODE_GRID, MODE_UNIF, Inputs, fill_bf16
from paper_2410_12247_b200 import MOE_GEMM_DENSE, MOE_GEMM_GROUPED, gemm_grouped, make_plan

from .gpu_util import assert_close, dev_bf16, layer_from_inputs, to_f32

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_device_generator_matches_numpy():
    from gen import device_fill_bf16
    for mode, param in [(MODE_UNIF, 0.0382), (MODE_GRID, 8.0), (MODE_GRID, 64.0)]:
        n, base = 100003, 12345678
        t = torch.empty(n, dtype=torch.int16, device="cuda")
        device_fill_bf16(t.data_ptr(), n, 20241016, 3, base, mode, param)
        torch.cuda.synchronize()
        ref = fill_bf16(n, 20241016, 3, base, mode, param)
        assert np.array_equal(t.cpu().numpy().view(np.uint16), ref)


# ---------------------------------------------------------------- GEMM family

def _rows_ref_swiglu(A, Wg, Wu):
    g = (oracle.bf16_bits_to_f64(A) @ oracle.bf16_bits_to_f64(Wg).T).astype(np.float32)
    u = (oracle.bf16_bits_to_f64(A) @ oracle.bf16_bits_to_f64(Wu).T).astype(np.float32)
    return oracle.round_bf16(oracle.silu_f32(g) * u)


@pytest.mark.parametrize("tile_m", [128, 256])
@pytest.mark.parametrize("counts", [[300, 0, 129, 1, 128], [5], [1000, 777], [257, 255, 511, 3]])
def test_grouped_gemm_swiglu_and_down(counts, tile_m):
    H, F = 256, 384
    G = len(counts)
    rng_rows = sum(counts)
    A = fill_bf16(rng_rows * H, 1, 1, 0, MODE_UNIF, 1.7).reshape(rng_rows, H)
    Wg = fill_bf16(G * F * H, 1, 3, 0, MODE_UNIF, 0.1).reshape(G * F, H)
    Wu = fill_bf16(G * F * H, 1, 4, 0, MODE_UNIF, 0.1).reshape(G * F, H)
    Wd = fill_bf16(G * H * F, 1, 5, 0, MODE_UNIF, 0.08).reshape(G * H, F)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    rs = torch.from_numpy(starts).cuda()
    rc = torch.from_numpy(np.array(counts, np.int32)).cuda()
    h = torch.zeros(rng_rows, F, dtype=torch.bfloat16, device="cuda")
    gemm_grouped(0, dev_bf16(A), dev_bf16(Wg), dev_bf16(Wu), F, h, rs, rc, F, tile_m=tile_m)
    o = torch.zeros(rng_rows, H, dtype=torch.bfloat16, device="cuda")
    gemm_grouped(1, h, dev_bf16(Wd), None, H, o, rs, rc, H, tile_m=tile_m)
    torch.cuda.synchronize()
    h_np, o_np = to_f32(h), to_f32(o)
    for g in range(G):
        a, b = starts[g], starts[g] + counts[g]
        if a == b:
            continue
        ref_h = _rows_ref_swiglu(A[a:b], Wg[g * F:(g + 1) * F], Wu[g * F:(g + 1) * F])
        assert_close(h_np[a:b], ref_h, f"h group {g}")
        # down GEMM checked on the GPU's own h (stage-wise) -> bit-level rounding only
        ref_o = oracle.round_bf16((h_np[a:b].astype(np.float64) @
                                   oracle.bf16_bits_to_f64(Wd[g * H:(g + 1) * H]).T).astype(np.float32))
        assert_close(o_np[a:b], ref_o, f"o group {g}")


def test_tile_shape_does_not_change_bits():
    """R14 picks the tile shape by load (128-row tiles on one CTA, cta_group::1,
    or 256-row tiles on a CTA pair, cta_group::2).  Every output element is the
    same k-ordered chain of K = 16 tensor-core steps either way, so the choice
    must not change a bit (the EP = D == EP = 1 and chunked == unchunked claims
    rely on it when shapes differ): all three epilogues, ragged groups."""
    H, F = 512, 384
    counts = [700, 0, 129, 1, 300]
    G, rows = len(counts), sum(counts)
    A = dev_bf16(fill_bf16(rows * H, 2, 1, 0, MODE_UNIF, 1.7).reshape(rows, H))
    Wg = dev_bf16(fill_bf16(G * F * H, 2, 3, 0, MODE_UNIF, 0.1).reshape(G * F, H))
    Wu = dev_bf16(fill_bf16(G * F * H, 2, 4, 0, MODE_UNIF, 0.1).reshape(G * F, H))
    Wd = dev_bf16(fill_bf16(G * H * F, 2, 5, 0, MODE_UNIF, 0.08).reshape(G * H, F))
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    rs = torch.from_numpy(starts).cuda()
    rc = torch.from_numpy(np.array(counts, np.int32)).cuda()
    out = {}
    for tm in (128, 256):
        h = torch.zeros(rows, F, dtype=torch.bfloat16, device="cuda")
        gemm_grouped(0, A, Wg, Wu, F, h, rs, rc, F, tile_m=tm)
        o = torch.zeros(rows, H, dtype=torch.bfloat16, device="cuda")
        gemm_grouped(1, h, Wd, None, H, o, rs, rc, H, tile_m=tm)
        lg = torch.zeros(rows, 160, dtype=torch.float32, device="cuda")   # router: fp32 epilogue, N = E padded
        Wr = dev_bf16(fill_bf16(256 * H, 2, 2, 0, MODE_UNIF, 0.05).reshape(256, H))
        one_s = torch.zeros(1, dtype=torch.int32, device="cuda")
        one_c = torch.full((1,), rows, dtype=torch.int32, device="cuda")
        gemm_grouped(2, A, Wr, None, 160, lg, one_s, one_c, 0, tile_m=tm)
        torch.cuda.synchronize()
        out[tm] = (h, o, lg)
    for a, b, name in zip(out[128], out[256], ("h", "o", "logits")):
        assert torch.equal(a, b), name


@pytest.mark.parametrize("tile_m", [128, 256])
def test_router_gemm_exact_on_grid(tile_m):
    T, H, E = 333, 512, 160
    x = fill_bf16(T * H, 2, 1, 0, MODE_GRID, 8.0).reshape(T, H)
    wr = fill_bf16(256 * H, 2, 2, 0, MODE_GRID, 64.0).reshape(256, H)
    bias = np.linspace(-1, 1, E).astype(np.float32)
    out = torch.zeros(T, E, dtype=torch.float32, device="cuda")
    rs = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = torch.full((1,), T, dtype=torch.int32, device="cuda")
    gemm_grouped(2, dev_bf16(x), dev_bf16(wr), None, E, out, rs, rc, 0, bias=torch.from_numpy(bias).cuda(),
                 tile_m=tile_m)
    torch.cuda.synchronize()
    ref = oracle.router_logits(x, wr[:E], bias)
    assert np.array_equal(out.cpu().numpy(), ref)


def test_gate_interleaved_tokens_bit_identical():
    """The gate kernel takes 4 tokens of a routing range at a time with the same
    per-token operations (EPSMOE_GATE_U=1, default) as the one-token loop: indices
    and weights bit-identical, at range lengths 1 (T = 1000, remainder path
    only), 8 and 32 (16 000 and 40 000 tokens), in a subprocess per setting (the
    switch is read once per process)."""
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from gen import Inputs
from tests.gpu_util import layer_from_inputs, dev_bf16
out = []
for T in (1000, 16000, 40000):
    inp = Inputs(E=160, k=6, H=256, F=128, T=T, seed=9)
    L = layer_from_inputs(inp, 6, 0)
    d, b = L.debug_buffers(T)
    L.forward(dev_bf16(inp.x), debug=d)
    torch.cuda.synchronize()
    out += [b["topk_idx"].cpu().numpy(), b["topk_w"].cpu().numpy().view(np.uint32), b["pos"].cpu().numpy()]
    L.close()
np.savez(sys.argv[1], *out)
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    res = []
    with tempfile.TemporaryDirectory() as td:
        for u in ("1", "0"):
            f = os.path.join(td, f"g{u}.npz")
            env = dict(os.environ, EPSMOE_GATE_U=u)
            subprocess.run([sys.executable, "-c", code, f], check=True, env=env, timeout=300)
            z = np.load(f)
            res.append([z[n] for n in z.files])
    for a, b in zip(*res):
        assert np.array_equal(a, b)


def test_tile_scheduling_is_bit_neutral():
    """Tile scheduling decides only WHICH CTA pair computes a tile and when, never
    a sum order: dynamic tickets published a tile ahead (default), published when
    loaded (EPSMOE_TICKET_AHEAD=0), static round robin for every GEMM
    (EPSMOE_DYN_SCHED=0) and for the DownGemm only (=2) give bit-identical h-path
    outputs: the layer's y (routed GEMMs, shared experts, router) on a DSv2-like
    layer, in a subprocess per setting (the switches are read once per process)."""
    import subprocess
    import sys
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from gen import Inputs
from tests.gpu_util import layer_from_inputs, dev_bf16
inp = Inputs(E=32, k=6, H=512, F=256, S=2, Fs=128, T=3000, seed=12)
L = layer_from_inputs(inp, 6, 0)
y = L.forward(dev_bf16(inp.x))
torch.cuda.synchronize()
np.save(sys.argv[1], y.view(torch.int16).cpu().numpy())
L.close()
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import tempfile
    res = []
    with tempfile.TemporaryDirectory() as td:
        for i, kv in enumerate([{}, {"EPSMOE_TICKET_AHEAD": "0"}, {"EPSMOE_DYN_SCHED": "0"},
                                {"EPSMOE_DYN_SCHED": "2"}]):
            f = os.path.join(td, f"y{i}.npy")
            subprocess.run([sys.executable, "-c", code, f], check=True, env=dict(os.environ, **kv), timeout=300)
            res.append(np.load(f))
    for r in res[1:]:
        assert np.array_equal(res[0], r)


# ---------------------------------------------------------------- full layer (EP = 1)

CASES = {
    # name: (Inputs kwargs, k, norm)
    "tiny": (dict(E=8, k=2, H=64, F=128, T=256), 2, 1),
    "mid_shared": (dict(E=16, k=4, H=512, F=384, S=1, Fs=256, T=1000), 4, 0),
    "e160_k6": (dict(E=160, k=6, H=256, F=128, S=2, Fs=128, T=700), 6, 0),
}


def _run_layer(inp, k, norm, plan=None, dbg=True):
    L = layer_from_inputs(inp, k, norm)
    x = dev_bf16(inp.x)
    d, bufs = L.debug_buffers(inp.T) if dbg else (None, None)
    y = L.forward(x, plan=plan, debug=d)
    torch.cuda.synchronize()
    return L, y, bufs


@pytest.mark.parametrize("name", list(CASES))
def test_layer_parity_grid(name):
    kw, k, norm = CASES[name]
    inp = Inputs(seed=31, grid=True, **kw)
    L, y, b = _run_layer(inp, k, norm)
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=norm,
                           ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
    # exact-logit grid: logits and routing bit-exact
    assert np.array_equal(b["logits"].cpu().numpy(), ref["logits"])
    assert np.array_equal(b["topk_idx"].cpu().numpy(), ref["idx"])
    w = b["topk_w"].cpu().numpy()
    assert np.allclose(w, ref["w"], rtol=1e-5, atol=0)
    lay = ref["layout"]
    assert np.array_equal(b["hist"].cpu().numpy(), lay["hist"][0])
    assert np.array_equal(b["seg_start"].cpu().numpy(), lay["send_start"][0])
    assert np.array_equal(b["pos"].cpu().numpy(), lay["pos"][0])
    assert np.array_equal(b["global_hist"][0], lay["hist"][0])
    if inp.S:
        assert_close(to_f32(b["shared_out"]), ref["s"], "shared")
    assert_close(to_f32(y), ref["y"], name)
    assert L.last_launches() > 0


@pytest.mark.parametrize("H,skew", [(1088, 0.0), (2048, 1.0), (5120, 1.0)])
def test_router_exact_on_grid_large_h_with_bias(H, skew):
    """Layer-level exact-logit grid check at production-size K (H = 1088: 17
    k-blocks; 2048; 5120 = DSv2's 80 k-blocks), with and without the skew bias:
    on the grid every fp32 partial sum is exact, so the GPU's logits equal the
    oracle's fp32(sum) + beta bit for bit; routing, layout and y as in the grid
    test above.  (Also the parity gate of the split-K router variant,
    tools/r02/router_ksplit.patch, measured and dropped: DESIGN §12.)"""
    E, k = 32, 4
    inp = Inputs(E=E, k=k, H=H, F=128, T=600, seed=41, grid=True, skew=skew)
    L, y, b = _run_layer(inp, k, 0)
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=0,
                           router_bias=inp.router_bias)
    assert np.array_equal(b["logits"].cpu().numpy(), ref["logits"])
    assert np.array_equal(b["topk_idx"].cpu().numpy(), ref["idx"])
    assert np.allclose(b["topk_w"].cpu().numpy(), ref["w"], rtol=1e-5, atol=0)
    assert np.array_equal(b["pos"].cpu().numpy(), ref["layout"]["pos"][0])
    assert_close(to_f32(y), ref["y"], f"H={H} skew={skew}")


@pytest.mark.parametrize("name", ["mid_shared", "e160_k6"])
def test_layer_parity_uniform(name):
    kw, k, norm = CASES[name]
    inp = Inputs(seed=77, **kw)
    L, y, b = _run_layer(inp, k, norm)
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=norm,
                           ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
    idx = b["topk_idx"].cpu().numpy()
    same = (idx == ref["idx"]).all(axis=1)
    assert same.mean() >= 0.999                 # fp32 accumulation order may flip a near-tie
    assert_close(to_f32(y)[same], ref["y"][same], name)


def test_chunked_equals_unchunked_and_kinds():
    kw, k, norm = CASES["e160_k6"]
    inp = Inputs(seed=5, **kw)
    L = layer_from_inputs(inp, k, norm)
    x = dev_bf16(inp.x)
    ys = []
    for n, kind, tm in [(1, MOE_GEMM_GROUPED, 128), (3, MOE_GEMM_GROUPED, 256), (7, MOE_GEMM_GROUPED, 128),
                        (1, MOE_GEMM_DENSE, 256), (4, MOE_GEMM_DENSE, 128), (1, MOE_GEMM_GROUPED, 256)]:
        ys.append(L.forward(x, plan=make_plan(n, kind, tile_m=tm)).clone())
    torch.cuda.synchronize()
    for v in ys[1:]:
        assert torch.equal(v, ys[0])


@pytest.mark.parametrize("tile_m", [128, 256])
def test_gathered_gateup_equals_materialised_split(tile_m, monkeypatch):
    """ep == 1: GateUp reading x through TMA tile::gather4 == reading the
    materialised expert-major send buffer, bit for bit."""
    kw, k, norm = CASES["mid_shared"]
    inp = Inputs(seed=12, **kw)
    x = dev_bf16(inp.x)
    ys = []
    for g in ("0", "1"):
        monkeypatch.setenv("EPSMOE_GATHER", g)
        L = layer_from_inputs(inp, k, norm)
        ys.append(L.forward(x, plan=make_plan(1, MOE_GEMM_GROUPED, tile_m=tile_m)).clone())
        torch.cuda.synchronize()
        L.close()
    assert torch.equal(ys[0], ys[1])


def test_fig_eps_overview_explicit_routing():
    fx = json.load(open(os.path.join(GOLDEN, "fig_eps_overview.json")))
    idx = np.array(fx["routing"], np.int32)
    w = np.array(fx["weights"], np.float32)
    inp = Inputs(E=6, k=2, H=64, F=128, T=10, seed=1)
    L = layer_from_inputs(inp, 2, 0)
    d, b = L.debug_buffers(10, override=(torch.from_numpy(idx), torch.from_numpy(w)))
    y = L.forward(dev_bf16(inp.x), debug=d)
    torch.cuda.synchronize()
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=2, norm_topk=0,
                           topk_override=(idx, w))
    assert b["hist"].cpu().numpy().tolist() == [4, 4, 3, 3, 3, 3]   # Expert0 [0,1,5,9], Expert1 [0,2,5,6]
    assert np.array_equal(b["pos"].cpu().numpy(), ref["layout"]["pos"][0])
    assert_close(to_f32(y), ref["y"], "fixture")


def test_calibrated_cost_model_drives_plan():
    """moe_layer_calibrate measures GEMM ms per expert vs rows for both kinds
    (the X2/X3 analog on B200); the plan then follows the measured model."""
    inp = Inputs(E=16, k=4, H=512, F=384, T=2000, seed=4)
    L = layer_from_inputs(inp, 4, 0, max_tokens=8192)
    m = L.calibrate()
    assert 3 <= m.n_points <= 12
    pts = list(m.m_points[:m.n_points])
    assert pts == sorted(pts)
    for kind in (0, 1):
        ms = list(m.gemm_ms[kind][:m.n_points])
        assert all(v > 0 for v in ms)
        assert ms[-1] > ms[0]                     # more rows, more time
    p = L.plan(8192)
    assert p.num_chunks == 1                      # ep == 1: nothing to overlap
    assert all(p.expert_kind[e] in (1, 2) for e in range(16))


def test_empty_and_single_token():
    inp = Inputs(E=8, k=2, H=64, F=128, T=1, seed=3)
    L = layer_from_inputs(inp, 2, 1, max_tokens=64)
    x = dev_bf16(inp.x)
    y = L.forward(x)
    torch.cuda.synchronize()
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=2, norm_topk=1)
    assert_close(to_f32(y), ref["y"], "T=1")
    y0 = L.forward(x[:0])
    torch.cuda.synchronize()
    assert y0.shape[0] == 0


def test_cuda_graph_capture_replay():
    """ep == 1 forward has no host synchronisation: it captures into a CUDA
    graph (side stream + events included) and replays bit-identically."""
    kw, k, norm = CASES["mid_shared"]
    inp = Inputs(seed=19, **kw)
    L = layer_from_inputs(inp, k, norm)
    x = dev_bf16(inp.x)
    ref = L.forward(x).clone()
    plan = make_plan(1, MOE_GEMM_GROUPED)
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        L.forward(x, y, plan=plan, stream=s)          # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        L.forward(x, y, plan=plan)
    y.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, ref)


@pytest.mark.parametrize("E,k,H,F,T", [(256, 8, 8192, 128, 300), (2, 1, 64, 128, 33)])
def test_extreme_shapes(E, k, H, F, T):
    """Limits of the ABI: 256 experts, top-8, hidden 8192; and the degenerate
    2-expert top-1 layer (norm_topk -> weight 1)."""
    inp = Inputs(E=E, k=k, H=H, F=F, T=T, seed=23, grid=True)
    L, y, b = _run_layer(inp, k, 1)
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=1)
    assert np.array_equal(b["topk_idx"].cpu().numpy(), ref["idx"])
    assert np.array_equal(b["pos"].cpu().numpy(), ref["layout"]["pos"][0])
    assert_close(to_f32(y), ref["y"], f"E{E} k{k} H{H}")


def test_capacity_and_invalid_errors():
    from paper_2410_12247_b200 import EpsMoeError
    inp = Inputs(E=8, k=2, H=64, F=128, T=40, seed=2)
    L = layer_from_inputs(inp, 2, 1, max_tokens=16)
    with pytest.raises(EpsMoeError, match="CAPACITY"):
        L.forward(dev_bf16(inp.x))


def test_forward_host_sliced_pipeline_matches_device():
    """forward_host splits big batches into token slices (copies overlap the
    layer); rows are independent, so the result equals the one-shot forward."""
    inp = Inputs(E=8, k=2, H=64, F=128, S=1, Fs=128, T=50001, seed=6)
    L = layer_from_inputs(inp, 2, 1, max_tokens=65536)
    x = dev_bf16(inp.x)
    y = L.forward(x)
    xh = x.cpu().pin_memory()
    yh = torch.zeros_like(xh).pin_memory()
    L.forward_host(xh, yh)
    torch.cuda.synchronize()
    assert torch.equal(yh, y.cpu())


def test_forward_host_matches_device():
    kw, k, norm = CASES["mid_shared"]
    inp = Inputs(seed=8, **kw)
    L = layer_from_inputs(inp, k, norm)
    x = dev_bf16(inp.x)
    y = L.forward(x)
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    L.forward_host(xh, yh)
    torch.cuda.synchronize()
    assert torch.equal(yh, y.cpu())


@pytest.mark.parametrize("name,T", [("mid_shared", 1000), ("e160_k6", 700), ("e160_k6", 9000)])
def test_fused_shared_down_combine_equals_unfused(name, T, monkeypatch):
    """ep == 1 with shared experts: the shared DownGemm with the K7 combine in
    its epilogue (EPI_COMBINE, mode 1) and the token-piece overlap (mode 2) ==
    shared DownGemm -> s -> combine kernel (mode 0), bit for bit (same bf16
    rounding of s, same slot-order fmaf chain, R4); T = 9000 takes the
    side-stream and 4-piece paths.  y vs the oracle as well."""
    kw, k, norm = CASES[name]
    kw = dict(kw, T=T)
    inp = Inputs(seed=23, grid=True, **kw)
    x = dev_bf16(inp.x)
    ys = []
    for f in ("0", "1", "2"):
        monkeypatch.setenv("EPSMOE_FUSE_COMBINE", f)
        L = layer_from_inputs(inp, k, norm)
        ys.append(L.forward(x).clone())
        torch.cuda.synchronize()
        L.close()
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2])
    if T <= 1000:
        ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=norm,
                               ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
        assert_close(to_f32(ys[1]), ref["y"], name + " fused")


@pytest.mark.parametrize("E,k,G,M,H", [(16, 4, 4, 2, 256), (160, 6, 8, 3, 256), (64, 6, 8, 1, 128)])
def test_device_limited_routing_exact(E, k, G, M, H):
    """NEXT-4 (R17): group-limited top-k on the exact-logit grid:
    indices bit-exact vs the oracle, every token within M groups, y vs oracle."""
    inp = Inputs(E=E, k=k, H=H, F=128, S=1, Fs=128, T=700, seed=44, grid=True)
    L = layer_from_inputs(inp, k, 1, route_groups=G, route_topk_groups=M)
    d, b = L.debug_buffers(inp.T)
    y = L.forward(dev_bf16(inp.x), debug=d)
    torch.cuda.synchronize()
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=1,
                           ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down,
                           route_groups=G, route_topk_groups=M)
    idx = b["topk_idx"].cpu().numpy()
    assert np.array_equal(idx, ref["idx"])
    assert max(len(set((row // (E // G)).tolist())) for row in idx) <= M
    assert not np.array_equal(idx, oracle.topk_gating(ref["logits"], k, 1)[0])   # the limit bites
    assert_close(to_f32(y), ref["y"], f"device-limited E{E} G{G} M{M}")
    L.close()


def test_forward_host_async_overlapped_calls():
    """moe_layer_forward_host_async: consecutive calls share the double-buffered
    staging (call i+1's copies overlap call i's compute); after host_sync every
    call's y_host equals the device-buffer forward of its x."""
    kw, k, norm = CASES["mid_shared"]
    inps = [Inputs(seed=60 + i, **dict(kw, T=3000)) for i in range(5)]
    base = inps[0]
    L = layer_from_inputs(base, k, norm, max_tokens=3000)
    xs_h = [torch.from_numpy(np.ascontiguousarray(i.x).view(np.int16)).view(torch.bfloat16).pin_memory() for i in inps]
    ys_h = [torch.empty_like(x) .pin_memory() for x in xs_h]
    for xh, yh in zip(xs_h, ys_h):
        L.forward_host_async(xh, yh)
    L.host_sync()
    for xh, yh in zip(xs_h, ys_h):
        ref = L.forward(xh.cuda())
        torch.cuda.synchronize()
        assert torch.equal(yh, ref.cpu())
    L.close()
