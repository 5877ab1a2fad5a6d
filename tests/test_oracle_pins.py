"""Pins for the CPU oracle (oracle/), each against something other than itself:
brute force written independently here, closed forms, library routines,
paper-printed values (tests/golden/), and invariants.  CPU only."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
from gen import Inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _f(bits):
    """bf16 bit patterns -> nested python floats (independent of oracle helpers)."""
    a = np.asarray(bits).astype(np.uint32) << np.uint32(16)
    return a.view(np.float32).astype(np.float64).tolist()


# --------------------------------------------------------------------------
# 1. Brute force per-token evaluation (plain Python, fp64) vs oracle exact mode
# --------------------------------------------------------------------------

def _brute_layer(x, wr, wg, wu, wd, k, norm, sg=None, su=None, sd=None):
    T, H = len(x), len(x[0])
    E, F = len(wg), len(wg[0])
    ys = []
    for t in range(T):
        logit = [sum(x[t][h] * wr[e][h] for h in range(H)) for e in range(E)]
        order = sorted(range(E), key=lambda e: (-logit[e], e))[:k]
        mx = max(logit)
        den = sum(math.exp(l - mx) for l in logit)
        p = [math.exp(logit[e] - mx) / den for e in order]
        if norm:
            ssum = sum(p)
            p = [v / ssum for v in p]
        y = [0.0] * H
        if sg is not None:
            Fs = len(sg)
            hs = []
            for f in range(Fs):
                g = sum(x[t][h] * sg[f][h] for h in range(H))
                u = sum(x[t][h] * su[f][h] for h in range(H))
                hs.append(g / (1 + math.exp(-g)) * u)
            for h in range(H):
                y[h] += sum(hs[f] * sd[h][f] for f in range(Fs))
        for wj, e in zip(p, order):
            hh = []
            for f in range(F):
                g = sum(x[t][h] * wg[e][f][h] for h in range(H))
                u = sum(x[t][h] * wu[e][f][h] for h in range(H))
                hh.append(g / (1 + math.exp(-g)) * u)
            for h in range(H):
                y[h] += wj * sum(hh[f] * wd[e][h][f] for f in range(F))
        ys.append(y)
    return np.array(ys)


@pytest.mark.parametrize("norm,S", [(0, 1), (1, 0)])
def test_oracle_exact_vs_brute_force(norm, S):
    inp = Inputs(E=4, k=2, H=16, F=8, S=S, Fs=8, T=12, seed=7)
    res = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=2,
                           norm_topk=norm, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up,
                           ws_down_bits=inp.ws_down, mode="exact")
    sh = (_f(inp.ws_gate), _f(inp.ws_up), _f(inp.ws_down)) if S else (None, None, None)
    ref = _brute_layer(_f(inp.x), _f(inp.w_router), _f(inp.w_gate), _f(inp.w_up), _f(inp.w_down),
                       2, norm, *sh)
    assert np.max(np.abs(res["y"] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


# --------------------------------------------------------------------------
# 2. Special case E=1,k=1,S=0,D=1,norm=1: the layer IS a dense SwiGLU MLP
# --------------------------------------------------------------------------

def test_dense_mlp_special_case_vs_torch():
    inp = Inputs(E=1, k=1, H=64, F=96, T=40, seed=11)
    ex = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=1,
                          norm_topk=1, mode="exact")
    ct = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=1,
                          norm_topk=1, mode="contract")
    t = lambda b: torch.from_numpy(np.asarray(b).astype(np.int16)).view(torch.bfloat16).double()
    x, wg, wu, wd = t(inp.x), t(inp.w_gate[0]), t(inp.w_up[0]), t(inp.w_down[0])
    ref = (torch.nn.functional.silu(x @ wg.T) * (x @ wu.T)) @ wd.T
    ref = ref.numpy()
    assert np.allclose(ex["y"], ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    # contract mode: bf16 roundings at h, o, y only -> within the bf16 band
    err = np.abs(ct["y"].astype(np.float64) - ref)
    assert err.max() <= 1e-2 * np.abs(ref).max()
    assert err.sum() / np.abs(ref).sum() <= 6e-3
    # and torch's own bf16 pipeline (RNE casts at h, o) agrees with contract o
    h = (torch.nn.functional.silu((x @ wg.T).float()) * (x @ wu.T).float()).bfloat16()
    o = (h.double() @ wd.T).float().bfloat16().float().numpy()
    assert np.array_equal(o, ct["y"])  # w == 1 and s == 0: y == bf16(fmaf(1, o, 0)) == o


# --------------------------------------------------------------------------
# 3. rounding helpers vs library routines / exact rationals
# --------------------------------------------------------------------------

def test_round_bf16_matches_torch():
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 10,
                        np.array([1.00390625, 1.01171875, -1.00390625, 3.0e-30, 65504.0], np.float32)])
    ref = torch.from_numpy(v).bfloat16().float().numpy()
    assert np.array_equal(oracle.round_bf16(v), ref)


def test_fmaf_correctly_rounded():
    rng = np.random.default_rng(1)
    n = 4000
    a = rng.standard_normal(n).astype(np.float32)
    b = oracle.round_bf16(rng.standard_normal(n).astype(np.float32))
    c = (rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))).astype(np.float32)
    # crafted double-rounding cases: a*b + c lands a hair off an fp32 midpoint
    a[:4] = np.float32(1.0)
    b[:4] = np.float32(2.0 ** -24)       # half an fp32 ulp of 1.0 ...
    c[:4] = np.float32(1.0)
    a[4:8] = np.float32(1.0 + 2.0 ** -23)
    b[4:8] = np.float32(2.0 ** -24)      # ... plus a tail below fp64 precision
    c[4:8] = np.float32(1.0)
    got = oracle.fmaf(a, b, c)
    for i in range(n):
        ex = Fraction(float(a[i])) * Fraction(float(b[i])) + Fraction(float(c[i]))
        lo = np.float32(float(ex))
        # correctly rounded fp32: nearest, ties to even -- check via exact rationals
        cands = [lo, np.nextafter(lo, np.float32(np.inf)), np.nextafter(lo, np.float32(-np.inf))]
        best = min(cands, key=lambda q: (abs(Fraction(float(q)) - ex),
                                         int(np.array([q], np.float32).view(np.uint32)[0]) & 1))
        assert got[i] == best, (i, a[i], b[i], c[i], got[i], best)


# --------------------------------------------------------------------------
# 4. Routing: exact-logit grid, ties, k = E, activated-experts formula
# --------------------------------------------------------------------------

@pytest.mark.parametrize("E,H", [(160, 512), (64, 2048), (8, 4096), (8, 64)])
def test_grid_logits_exact(E, H):
    inp = Inputs(E=E, k=2, H=H, F=64, T=32, seed=3, grid=True)
    l32 = oracle.router_logits(inp.x, inp.w_router)
    l64 = oracle.router_logits(inp.x, inp.w_router, mode="exact")
    # every fp64 sum is representable in fp32 (multiples of 2^-9, |sum| < 2^13)
    assert np.array_equal(l32.astype(np.float64), l64)
    # and independent of summation order (reverse order, python floats)
    xf, wf = _f(inp.x), _f(inp.w_router)
    for t in range(0, 32, 7):
        for e in range(0, E, max(1, E // 5)):
            s = 0.0
            for h in reversed(range(H)):
                s += xf[t][h] * wf[e][h]
            assert s == l64[t, e]


def test_routing_vs_stable_argsort_and_ties():
    inp = Inputs(E=16, k=4, H=128, F=64, T=300, seed=5, grid=True)
    inp.duplicate_router_rows(3, 9)           # tie fixture: e3 and e9 always tie
    logits = oracle.router_logits(inp.x, inp.w_router)
    idx, w = oracle.topk_gating(logits, 4, norm_topk=0)
    for t in range(300):
        order = sorted(range(16), key=lambda e: (-float(logits[t, e]), e))
        assert list(idx[t]) == order[:4]
        if 9 in idx[t]:
            assert 3 in idx[t] and list(idx[t]).index(3) < list(idx[t]).index(9)
    # grid inputs produce real k-th/(k+1)-th ties beyond the fixture
    srt = -np.sort(-logits, axis=1)
    assert np.any(srt[:, 3] == srt[:, 4])


def test_softmax_weights_brute_force():
    inp = Inputs(E=8, k=2, H=64, F=64, T=50, seed=9)
    logits = oracle.router_logits(inp.x, inp.w_router)
    for norm in (0, 1):
        idx, w = oracle.topk_gating(logits, 2, norm_topk=norm, routed_scale=1.0)
        for t in range(50):
            l = [float(v) for v in logits[t]]
            z = sum(math.exp(v) for v in l)
            p = [math.exp(l[e]) / z for e in idx[t]]
            if norm:
                p = [v / sum(p) for v in p]
            assert np.allclose(w[t], p, rtol=1e-6, atol=0)


def test_k_equals_E_routes_every_token_everywhere():
    inp = Inputs(E=4, k=4, H=32, F=32, T=20, seed=2)
    res = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=4,
                           norm_topk=1, D=2, N=2)
    assert np.array_equal(res["layout"]["hist"], np.full((2, 4), 10))
    assert np.allclose(res["w"].sum(axis=1), 1.0, atol=1e-6)


def test_activated_experts_formula():
    # P:133 (A2): E(1-(1-k/E)^m) experts touched by m tokens; closed-form example
    assert abs(oracle.activated_experts(16, 2, 8) - 10.502) < 1e-3
    assert abs(oracle.activated_experts(160, 6, 10 ** 6) - 160) < 1e-9
    # statistical pin of the routing on the performance distribution
    E, k, m = 64, 6, 8
    inp = Inputs(E=E, k=k, H=256, F=64, T=4000, seed=13)
    idx, _ = oracle.topk_gating(oracle.router_logits(inp.x, inp.w_router), k, 0)
    distinct = [len(np.unique(idx[i:i + m])) for i in range(0, 4000, m)]
    assert abs(np.mean(distinct) - oracle.activated_experts(E, k, m)) < 0.06 * oracle.activated_experts(E, k, m)


# --------------------------------------------------------------------------
# 5. The paper's worked example, fig:eps_overview
# --------------------------------------------------------------------------

def test_fig_eps_overview_fixture():
    fx = json.load(open(os.path.join(GOLDEN, "fig_eps_overview.json")))
    E, k, D, N = fx["E"], fx["k"], fx["D"], fx["N"]
    idx = np.array(fx["routing"], np.int32)
    w = np.array(fx["weights"], np.float32)
    # printed: Expert0 takes [0,1,5,9], Expert1 takes [0,2,5,6]
    for e, toks in fx["paper_printed"]["expert_tokens"].items():
        assert sorted(np.nonzero((idx == int(e)).any(axis=1))[0].tolist()) == toks
    inp = Inputs(E=E, k=k, H=16, F=16, T=10, seed=1)
    res = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k,
                           norm_topk=0, D=D, N=N, topk_override=(idx, w))
    lay = res["layout"]
    send = res["send_counts"]
    for tr in fx["paper_printed"]["chunk0_transfers"]:
        assert send[0, tr["src"], tr["dst"]] == len(tr["tokens"])
        # the rows src sends dst in chunk 0 are exactly those tokens, in order
        src, e = tr["src"], tr["expert"]
        p = lay["pos"][src]
        start = lay["token_start"][src]
        loc = idx[start:start + p.shape[0]]
        tok, slot = np.nonzero(loc == e)
        order = np.argsort(p[tok, slot])
        assert (tok[order] + start).tolist() == tr["tokens"]
    # chunk 0 on rank 0 computes expert 0 over tokens [0,1,5,9] (recv order src, t)
    assert lay["recv_start"][0, 0].tolist() == [0, 2]
    assert lay["hist"].tolist() == [[2, 2, 2, 2, 1, 1], [2, 2, 1, 1, 2, 2]]
    assert res["group_begin"].tolist() == [0, 1, 2, 3]
    # pos is the (e, t) stable order on rank 0 (R6)
    assert lay["pos"][0].tolist() == [[0, 2], [1, 6], [3, 4], [7, 8], [5, 9]]


# --------------------------------------------------------------------------
# 6. Conservation, chunked == unchunked, EP=D == EP=1 (bit-exact, contract)
# --------------------------------------------------------------------------

def _tiny(seed=21, T=60):
    return Inputs(E=8, k=2, H=32, F=64, S=1, Fs=32, T=T, seed=seed)


def test_conservation_and_counts():
    inp = _tiny()
    for D in (1, 2, 4):
        for N in range(1, 8 // D + 1):
            res = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=2,
                                   norm_topk=1, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up,
                                   ws_down_bits=inp.ws_down, D=D, N=N)
            lay, send = res["layout"], res["send_counts"]
            T_loc = np.diff(lay["token_start"])
            assert np.array_equal(lay["hist"].sum(axis=1), T_loc * 2)
            for r in range(D):            # every (t, j) goes out and returns exactly once
                assert sorted(lay["pos"][r].ravel().tolist()) == list(range(T_loc[r] * 2))
            assert send.sum() == 60 * 2
            for d in range(D):
                assert send[:, :, d].sum() == lay["recv_total"][d]
                E_loc = 8 // D
                assert lay["recv_total"][d] == lay["hist"][:, d * E_loc:(d + 1) * E_loc].sum()


def test_chunked_equals_unchunked_and_ep_invariance():
    inp = _tiny(T=64)
    args = (inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down)
    kw = dict(k=2, norm_topk=0, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
    base = oracle.moe_layer(*args, D=1, N=1, **kw)["y"]
    for D, N, S in [(1, 3, 1), (1, 8, 1), (2, 2, 1), (2, 1, 3), (4, 2, 2), (8, 1, 2)]:
        y = oracle.moe_layer(*args, D=D, N=N, token_slices=S, **kw)["y"]
        assert np.array_equal(y, base), (D, N, S)


def test_contract_vs_exact_band():
    inp = Inputs(E=8, k=2, H=256, F=192, S=1, Fs=128, T=64, seed=4)
    args = (inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down)
    kw = dict(k=2, norm_topk=1, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
    ex = oracle.moe_layer(*args, mode="exact", **kw)
    ct = oracle.moe_layer(*args, mode="contract", **kw)
    assert np.array_equal(ex["idx"], ct["idx"])
    rel = np.abs(ct["y"] - ex["y"]).sum() / np.abs(ex["y"]).sum()
    assert 3e-4 < rel < 6e-3          # three bf16 rounding points (R4)
    # y values are bf16-representable
    assert np.array_equal(oracle.round_bf16(ct["y"]), ct["y"])


def test_moe_tokens_matches_moe_layer_subset():
    inp = _tiny(T=40)
    full = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=2, norm_topk=1,
                            ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
    sub = [3, 17, 39]
    r = oracle.moe_tokens(inp.x[sub], inp.w_router,
                          lambda e: (inp.w_gate[e], inp.w_up[e], inp.w_down[e]), 2, 1,
                          shared=(inp.ws_gate, inp.ws_up, inp.ws_down))
    assert np.array_equal(r["y"], full["y"][sub])


# --------------------------------------------------------------------------
# 7. FP8 dispatch payload (NEXT-2, R15)
# --------------------------------------------------------------------------

def _e4m3_values():
    """All finite OCP e4m3 (fn) values from the format definition: sign, 4-bit
    exponent (bias 7), 3-bit mantissa, subnormals at exponent 0; S.1111.111 is NaN."""
    vals = []
    for code in range(256):
        s, e, m = code >> 7, (code >> 3) & 15, code & 7
        if e == 15 and m == 7:
            continue
        v = (m / 8.0) * 2.0 ** -6 if e == 0 else (1 + m / 8.0) * 2.0 ** (e - 7)
        vals.append((-v if s else v, m))
    return vals


def test_fp8_block_exponent_closed_form():
    assert oracle.fp8_block_exponent(448.0) == 0
    assert oracle.fp8_block_exponent(449.0) == 1
    assert oracle.fp8_block_exponent(1.0) == -8
    rng = np.random.default_rng(4)
    for a in np.exp(rng.uniform(-20, 20, 2000)):
        s = oracle.fp8_block_exponent(float(a))
        assert a / 2.0 ** s <= 448.0 < a / 2.0 ** (s - 1)


def test_fp8_roundtrip_vs_format_definition():
    """Brute force: every element of the round trip is the nearest e4m3 value
    (ties to even mantissa) of x 2^-s, times 2^s."""
    vals = _e4m3_values()
    grid = np.array([v for v, _ in vals])
    mant = np.array([m for _, m in vals])
    inp = Inputs(E=1, k=1, H=256, F=128, T=12, seed=8)
    x = oracle.bf16_bits_to_f64(inp.x)
    x[3, :128] *= 1e-3          # a block with a very different scale
    x[5, 128:] = 0.0            # an all-zero block
    xb = oracle.bf16_value_to_bits(x.astype(np.float32))
    got = oracle.bf16_bits_to_f64(oracle.fp8_dispatch_roundtrip(xb))
    x = oracle.bf16_bits_to_f64(xb)
    for r in range(12):
        for b0 in (0, 128):
            blk = x[r, b0:b0 + 128]
            s = oracle.fp8_block_exponent(float(np.abs(blk).max()))
            for c, v in enumerate(blk * 2.0 ** (-s)):
                d = np.abs(grid - v)
                cand = np.nonzero(d == d.min())[0]
                best = cand[0] if len(cand) == 1 else cand[np.argmin(mant[cand] & 1)]
                assert got[r, b0 + c] == grid[best] * 2.0 ** s, (r, b0 + c)
    # idempotent, bf16-exact, relative error <= 2^-4 on normal e4m3 values
    again = oracle.fp8_dispatch_roundtrip(oracle.bf16_value_to_bits(got.astype(np.float32)))
    assert np.array_equal(oracle.bf16_bits_to_f64(again), got)


def test_fp8_dispatch_layer_band():
    inp = Inputs(E=8, k=2, H=256, F=128, S=1, Fs=128, T=48, seed=5)
    args = (inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down)
    kw = dict(k=2, norm_topk=1, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)
    y = oracle.moe_layer(*args, **kw)["y"]
    y8 = oracle.moe_layer(*args, dispatch_fp8=True, **kw)
    rel = np.abs(y8["y"] - y).sum() / np.abs(y).sum()
    assert 1e-3 < rel < 5e-2              # e4m3 carries 3 mantissa bits
    assert np.array_equal(y8["idx"], oracle.moe_layer(*args, **kw)["idx"])   # routing sees x, not x'
    # chunked / EP invariance holds in FP8 mode too
    assert np.array_equal(oracle.moe_layer(*args, dispatch_fp8=True, D=2, N=2, **kw)["y"], y8["y"])


# --------------------------------------------------------------------------
# 8. Pipeline-number rule: closed form vs grid argmax
# --------------------------------------------------------------------------

def test_pn_closed_form_example():
    n, v = oracle.pn_optimum_grid(t_comm=10.0, t_comp=12.0, k=0.1, b=0.5, e_loc=20)
    assert n == 10
    assert abs(oracle.pn_gain(10, 10.0, 12.0, 0.1, 0.5) - 7.5) < 1e-12
    assert abs(oracle.pn_gain(10, 10.0, 12.0, 0.1, 0.5) - (10 - 0.5 - 2 * math.sqrt(0.1 * 10))) < 1e-12
    assert oracle.pn_optimum_closed_form(10.0, 12.0, 0.1) == pytest.approx(10.0)


def test_pn_grid_within_one_of_closed_form():
    rng = np.random.default_rng(3)
    for _ in range(200):
        tc, tp = rng.uniform(0.1, 10, 2)
        k, b = rng.uniform(0.001, 0.5), rng.uniform(0, 1)
        e_loc = int(rng.integers(1, 64))
        n, _ = oracle.pn_optimum_grid(tc, tp, k, b, e_loc)
        nstar = min(max(oracle.pn_optimum_closed_form(tc, tp, k), 1), e_loc)
        assert abs(n - nstar) <= 1.0 + 1e-9
    # k = 0: more pipelines always better -> N = E
    assert oracle.pn_optimum_grid(3.0, 5.0, 0.0, 0.2, 20)[0] == 20
    # small C (few tokens) -> no gain from pipelining -> N = 1
    assert oracle.pn_optimum_grid(0.01, 0.01, 0.05, 0.0, 20)[0] == 1


# --------------------------------------------------------------------------
# 8. Expert-side LocalReduce with per-(token, destination, chunk) dedup
#    (NEXT-3, R16)
# --------------------------------------------------------------------------

def test_local_reduce_fixture_counts_by_hand():
    """fig:eps_overview routing (F-8a completion).  N = 1: rank 0
    sends rank 0 tokens {0,1,2,4} (t0: e0,e1 and t2: e1,e2 merge) and rank 1
    tokens {1,3,4} (t3: e3,e4 merge); rank 1 sends rank 0 {5,6,8,9} and rank 1
    {6,7,8,9}: 15 rows instead of 20 pairs.  N = 3 (chunk = local expert):
    every (token, rank, chunk) holds one pair, so no row is saved."""
    fx = json.load(open(os.path.join(GOLDEN, "fig_eps_overview.json")))
    idx = np.array(fx["routing"])
    lay1 = oracle.lr_layout(idx, 6, 2, 1)
    assert lay1["u_hist"].tolist() == [[4, 3], [4, 4]]
    # rank 0's send rows, (g asc, t asc): g0 = {0,1,2,4}, g1 = {1,3,4}
    assert lay1["posg"][0].tolist() == [[0, -1], [1, 4], [2, -1], [5, -1], [3, 6]]
    assert lay1["recv_u_start"][1].tolist() == [[0, 3]]
    lay3 = oracle.lr_layout(idx, 6, 2, 3)
    ref = oracle.dispatch_layout(idx, 6, 2)
    assert lay3["u_hist"].sum() == 20
    # g = c*D + d with c = local expert id: u_hist[r][c*2+d] = pairs of r to expert d*3+c
    for r in range(2):
        for c in range(3):
            for d in range(2):
                assert lay3["u_hist"][r, c * 2 + d] == ref["hist"][r, d * 3 + c]


def test_local_reduce_exact_mode_equals_plain_sum():
    """In exact arithmetic regrouping the sum changes nothing: R16's y equals
    the plain layer's y to fp64 rounding for any (D, N).  A dropped, doubled
    or mis-weighted pair in the grouping fails this."""
    inp = _tiny(T=48)
    args = (inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down)
    kw = dict(k=2, norm_topk=0, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down,
              mode="exact")
    base = oracle.moe_layer(*args, **kw)["y"]
    for D, N in [(1, 1), (1, 4), (2, 1), (2, 3), (4, 2), (8, 1)]:
        y = oracle.moe_layer(*args, D=D, N=N, local_reduce=True, **kw)["y"]
        assert np.allclose(y, base, rtol=1e-12, atol=1e-12 * np.abs(base).max()), (D, N)


def test_local_reduce_single_group_without_shared_is_plain_contract():
    """D = 1, N = 1, no shared experts: every token is one group, so
    y = bf16(0 + bf16(fmaf chain)) = bf16(fmaf chain) = the plain contract."""
    inp = Inputs(E=8, k=3, H=32, F=64, T=50, seed=8)
    args = (inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down)
    a = oracle.moe_layer(*args, k=3, norm_topk=1)["y"]
    b = oracle.moe_layer(*args, k=3, norm_topk=1, local_reduce=True)["y"]
    assert np.array_equal(a, b)
    c = oracle.moe_layer(*args, k=3, norm_topk=1, D=2, N=2, local_reduce=True)["y"]
    assert not np.array_equal(a, c)     # several groups: one more bf16 rounding per partial


def test_local_reduce_layout_invariants():
    inp = _tiny(T=70)
    idx = oracle.topk_gating(oracle.router_logits(inp.x, inp.w_router), 2, 1)[0]
    for D, N in [(1, 3), (2, 1), (2, 4), (4, 2)]:
        lay = oracle.lr_layout(idx, 8, D, N)
        for r in range(D):
            pg, gid = lay["posg"][r], lay["gid"][r]
            ng = np.array([len(set(row)) for row in gid.tolist()])
            assert np.array_equal((pg >= 0).sum(axis=1), ng)
            # every send row is used by exactly one (token, group)
            assert sorted(pg[pg >= 0].tolist()) == list(range(int(lay["u_hist"][r].sum())))
            # rows of group g lie in [u_start[g], u_start[g+1])
            for t in range(pg.shape[0]):
                for i, g in enumerate(sorted(set(gid[t].tolist()))):
                    assert lay["u_start"][r][g] <= pg[t, i] < lay["u_start"][r][g + 1]
        # receive side is the transpose of the send side
        for d in range(D):
            tot = sum(int(lay["u_hist"][src, c * D + d]) for c in range(N) for src in range(D))
            last = lay["recv_u_start"][d][N - 1][D - 1] + lay["u_hist"][D - 1, (N - 1) * D + d]
            assert last == tot


def test_local_reduce_distinct_devices_closed_form():
    """With N = 1 a token sends one row per distinct destination rank.  For k
    distinct experts drawn uniformly from E (E_loc per rank), the expected
    number of distinct ranks is D (1 - C(E-E_loc, k) / C(E, k))
    (hypergeometric: a rank is missed iff all k experts avoid its E_loc).
    DSv2 at EP = 8: E = 160, k = 6 -> 4.4586 rows per token instead of 6."""
    E, k, D, T = 160, 6, 8, 20000
    rng = np.random.default_rng(3)
    idx = np.argsort(rng.random((T, E)), axis=1)[:, :k]
    lay = oracle.lr_layout(idx, E, D, 1)
    mean = lay["u_hist"].sum() / T
    expect = D * (1 - math.comb(E - E // D, k) / math.comb(E, k))
    assert abs(expect - 4.4586) < 1e-4
    assert abs(mean - expect) < 0.02     # sd of a token's count < 1, so 3 sd/sqrt(T) < 0.02


def test_local_reduce_contract_vs_exact_band():
    inp = Inputs(E=8, k=4, H=256, F=192, S=1, Fs=128, T=64, seed=4)
    args = (inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down)
    kw = dict(k=4, norm_topk=1, ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down,
              D=2, N=2, local_reduce=True)
    ex = oracle.moe_layer(*args, mode="exact", **kw)
    ct = oracle.moe_layer(*args, mode="contract", **kw)
    rel = np.abs(ct["y"] - ex["y"]).sum() / np.abs(ex["y"]).sum()
    assert 3e-4 < rel < 6e-3
    assert np.array_equal(oracle.round_bf16(ct["y"]), ct["y"])


# --------------------------------------------------------------------------
# 9. Device-limited routing (NEXT-4, R17)
# --------------------------------------------------------------------------

def test_device_limited_routing_hand_fixture():
    fx = json.load(open(os.path.join(GOLDEN, "device_limited_routing.json")))
    lg = np.array([c["logits"] for c in fx["cases"]], dtype=np.float32)
    idx, _ = oracle.topk_gating(lg, fx["k"], 0, route_groups=fx["route_groups"],
                                route_topk_groups=fx["route_topk_groups"])
    assert idx.tolist() == [c["idx"] for c in fx["cases"]]
    plain, _ = oracle.topk_gating(lg, fx["k"], 0)
    assert plain.tolist() == [c["plain_idx"] for c in fx["cases"]]


def test_device_limited_routing_special_cases_and_bound():
    """M = number of groups: plain routing.  Any M: a token's experts span at
    most M groups (g <= min(k, D)), so with groups = EP ranks, N = 1 and
    the dedup of R16 a token sends at most M rows (M = 1: exactly one)."""
    inp = Inputs(E=16, k=4, H=64, F=128, T=300, seed=33)
    lg = oracle.router_logits(inp.x, inp.w_router)
    plain = oracle.topk_gating(lg, 4, 1)
    same = oracle.topk_gating(lg, 4, 1, route_groups=4, route_topk_groups=4)
    assert np.array_equal(plain[0], same[0]) and np.array_equal(plain[1], same[1])
    for M in (1, 2, 3):
        idx, w = oracle.topk_gating(lg, 4, 1, route_groups=4, route_topk_groups=M)
        assert max(len(set((row // 4).tolist())) for row in idx) <= M
        assert np.allclose(w.sum(axis=1), 1.0, atol=1e-6)          # norm_topk over the kept experts
        lay = oracle.lr_layout(idx, 16, 4, 1)
        assert lay["u_hist"].sum() <= M * 300
        if M == 1:
            assert lay["u_hist"].sum() == 300
    # the restriction can only lower the selected logits
    idx2, _ = oracle.topk_gating(lg, 4, 1, route_groups=4, route_topk_groups=2)
    assert (np.take_along_axis(lg, idx2, 1).sum(1) <= np.take_along_axis(lg, plain[0], 1).sum(1)).all()


def test_comm_volume_bounds_p265():
    """with tokens routed to g devices, the DP+EP all2all volume lies
    in [2P(D-1)/D, g 2P(D-1)/D] (P = the batch's activation bytes; dispatch +
    combine).  With the dedup of R16 (one row per destination) and device-
    limited routing (R17) with groups = ranks, M = g: a token reaches at most g
    ranks (almost always exactly g once k >= g), so the volume sits at the upper
    bound; g = 1 is the lower bound."""
    D, E, k, T = 8, 64, 6, 20000
    rng = np.random.default_rng(11)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    P = T * 1.0                                      # in units of one activation row
    for g in (1, 2, 3):
        idx, _ = oracle.topk_gating(logits, k, 1, route_groups=D, route_topk_groups=g)
        lay = oracle.lr_layout(idx, E, D, 1)
        start = lay["token_start"]
        remote = 0
        for r in range(D):                           # rows each rank sends to other ranks
            remote += int(lay["u_hist"][r].sum() - lay["u_hist"][r][r])
        V = 2 * remote                               # dispatch + combine
        lo, hi = 2 * P * (D - 1) / D, g * 2 * P * (D - 1) / D
        assert lo - 1e-9 <= V * (1 + 0.02) and V <= hi * 1.02
        assert abs(V - hi) / hi < 0.02               # a token's g devices: (D-1)/D of them remote on average
        # per token: at most g destination ranks, almost always exactly g
        ng = np.array([len(set((row // (E // D)).tolist())) for row in idx])
        assert ng.max() <= g and (ng == g).mean() > 0.99


# --------------------------------------------------------------------------
# 10. Chunk / slice / shard rules (R8, R12) vs tables written out by hand
# --------------------------------------------------------------------------

def _rules():
    return json.load(open(os.path.join(GOLDEN, "chunk_rules.json")))


def test_chunk_groups_vs_survey_table():
    """SURVEY §8(c) table (S:307 rule): the first E_loc mod N groups get one
    more expert.  Remainder experts going to the LAST groups, or a rounded
    split, fail here."""
    for e_loc, per_n in _rules()["chunk_group_sizes"].items():
        for n, sizes in per_n.items():
            gb = oracle.chunk_groups(int(e_loc), int(n))
            assert np.diff(gb).tolist() == sizes, (e_loc, n)
            assert gb[0] == 0 and gb[-1] == int(e_loc)
    with pytest.raises(ValueError):
        oracle.chunk_groups(3, 4)        # N > E_loc is not an expert grouping


def test_slice_ranges_and_token_shards_vs_hand_tables():
    for c in _rules()["slice_ranges"]:
        assert oracle.slice_ranges(c["T_loc"], c["S"]).tolist() == c["begin"], c
    for c in _rules()["token_shards"]:
        assert oracle.token_shards(c["T"], c["D"]).tolist() == c["start"], c


def test_token_sliced_send_counts_vs_hand_fixture():
    """fig:eps_overview routing with token slices (R8 extension), counted by hand."""
    fx = json.load(open(os.path.join(GOLDEN, "fig_eps_overview.json")))
    idx = np.array(fx["routing"], np.int32)
    hist = oracle.dispatch_layout(idx, 6, 2)["hist"]
    for c in _rules()["sliced_send_counts"]:
        got = oracle.chunk_send_counts(hist, 6, 2, c["N"], token_slices=c["S"], idx=idx)
        assert got.tolist() == c["send"], c
        # summed over slices, the sliced counts are the unsliced chunk counts
        plain = oracle.chunk_send_counts(hist, 6, 2, c["N"])
        assert np.array_equal(got.reshape(c["N"], c["S"], 2, 2).sum(axis=1), plain)


def _round_frac(q, p):
    """Exact round-to-nearest-even of a Fraction to p significant bits (binary,
    exponent >= -126, no overflow): fp32 for p = 24, bf16 for p = 8."""
    if q == 0:
        return Fraction(0)
    sgn = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1                                   # now 2^e <= a < 2^(e+1)
    e = max(e, -126)
    ulp = Fraction(2) ** (e - p + 1)
    m = a / ulp
    r = m.numerator // m.denominator
    rem = m - r
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and r % 2 == 1):
        r += 1
    return sgn * r * ulp


def _fma_sensitive_pair():
    """(w fp32, o bf16) with q = fp32(w o) = 2^-1 + 2^-8 + 2^-24 exactly and
    w o - q > 0: from acc = 1, 1 + q is an fp32 tie (1.5 + 2^-8 + 2^-24) whose
    even side 1.5 + 2^-8 is itself a bf16 tie, so fmaf(w, o, 1) -> bf16 rounds
    up while fp32(1 + fp32(w o)) -> bf16 rounds down.  Found by scanning bf16
    mantissas of o with exact rationals."""
    q = Fraction(1, 2) + Fraction(1, 2 ** 8) + Fraction(1, 2 ** 24)
    for om in range(128):
        o = Fraction(128 + om, 128)                     # bf16: 8 significant bits
        wq = q / o                                      # in [0.25, 0.5]
        ulp_w = Fraction(1, 2 ** 25) if wq >= Fraction(1, 4) else Fraction(1, 2 ** 26)
        m = (wq / ulp_w).numerator // (wq / ulp_w).denominator + 1
        w = m * ulp_w
        p = w * o
        if 0 < p - q < Fraction(1, 2 ** 25) and _round_frac(p, 24) == q:
            fused = _round_frac(_round_frac(1 + p, 24), 8)
            split = _round_frac(_round_frac(1 + q, 24), 8)
            if fused != split:
                return np.float32(float(w)), np.float32(float(o))
    raise AssertionError("no sensitive pair found")


def test_contract_combine_vs_exact_rational_fmaf_chain():
    """R4 combine: acc = fp32(s); acc = fmaf(w_j, o_j, acc) for j in slot order;
    y = bf16(acc).  Brute force with exact rationals and an independent
    rounding.  Two crafted tokens make the plausible mistakes visible in y:
    token A (s added last instead of first: 1 + 2^-8 then three 2^-25 terms),
    token B (a separately rounded multiply-add instead of fmaf: an exact product
    just above an fp32 tie that is also a bf16 tie)."""
    rng = np.random.default_rng(17)
    T, k, H = 24, 6, 16
    s = oracle.round_bf16(rng.standard_normal((T, H)).astype(np.float32))
    o = oracle.round_bf16((rng.standard_normal((T, k, H)) * 8).astype(np.float32))
    w = (rng.random((T, k)) / 3).astype(np.float32)
    # token A: s = 1, products 2^-8, 2^-25 x 3 (0.25 fp32 ulp each), then zeros
    s[0] = 1.0
    o[0, :, :] = np.array([2.0 ** -8, 2.0 ** -25, 2.0 ** -25, 2.0 ** -25, 1.0, 1.0], np.float32)[:, None]
    w[0] = np.array([1, 1, 1, 1, 0, 0], np.float32)
    # token B: s = 1, one product just above the 1 + 2^-8 + 2^-24 double tie
    wb, ob = _fma_sensitive_pair()
    s[1] = 1.0
    o[1, :, :] = ob
    w[1] = 0.0
    w[1, 0] = wb
    got = oracle.combine(s, o, w)
    for t in range(T):
        for h in range(H):
            acc = Fraction(float(s[t, h]))
            for j in range(k):
                acc = _round_frac(Fraction(float(w[t, j])) * Fraction(float(o[t, j, h])) + acc, 24)
            assert Fraction(float(got[t, h])) == _round_frac(acc, 8), (t, h)
    # the two crafted tokens separate the contract from the plausible mistakes
    acc = np.zeros((T, H), np.float32)
    for j in range(k):
        acc = oracle.fmaf(np.broadcast_to(w[:, j][:, None], (T, H)), o[:, j, :], acc)
    s_last = oracle.round_bf16((acc + s).astype(np.float32))
    acc = s.copy()
    for j in range(k):
        acc = (acc + (w[:, j][:, None] * o[:, j, :]).astype(np.float32)).astype(np.float32)
    mul_add = oracle.round_bf16(acc)
    assert not np.array_equal(s_last[0], got[0]) and not np.array_equal(mul_add[1], got[1])


def test_pn_grid_with_token_slices_vs_hand_candidates():
    """R8 extension: the candidates are N = 1..E_loc and E_loc*S for
    S = 2..slice_max (nothing in between).  Objective L - R of P:408-415 with
    C = min(4, 5) = 4, k = 0.1, b = 0 (N* = sqrt(40) = 6.32 by P:425):
      E_loc = 1, slice_max = 8: {1..8}            -> 6 (3.3333-0.6 > 3.4286-0.7)
      E_loc = 3, slice_max = 3: {1,2,3,6,9}       -> 6 (2.7333 > 2.6556 > 2.3667)
      E_loc = 4, slice_max = 2: {1,2,3,4,8}       -> 8 (2.7 > 2.6; 5 is no candidate)
      E_loc = 3, slice_max = 1: {1,2,3}           -> 3"""
    f = lambda n: 4.0 / n * (n - 1) - 0.1 * n
    for e_loc, smax, cands, want in [(1, 8, [1, 2, 3, 4, 5, 6, 7, 8], 6), (3, 3, [1, 2, 3, 6, 9], 6),
                                     (4, 2, [1, 2, 3, 4, 8], 8), (3, 1, [1, 2, 3], 3)]:
        best = max(cands, key=lambda n: (f(n), -n))
        assert best == want
        n, v = oracle.pn_optimum_grid(4.0, 5.0, 0.1, 0.0, e_loc, slice_max=smax)
        assert n == want and abs(v - f(want)) < 1e-12, (e_loc, smax, n)


def test_nan_logits_rank_below_every_number():
    """R18: a NaN logit (NaN / Inf inputs) is never selected ahead of a number
    and adds 0 to the softmax; a row of NaNs selects experts 0..k-1 with NaN
    weights.  Brute force over the finite logits."""
    rng = np.random.default_rng(2)
    lg = rng.standard_normal((6, 12)).astype(np.float32)
    lg[0, [1, 5]] = np.nan
    lg[1, :] = np.nan
    lg[2, 0] = np.nan
    idx, w = oracle.topk_gating(lg, 3, norm_topk=0)
    for t in (0, 2, 3):
        fin = [e for e in range(12) if not math.isnan(float(lg[t, e]))]
        order = sorted(fin, key=lambda e: (-float(lg[t, e]), e))[:3]
        assert idx[t].tolist() == order
        z = sum(math.exp(float(lg[t, e])) for e in fin)
        assert np.allclose(w[t], [math.exp(float(lg[t, e])) / z for e in order], rtol=1e-6)
    assert idx[1].tolist() == [0, 1, 2] and np.isnan(w[1]).all()
