"""CPU-only checks of the C ABI: the library loads, exports every symbol the
header declares, validates configs, and its host-only planner / layout logic
matches the oracle and the paper's closed forms (no GPU calls)."""
import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from gen import Inputs
from paper_2410_12247_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "epsmoe.h")).read()
    declared = set(re.findall(r"^(?:moe_status_t|size_t|int32_t|const char\*)\s+(moe_[a-z_]+)\s*\(", header,
                              re.MULTILINE))
    assert len(declared) >= 15
    lib = C.CDLL(abi.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and the binding mirrors them all
    assert declared <= set(abi._SIGS), declared - set(abi._SIGS)


def test_struct_sizes_match_header_layout(tmp_path):
    """The ctypes mirrors have the C header's sizes and field offsets (compiled
    with gcc against include/epsmoe.h)."""
    structs = {"moe_config_t": abi.moe_config_t, "moe_weights_t": abi.moe_weights_t,
               "moe_plan_t": abi.moe_plan_t, "moe_cost_model_t": abi.moe_cost_model_t,
               "moe_debug_t": abi.moe_debug_t}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "epsmoe.h"', 'int main(void) {']
    for name, cls in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'  printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    lines += ['  return 0;', '}']
    src = tmp_path / "sizes.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(out[name]) == C.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(out[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


@pytest.mark.parametrize("bad", [
    dict(E=6, D=4),            # E % D != 0 (R12)
    dict(k=9),                 # top_k > 8
    dict(H=100),               # hidden not a multiple of 64
    dict(F=200),               # ffn not a multiple of 128
    dict(E=300, D=1),          # > 256 experts
])
def test_invalid_configs_rejected(bad):
    E, D = bad.get("E", 8), bad.get("D", 1)
    cfg = abi.make_config(E, bad.get("k", 2), bad.get("H", 64), bad.get("F", 128), ep=D, max_tokens=16)
    assert abi.lib().moe_layer_workspace_bytes(C.byref(cfg)) == 0
    with pytest.raises(abi.EpsMoeError):
        abi.plan_compute(cfg, 16)


def test_workspace_bytes_cover_the_layout():
    cfg = abi.make_config(160, 6, 5120, 1536, 2, 1536, ep=1, max_tokens=65536)
    n = abi.lib().moe_layer_workspace_bytes(C.byref(cfg))
    T, k, H, F = 65536, 6, 5120, 1536
    assert n >= 2 * T * k * H * 2 + T * k * F * 2   # send + o + h at least
    assert n < 40e9


def _cost(k_ms=0.1, b_ms=0.5):
    c = abi.moe_cost_model_t()
    c.n_points = 2
    c.m_points[0], c.m_points[1] = 100.0, 10000.0
    c.a2a_fixed_ms, c.a2a_gbps, c.k_ms, c.b_ms = 0.0, 100.0, k_ms, b_ms
    return c


def test_planner_matches_oracle_pn_rule():
    """moe_plan_compute's N == the oracle's exhaustive argmax for the
    T_comm / T_comp the cost model implies."""
    rng = np.random.default_rng(0)
    for trial in range(40):
        E, D = [(160, 8), (64, 8), (16, 2), (8, 1), (64, 4)][trial % 5]
        k = 6 if E >= 16 else 2
        cfg = abi.make_config(E, k, 2048, 1408, ep=D, max_tokens=1 << 16)
        c = _cost(k_ms=float(rng.uniform(0.001, 0.2)), b_ms=float(rng.uniform(0, 0.5)))
        gm = float(rng.uniform(0.001, 0.05))
        for kind in (0, 1):
            c.gemm_ms[kind][0], c.gemm_ms[kind][1] = gm, gm * 100 * (1 + 0.1 * kind)
        T = int(rng.integers(1000, 100000))
        hist = rng.multinomial(T * k // D, np.ones(E) / E, size=D).astype(np.int32)
        plan = abi.plan_compute(cfg, T, hist, c)
        E_loc = E // D
        # token slices (R8 extension): <= 8, <= 64 chunks, >= 256 tokens per slice
        s_max = max(1, min(8, 64 // E_loc, (T // D) // 256)) if D > 1 else 1
        n_ref, _ = oracle.pn_optimum_grid(plan.pred_comm_ms, plan.pred_comp_ms, c.k_ms, c.b_ms, E_loc, s_max)
        assert plan.num_chunks == n_ref
        S = plan.token_slices
        assert S == (n_ref // E_loc if n_ref > E_loc else 1)
        g = plan.group_begin[:plan.num_chunks // S + 1]
        assert list(g) == oracle.chunk_groups(E_loc, plan.num_chunks // S).tolist()
        if D == 1:
            assert plan.num_chunks == 1 and plan.pred_comm_ms == 0.0   # no all2all -> nothing to hide


def test_planner_closed_form_example():
    """P:421-425 example: C=10, k=0.1, b=0.5, E=20 -> N=10, G=7.5."""
    cfg = abi.make_config(160, 6, 2048, 1408, ep=8, max_tokens=1 << 16)
    c = _cost(k_ms=0.1, b_ms=0.5)
    # T_comp huge, T_comm = 10 ms: a2a of the uniform histogram at chosen GB/s
    for kind in (0, 1):
        c.gemm_ms[kind][0], c.gemm_ms[kind][1] = 100.0, 10000.0
    T = 65536
    hist = np.full((8, 160), T * 6 // 8 // 160, np.int32)
    rows = hist.sum() / 8 * 7 / 8                 # cross-rank rows per rank
    bytes_one = rows * 2048 * 2
    c.a2a_gbps = float(bytes_one / 5e-3 / 1e9)    # 5 ms per direction -> T_comm = 10 ms
    plan = abi.plan_compute(cfg, T, hist, c)
    assert abs(plan.pred_comm_ms - 10.0) < 1e-3
    assert plan.num_chunks == 10
    assert abs(plan.pred_gain_ms - 7.5) < 1e-3
    assert abs(plan.pred_gain_ms - (10 - 0.5 - 2 * math.sqrt(0.1 * 10))) < 1e-3


def test_kind_choice_follows_cost_model():
    """A8 / P:357: per-expert GroupGemm vs DenseGemm by modelled load."""
    cfg = abi.make_config(16, 2, 1024, 1024, ep=1, max_tokens=1 << 16)
    c = _cost()
    c.gemm_ms[0][0], c.gemm_ms[0][1] = 0.01, 1.0     # grouped: better at small m
    c.gemm_ms[1][0], c.gemm_ms[1][1] = 0.02, 0.8     # dense: better at large m
    hist = np.zeros((1, 16), np.int32)
    hist[0, :8] = 50
    hist[0, 8:] = 9000
    plan = abi.plan_compute(cfg, 40000, hist, c)
    assert list(plan.expert_kind[:8]) == [abi.MOE_GEMM_GROUPED] * 8
    assert list(plan.expert_kind[8:16]) == [abi.MOE_GEMM_DENSE] * 8


def test_exchange_layout_matches_oracle_single_process():
    inp = Inputs(E=8, k=2, H=64, F=128, T=50, seed=3)
    for D in (1, 2, 4):
        res = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=2, norm_topk=1, D=D,
                               N=min(2, 8 // D))
        lay = res["layout"]
        gh = lay["hist"].astype(np.int32)
        for r in range(D):
            cfg = abi.make_config(8, 2, 64, 128, ep=D, rank=r, max_tokens=64)
            plan = abi.make_plan(min(2, 8 // D))
            send_off, recv_off, cs, cr = abi.exchange_layout(cfg, plan, gh)
            assert send_off.tolist() == lay["send_start"][r].tolist()
            assert recv_off[:-1].reshape(8 // D, D).tolist() == lay["recv_start"][r].tolist()
            assert recv_off[-1] == lay["recv_total"][r]
            assert np.array_equal(cs, res["send_counts"][:, r, :])
            assert np.array_equal(cr, res["send_counts"][:, :, r])


def test_planner_token_slices_when_one_expert_per_rank():
    """Mixtral at EP = 8 has E_loc = 1: without token slices no chunking is
    possible; with a communication-heavy cost model the planner splits tokens."""
    cfg = abi.make_config(8, 2, 4096, 14336, ep=8, max_tokens=1 << 16)
    c = _cost(k_ms=0.02, b_ms=0.0)
    for kind in (0, 1):
        c.gemm_ms[kind][0], c.gemm_ms[kind][1] = 1.0, 100.0
    c.a2a_gbps = 50.0
    hist = np.full((8, 8), 16384 * 2 // 8 // 8, np.int32)
    plan = abi.plan_compute(cfg, 16384, hist, c)
    assert plan.token_slices > 1 and plan.num_chunks == plan.token_slices
    assert plan.group_begin[0] == 0 and plan.group_begin[1] == 1
    # local_reduce keeps expert-only chunks (R16)
    cfg_lr = abi.make_config(8, 2, 4096, 14336, ep=8, max_tokens=1 << 16, local_reduce=1)
    assert abi.plan_compute(cfg_lr, 16384, hist, c).num_chunks == 1


# ---------------------------------------------------------------- planner: wire bytes and SM partition

def _flat_cost(gbps=700.0):
    """GEMMs cheap enough that the comm side decides nothing about N; per-chunk
    cost so high that N = 1 (T_comm is then the unsplit all2all)."""
    c = _cost(k_ms=1e3, b_ms=0.0)
    c.a2a_fixed_ms, c.a2a_gbps = 0.0, gbps
    for kind in (0, 1):
        c.gemm_ms[kind][0], c.gemm_ms[kind][1] = 0.01, 1.0
    return c


def test_planner_prices_fp8_and_dedup_wire_bytes():
    """T_comm counts the bytes that cross: FP8 dispatch rows of
    H + H/128 bytes padded to 16 (R15) against bf16 combine rows, and under
    expert-side LocalReduce (R16) one row per distinct destination rank instead
    of one per pair, i.e. D (1 - C(E - E_loc, k) / C(E, k)) / k of the rows
    (DSv2 at EP 8: 4.4586 / 6 = 0.7431)."""
    E, D, k, H, F = 160, 8, 6, 5120, 1536
    T = 65536
    mk = lambda **kw: abi.make_config(E, k, H, F, ep=D, max_tokens=T // D, **kw)  # noqa: E731
    c = _flat_cost()
    base = abi.plan_compute(mk(), T, None, c)
    fp8 = abi.plan_compute(mk(dispatch_fp8=1), T, None, c)
    lr = abi.plan_compute(mk(local_reduce=1), T, None, c)
    both = abi.plan_compute(mk(dispatch_fp8=1, local_reduce=1), T, None, c)
    assert base.num_chunks == fp8.num_chunks == lr.num_chunks == 1
    q_row = ((H + H // 128) + 15) & ~15
    f_fp8 = (q_row + 2 * H) / (4 * H)
    f_lr = D * (1 - math.comb(E - E // D, k) / math.comb(E, k)) / k
    assert abs(f_lr - 4.4586 / 6) < 1e-4
    assert fp8.pred_comm_ms / base.pred_comm_ms == pytest.approx(f_fp8, rel=1e-5)
    assert lr.pred_comm_ms / base.pred_comm_ms == pytest.approx(f_lr, rel=1e-5)
    assert both.pred_comm_ms / base.pred_comm_ms == pytest.approx(f_fp8 * f_lr, rel=1e-5)
    # the uniform T_comm itself: 2 directions x cross-rank pairs x row bytes / GB/s
    pairs = T * k * (D - 1) / D / D
    assert base.pred_comm_ms == pytest.approx(2 * pairs * 2 * H / 700e9 * 1e3, rel=1e-5)


def test_planner_lr_rows_grow_with_chunks():
    """R16 with N chunks: a token sends one row per distinct (rank, chunk) group,
    so the rows per pair rise with N toward 1.  The expectation (G - N)(1 - q) /
    (k (D - 1) / D), G = N D, q = C(E - E/G, k) / C(E, k), is pinned by brute
    force over random top-k sets; the planner's T_comm(N) under local_reduce
    follows it (checked at N = E_loc, which a compute-dominated model picks)."""
    E, D, k = 64, 4, 6
    rng = np.random.default_rng(5)
    sets = np.argsort(rng.random((40000, E)), axis=1)[:, :k]
    home = rng.integers(0, D, size=len(sets))           # the token's own rank
    prev = 0.0
    for N in (1, 2, 4, 8, 16):
        gsz = E // (N * D)
        grp = sets // gsz                                   # group id = rank * N + chunk
        rank = sets // (E // D)
        remote_groups = np.array([len(set(g[r != h].tolist())) for g, r, h in zip(grp, rank, home)])
        remote_pairs = (rank != home[:, None]).sum(axis=1)
        f_mc = remote_groups.sum() / remote_pairs.sum()
        assert f_mc == pytest.approx(_lr_factor(E, D, k, N), rel=0.02), (N, f_mc)
        assert _lr_factor(E, D, k, N) > prev
        prev = _lr_factor(E, D, k, N)
    # planner: GEMMs dominate, no per-chunk cost -> N = E_loc; T_comm(E_loc) / T_comm(plain) = f(E_loc)
    E, D, k, T = 32, 4, 6, 1 << 16
    c = _flat_cost()
    c.k_ms = 0.0
    for kind in (0, 1):
        c.gemm_ms[kind][0], c.gemm_ms[kind][1] = 10.0, 1000.0
    plain = abi.plan_compute(abi.make_config(E, k, 2048, 1408, ep=D, max_tokens=T // D), T, None, c)
    lr = abi.plan_compute(abi.make_config(E, k, 2048, 1408, ep=D, max_tokens=T // D, local_reduce=1), T, None, c)
    assert lr.num_chunks == E // D
    assert lr.pred_comm_ms / plain.pred_comm_ms == pytest.approx(_lr_factor(E, D, k, E // D), rel=1e-5)


def _lr_factor(E, D, k, N):
    G = N * D
    q = math.prod((E - E / G - i) / (E - i) for i in range(k))
    return (G - N) * (1 - q) / (k * (D - 1) / D)


def test_planner_picks_the_sm_partition_from_the_cost_model():
    """NEXT-1 (Table IV): the plan's (sm_gemm,
    comm_ctas) is the comm budget whose modelled pipelined layer time
    T_comp * scale + T_comm(GB/s at that budget) - G(N) is least.  SMs precious
    (steep GEMM scaling, flat all2all rate) -> the smallest budget; all2all
    dominant with a rate that grows with CTAs -> the largest; the copy-engine
    plane reserves none; ep = 1 has no partition."""
    E, D, k, H, F, T = 160, 8, 6, 5120, 1536, 65536
    cfg = abi.make_config(E, k, H, F, ep=D, max_tokens=T // D)

    def model(scales, rates, gemm):
        c = _cost(k_ms=0.05, b_ms=0.0)
        c.a2a_fixed_ms = 0.01
        for kind in (0, 1):
            c.gemm_ms[kind][0], c.gemm_ms[kind][1] = gemm * 0.01, gemm
        c.num_sms, c.n_comm = 148, 4
        for i, (cc, s, r) in enumerate(zip((4, 8, 12, 16), scales, rates)):
            c.comm_ctas[i], c.gemm_scale_at[i], c.a2a_gbps_at[i] = cc, s, r
        c.a2a_gbps = max(rates)
        return c
    precious = abi.plan_compute(cfg, T, None, model((1.06, 1.12, 1.19, 1.27), (700, 700, 700, 700), 1.0))
    assert (precious.comm_ctas, precious.sm_gemm) == (4, 140)
    comm = abi.plan_compute(cfg, T, None, model((1.03, 1.06, 1.09, 1.12), (100, 200, 400, 800), 0.05))
    assert (comm.comm_ctas, comm.sm_gemm) == (16, 116)
    # the choice is the argmin of the modelled time over the four budgets, checked by brute force
    for m in (model((1.06, 1.12, 1.19, 1.27), (300, 500, 650, 720), 0.3),
              model((1.02, 1.05, 1.30, 1.31), (200, 600, 610, 615), 0.2)):
        p = abi.plan_compute(cfg, T, None, m)
        best = None
        for i in range(4):
            mi = abi.moe_cost_model_t.from_buffer_copy(bytes(m))
            mi.n_comm = 1
            mi.comm_ctas[0], mi.gemm_scale_at[0], mi.a2a_gbps_at[0] = m.comm_ctas[i], m.gemm_scale_at[i], m.a2a_gbps_at[i]
            pi = abi.plan_compute(cfg, T, None, mi)
            t = pi.pred_comp_ms + pi.pred_comm_ms - pi.pred_gain_ms
            if best is None or t < best[0] - 1e-6:
                best = (t, m.comm_ctas[i])
        assert p.comm_ctas == best[1]
    ce = abi.plan_compute(abi.make_config(E, k, H, F, ep=D, max_tokens=T // D, a2a_p2p=2), T, None,
                          model((1.06, 1.12, 1.19, 1.27), (100, 200, 400, 800), 0.05))
    assert (ce.comm_ctas, ce.sm_gemm) == (0, 148)
    one = abi.plan_compute(abi.make_config(E, k, H, F, ep=1, max_tokens=T), T, None,
                           model((1.06, 1.12, 1.19, 1.27), (100, 200, 400, 800), 0.05))
    assert (one.comm_ctas, one.sm_gemm, one.num_chunks) == (0, 0, 1)


def test_hostcoll_create_rejects_the_nccl_plane():
    """moe_layer_create_hostcoll carries counts only: a2a_p2p = 0 (rows over
    NCCL) is refused before any device work."""
    cfg = abi.make_config(16, 2, 64, 128, ep=2, rank=0, max_tokens=16, a2a_p2p=0)
    fake = C.c_void_p(0x1000)
    w = abi.moe_weights_t(fake, fake, fake, fake, None, None, None, None)
    cb = abi.HOST_ALLGATHER_FN(lambda ctx, s, r, n: 0)
    h = C.c_void_p()
    st = abi.lib().moe_layer_create_hostcoll(C.byref(cfg), C.byref(w), cb, None, None, 0, C.byref(h))
    assert st == 1 and "a2a_p2p" in abi.lib().moe_last_error().decode()
