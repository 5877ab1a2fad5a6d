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
