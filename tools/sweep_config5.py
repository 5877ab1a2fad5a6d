#!/usr/bin/env python
"""BASELINE config 5: the DeepSeek-V2 layer under skewed routing, sweeping the
pipeline chunk count 1..8 and the GroupGemm / DenseGemm choice (P:305-338
Table II analog), plus the measured cost model (GEMM ms per expert vs rows for
both kinds: the B200 re-measurement of the paper's Fig. mfu_of_gemm).

One GPU => EP = 1: there is no all2all to hide, so this isolates the compute
side of chunking (more, smaller grouped launches) and of the kernel choice.

  python tools/sweep_config5.py [--skews 0,0.5,1.0] [--chunks 1,2,4,8] [--steps 5]
Writes one JSON line per point to stdout and a markdown table to --out.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import (CONFIGS, MODE_UNIF, TID_WDOWN, TID_WGATE, TID_WR, TID_WS_DOWN, TID_WS_GATE, TID_WS_UP,  # noqa: E402
                 TID_WUP, TID_X, device_fill_bf16, router_skew_bias, unif_scale)
from paper_2410_12247_b200 import (MOE_GEMM_AUTO, MOE_GEMM_DENSE, MOE_GEMM_GROUPED, MoELayer,  # noqa: E402
                                   make_plan)

KINDS = {"grouped": MOE_GEMM_GROUPED, "dense": MOE_GEMM_DENSE, "auto": MOE_GEMM_AUTO}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dsv2")
    ap.add_argument("--skews", default="0,0.5,1.0")
    ap.add_argument("--chunks", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--kinds", default="grouped,dense,auto")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=3, help="interleaved repetitions (median reported)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_config5_sweep.md"))
    ap.add_argument("--sm-sweep", action="store_true",
                    help="Table IV analog (P:467-490): layer ms vs GEMM SM budget for several token counts")
    a = ap.parse_args()
    if a.sm_sweep:
        return sm_sweep(a)
    c = CONFIGS[a.config]
    E, k, H, F, S, Fs, T = c["E"], c["k"], c["H"], c["F"], c["S"], c["Fs"], c["T"]
    seed = 20241016
    dev = torch.device("cuda", 0)

    def gen(shape, tid, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        device_fill_bf16(t.data_ptr(), t.numel(), seed, tid, 0, MODE_UNIF, float(scale))
        return t
    sH = unif_scale(H)
    base_w = dict(w_router=gen((E, H), TID_WR, sH), w_gate=gen((E, F, H), TID_WGATE, sH),
                  w_up=gen((E, F, H), TID_WUP, sH), w_down=gen((E, H, F), TID_WDOWN, unif_scale(F)))
    if S:
        base_w.update(ws_gate=gen((S * Fs, H), TID_WS_GATE, sH), ws_up=gen((S * Fs, H), TID_WS_UP, sH),
                      ws_down=gen((H, S * Fs), TID_WS_DOWN, unif_scale(S * Fs)))
    x = gen((T, H), TID_X, unif_scale(1))
    rows = []
    calib = None
    for s in [float(v) for v in a.skews.split(",")]:
        w = dict(base_w)
        if s:
            w["router_bias"] = torch.from_numpy(router_skew_bias(E, s, seed)).to(dev)
        L = MoELayer(E, k, H, F, w, S=S, Fs=Fs, max_tokens=T, norm_topk=c["norm_topk"])
        if calib is None:
            m = L.calibrate()
            calib = dict(m_points=list(m.m_points[:m.n_points]), grouped_ms=list(m.gemm_ms[0][:m.n_points]),
                         dense_ms=list(m.gemm_ms[1][:m.n_points]))
        d, b = L.debug_buffers(T)
        L.forward(x, debug=d)
        torch.cuda.synchronize()
        hist = b["hist"].cpu().numpy()
        skew_stats = dict(max_over_mean=float(hist.max() / hist.mean()), zero_experts=int((hist == 0).sum()))
        auto_plan = L.plan(T, hist[None, :])
        points = [(kind, n) for kind in a.kinds.split(",") for n in [int(v) for v in a.chunks.split(",")]
                  if not (kind == "auto" and n != 1)]
        # interleaved rounds in a shuffled order, median per point: a sequential sweep
        # on a power-capped GPU drifts (later points run hotter) and biases the ranking
        times = {p: [] for p in points}
        rng = np.random.default_rng(0)
        for rnd in range(a.rounds):
            for i in rng.permutation(len(points)):
                kind, n = points[i]
                plan = None if kind == "auto" else make_plan(n, KINDS[kind])
                for _ in range(2):
                    L.forward(x, plan=plan)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.steps):
                    L.forward(x, plan=plan)
                e1.record()
                torch.cuda.synchronize()
                times[(kind, n)].append(e0.elapsed_time(e1) / a.steps)
        for kind, n in points:
            plan = None if kind == "auto" else make_plan(n, KINDS[kind])
            L.forward(x, plan=plan)
            ms = float(np.median(times[(kind, n)]))
            r = dict(config=a.config, skew=s, kind=kind, chunks=n, ms=ms, ms_rounds=times[(kind, n)],
                     tokens_per_s=T / ms * 1e3, launches=L.last_launches(), **skew_stats)
            if kind == "auto":
                r["auto_kinds"] = {"grouped": int(sum(1 for e in range(E) if auto_plan.expert_kind[e] == 1)),
                                   "dense": int(sum(1 for e in range(E) if auto_plan.expert_kind[e] == 2))}
            rows.append(r)
            print(json.dumps(r), flush=True)
        L.close()
    with open(a.out, "w") as f:
        f.write(f"# Config-5 sweep ({a.config}, EP=1, B200) — generated by tools/sweep_config5.py\n\n")
        f.write("Measured cost model (ms per expert, GateUp+Down, 8-expert grouped launch vs per-expert launches):\n\n")
        f.write("| rows/expert | grouped ms | dense ms |\n|---|---|---|\n")
        for mp, g, dn in zip(calib["m_points"], calib["grouped_ms"], calib["dense_ms"]):
            f.write(f"| {mp:.0f} | {g:.4f} | {dn:.4f} |\n")
        f.write("\n| skew s | max/mean expert load | zero-load experts | kind | chunks | ms/layer (median of rounds) | tokens/s | launches |\n")
        f.write("|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['skew']} | {r['max_over_mean']:.2f} | {r['zero_experts']} | {r['kind']} | {r['chunks']} | "
                    f"{r['ms']:.3f} | {r['tokens_per_s'] / 1e6:.3f} M | {r['launches']} |\n")


def sm_sweep(a):
    """Layer time vs persistent-GEMM SM budget (plan.sm_gemm) at several
    per-expert loads m: the B200 analog of the paper's Table IV,
    which found 116 of 132 H800 SMs optimal once comm kernels share the GPU."""
    c = CONFIGS[a.config]
    E, k, H, F, S, Fs, T = c["E"], c["k"], c["H"], c["F"], c["S"], c["Fs"], c["T"]
    seed = 20241016
    dev = torch.device("cuda", 0)

    def gen(shape, tid, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        device_fill_bf16(t.data_ptr(), t.numel(), seed, tid, 0, MODE_UNIF, float(scale))
        return t
    sH = unif_scale(H)
    w = dict(w_router=gen((E, H), TID_WR, sH), w_gate=gen((E, F, H), TID_WGATE, sH),
             w_up=gen((E, F, H), TID_WUP, sH), w_down=gen((E, H, F), TID_WDOWN, unif_scale(F)))
    if S:
        w.update(ws_gate=gen((S * Fs, H), TID_WS_GATE, sH), ws_up=gen((S * Fs, H), TID_WS_UP, sH),
                 ws_down=gen((H, S * Fs), TID_WS_DOWN, unif_scale(S * Fs)))
    x = gen((T, H), TID_X, unif_scale(1))
    L = MoELayer(E, k, H, F, w, S=S, Fs=Fs, max_tokens=T, norm_topk=c["norm_topk"])
    sms = [148, 140, 132, 124, 116, 108, 100, 92]
    res = {}
    for div in (1, 2, 4, 8, 16):
        Tn = T // div
        for sm in sms:
            plan = make_plan(1, MOE_GEMM_GROUPED, sm_gemm=sm)
            for _ in range(2):
                L.forward(x[:Tn], plan=plan)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                L.forward(x[:Tn], plan=plan)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            res[(Tn, sm)] = ms
            print(json.dumps(dict(tokens=Tn, rows_per_expert=Tn * k / E, sm_gemm=sm, ms=ms)), flush=True)
    out = os.path.join(ROOT, "profiles", "r01_table4_sm_sweep.md")
    with open(out, "w") as f:
        f.write(f"# Table IV analog on B200 ({a.config}, EP=1): layer ms vs GEMM SM budget — tools/sweep_config5.py --sm-sweep\n\n")
        f.write("| tokens | rows/expert (m) | " + " | ".join(f"{s} SMs" for s in sms) + " |\n")
        f.write("|---|---|" + "---|" * len(sms) + "\n")
        for div in (1, 2, 4, 8, 16):
            Tn = T // div
            best = min(res[(Tn, s)] for s in sms)
            cells = [(f"**{res[(Tn, s)]:.3f}**" if res[(Tn, s)] == best else f"{res[(Tn, s)]:.3f}") for s in sms]
            f.write(f"| {Tn} | {Tn * k / E:.0f} | " + " | ".join(cells) + " |\n")
    L.close()


if __name__ == "__main__":
    main()
