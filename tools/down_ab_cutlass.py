#!/usr/bin/env python
"""Dev: timed A/B of our grouped Down GEMM vs torch._grouped_mm (CUTLASS) on the
same routed-expert Down problem: ABBA order, N rounds, each launch bracketed by
CUDA events with a synchronize (mean and min ms per side), plus a back-to-back
burst of 10 launches per side (the layer's regime).

  python tools/down_ab_cutlass.py [--config dsv2] [--rounds 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import CONFIGS, MODE_UNIF, device_fill_bf16, unif_scale  # noqa: E402
from paper_2410_12247_b200 import gemm_grouped  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dsv2")
    ap.add_argument("--rounds", type=int, default=20)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    E, k, H, F, T = c["E"], c["k"], c["H"], c["F"], c["T"]
    rows = T * k
    counts = np.random.default_rng(0).multinomial(rows, np.ones(E) / E).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)

    def gen(shape, tid, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        device_fill_bf16(t.data_ptr(), t.numel(), 1, tid, 0, MODE_UNIF, float(scale))
        return t
    rs, rc = torch.from_numpy(starts).cuda(), torch.from_numpy(counts).cuda()
    offs = torch.from_numpy(np.cumsum(counts).astype(np.int32)).cuda()
    h = gen((rows, F), 1, 1.0)
    Wd = gen((E * H, F), 5, unif_scale(F))
    o = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    Wt = Wd.view(E, H, F).transpose(-2, -1)
    fns = {"ours": lambda: gemm_grouped(1, h, Wd, None, H, o, rs, rc, H, tile_m=256),
           "cutlass": lambda: torch._grouped_mm(h, Wt, offs=offs)}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for f in fns.values():
        f()
        f()
    torch.cuda.synchronize()
    single = {n: [] for n in fns}
    for r in range(a.rounds):
        order = ["ours", "cutlass"] if r % 2 == 0 else ["cutlass", "ours"]
        for n in order:
            ev0.record()
            fns[n]()
            ev1.record()
            torch.cuda.synchronize()
            single[n].append(ev0.elapsed_time(ev1))
    burst = {n: [] for n in fns}
    for r in range(4):
        order = ["ours", "cutlass"] if r % 2 == 0 else ["cutlass", "ours"]
        for n in order:
            ev0.record()
            for _ in range(10):
                fns[n]()
            ev1.record()
            torch.cuda.synchronize()
            burst[n].append(ev0.elapsed_time(ev1) / 10)
    fl = 2.0 * rows * H * F
    out = {"config": a.config}
    for n in fns:
        out[n] = {"single_mean_ms": float(np.mean(single[n])), "single_min_ms": float(np.min(single[n])),
                  "burst_ms": [round(x, 4) for x in burst[n]],
                  "burst_tflops": fl / np.mean(burst[n]) / 1e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
