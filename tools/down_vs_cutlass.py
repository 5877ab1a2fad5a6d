#!/usr/bin/env python
"""Dev: one launch each of our grouped Down GEMM and torch._grouped_mm (CUTLASS) on
the same routed-expert Down problem, after two warm-ups each, for ncu capture
(ncu captures every launch; the last two GEMM launches are the measured pair).  --gateup does the same for GateUp
(torch's output is [rows, 2F] without the SwiGLU).

  python tools/down_vs_cutlass.py [--config dsv2] [--gateup]
"""
import argparse
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
    ap.add_argument("--gateup", action="store_true")
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
    if a.gateup:
        A = gen((rows, H), 1, 1.0)
        Wg, Wu = gen((E * F, H), 3, unif_scale(H)), gen((E * F, H), 4, unif_scale(H))
        Wgu = torch.cat([Wg.view(E, F, H), Wu.view(E, F, H)], dim=1)
        h = torch.empty(rows, F, dtype=torch.bfloat16, device="cuda")
        ours = lambda: gemm_grouped(0, A, Wg, Wu, F, h, rs, rc, F, tile_m=256)  # noqa: E731
        theirs = lambda: torch._grouped_mm(A, Wgu.transpose(-2, -1), offs=offs)  # noqa: E731
    else:
        h = gen((rows, F), 1, 1.0)
        Wd = gen((E * H, F), 5, unif_scale(F))
        o = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
        ours = lambda: gemm_grouped(1, h, Wd, None, H, o, rs, rc, H, tile_m=256)  # noqa: E731
        theirs = lambda: torch._grouped_mm(h, Wd.view(E, H, F).transpose(-2, -1), offs=offs)  # noqa: E731
    for _ in range(2):
        ours()
        theirs()
    torch.cuda.synchronize()
    ours()
    theirs()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
