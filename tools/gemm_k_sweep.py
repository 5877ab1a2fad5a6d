#!/usr/bin/env python
"""Dev microbenchmark: Down-shaped grouped GEMM (bf16 epilogue) at several K with the
FLOPs held fixed, to see how per-tile overhead scales (shorter K = more tiles).

  python tools/gemm_k_sweep.py [--tile-m 128|256] [--ks 768,1536,...] [--epi 1]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import MODE_UNIF, device_fill_bf16, unif_scale  # noqa: E402
from paper_2410_12247_b200 import gemm_grouped  # noqa: E402

import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tile-m", type=int, default=128)
ap.add_argument("--ks", default="")
ap.add_argument("--epi", type=int, default=1)
args = ap.parse_args()
N, G = 5120, 160
cases = ([(int(k), args.epi) for k in args.ks.split(",")] if args.ks else
         [(768, 1), (1536, 1), (3072, 1), (6144, 1), (1536, 0), (5120, 0)])
for K, epi in cases:
    rows = int(393216 * 1536 / K)
    rows -= rows % G
    counts = np.full(G, rows // G, np.int32)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    def gen(shape, tid, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        device_fill_bf16(t.data_ptr(), t.numel(), 1, tid, 0, MODE_UNIF, float(scale))
        return t
    A = gen((rows, K), 1, 1.0)
    nb = N if epi == 1 else 1536
    B0 = gen((G * nb, K), 2, unif_scale(K))
    B1 = gen((G * nb, K), 3, unif_scale(K)) if epi == 0 else None
    out = torch.empty(rows, nb, dtype=torch.bfloat16, device="cuda")
    rs, rc = torch.from_numpy(starts).cuda(), torch.from_numpy(counts).cuda()
    for _ in range(2):
        gemm_grouped(epi, A, B0, B1, nb, out, rs, rc, nb, tile_m=args.tile_m)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gemm_grouped(epi, A, B0, B1, nb, out, rs, rc, nb, tile_m=args.tile_m)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    flop = (4.0 if epi == 0 else 2.0) * rows * K * nb
    print(f"epi={epi} K={K} rows={rows} rows/expert={rows // G}: {ms:.3f} ms {flop / ms / 1e9:.0f} TF/s", flush=True)
    del A, B0, B1, out
