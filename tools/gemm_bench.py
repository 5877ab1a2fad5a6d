#!/usr/bin/env python
"""Dev microbenchmark: the layer's grouped GEMMs alone on DeepSeek-V2 / Mixtral
expert shapes (EP = 1), timed with CUDA events.  Not part of the product or
the driver contract; used to tune tile shape / rasterisation.

  python tools/gemm_bench.py [--config dsv2] [--tile-m 256] [--reps 10]
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
    ap.add_argument("--tile-m", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ctas", type=int, default=148)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    E, k, H, F, T = c["E"], c["k"], c["H"], c["F"], c["T"]
    rows = T * k
    rng = np.random.default_rng(0)
    counts = rng.multinomial(rows, np.ones(E) / E).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)

    def gen(shape, tid, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        device_fill_bf16(t.data_ptr(), t.numel(), 1, tid, 0, MODE_UNIF, float(scale))
        return t
    A = gen((rows, H), 1, 1.0)
    Wg, Wu = gen((E * F, H), 3, unif_scale(H)), gen((E * F, H), 4, unif_scale(H))
    Wd = gen((E * H, F), 5, unif_scale(F))
    h = torch.empty(rows, F, dtype=torch.bfloat16, device="cuda")
    o = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    rs, rc = torch.from_numpy(starts).cuda(), torch.from_numpy(counts).cuda()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(2):
        gemm_grouped(0, A, Wg, Wu, F, h, rs, rc, F, tile_m=a.tile_m, num_ctas=a.ctas)
        gemm_grouped(1, h, Wd, None, H, o, rs, rc, H, tile_m=a.tile_m, num_ctas=a.ctas)
    torch.cuda.synchronize()
    t1 = t2 = 0.0
    for _ in range(a.reps):
        ev[0].record()
        gemm_grouped(0, A, Wg, Wu, F, h, rs, rc, F, tile_m=a.tile_m, num_ctas=a.ctas)
        ev[1].record()
        gemm_grouped(1, h, Wd, None, H, o, rs, rc, H, tile_m=a.tile_m, num_ctas=a.ctas)
        ev[2].record()
        torch.cuda.synchronize()
        t1 += ev[0].elapsed_time(ev[1])
        t2 += ev[1].elapsed_time(ev[2])
    t1 /= a.reps
    t2 /= a.reps
    f1, f2 = 4.0 * H * F * rows, 2.0 * H * F * rows
    print(f"{a.config} tile_m={a.tile_m} raster={os.environ.get('EPSMOE_RASTER_GM', '1')} ctas={a.ctas}: "
          f"gateup {t1:.3f} ms {f1 / t1 / 1e9:.0f} TF/s | down {t2:.3f} ms {f2 / t2 / 1e9:.0f} TF/s")


if __name__ == "__main__":
    main()
