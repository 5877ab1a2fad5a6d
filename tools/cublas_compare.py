#!/usr/bin/env python
"""Dev comparison: the layer's tcgen05 GEMMs vs the library GEMMs of this image on
identical problems (same inputs, same box, alternating, CUDA events):

  * dense (one group, the shared experts' shapes): ours vs cuBLAS (torch.mm), GateUp
    also vs cuBLAS + torch's SiLU*mul (what our fused epilogue replaces);
  * grouped (the routed experts, multinomial rows per expert): ours vs one
    cuBLAS GEMM per expert (the paper's DenseGemm) and vs
    torch._grouped_mm (CUTLASS grouped GEMM), when it runs on this GPU.

Not part of the product; prints one JSON line per case.

  python tools/cublas_compare.py [--config dsv2] [--reps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.nn.functional as Fn  # noqa: E402

from gen import CONFIGS, MODE_UNIF, device_fill_bf16, unif_scale  # noqa: E402
from paper_2410_12247_b200 import gemm_grouped  # noqa: E402


def timed(fns, reps):
    """Alternate the candidates rep by rep; mean ms of each."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    tot = [0.0] * len(fns)
    for f in fns:
        f()
    torch.cuda.synchronize()
    for _ in range(reps):
        for i, f in enumerate(fns):
            ev[0].record()
            f()
            ev[1].record()
            torch.cuda.synchronize()
            tot[i] += ev[0].elapsed_time(ev[1])
    return [t / reps for t in tot]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="dsv2")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    E, k, H, F, T, SF = c["E"], c["k"], c["H"], c["F"], c["T"], c["S"] * c["Fs"]

    def gen(shape, tid, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
        device_fill_bf16(t.data_ptr(), t.numel(), 1, tid, 0, MODE_UNIF, float(scale))
        return t

    out = []
    # ---- dense: the shared experts' GEMMs (one group of T rows)
    if SF:
        x = gen((T, H), 1, 1.0)
        wg, wu = gen((SF, H), 6, unif_scale(H)), gen((SF, H), 7, unif_scale(H))
        wgu = torch.cat([wg, wu])
        wd = gen((H, SF), 8, unif_scale(SF))
        h = torch.empty(T, SF, dtype=torch.bfloat16, device="cuda")
        o = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
        rs = torch.zeros(1, dtype=torch.int32, device="cuda")
        rc = torch.full((1,), T, dtype=torch.int32, device="cuda")
        hc = torch.empty(T, 2 * SF, dtype=torch.bfloat16, device="cuda")

        def ours_gu():
            gemm_grouped(0, x, wg, wu, SF, h, rs, rc, SF, tile_m=256)

        def cub_gu():
            torch.mm(x, wgu.t(), out=hc)

        def cub_gu_swiglu():
            torch.mm(x, wgu.t(), out=hc)
            torch.mul(Fn.silu(hc[:, :SF]), hc[:, SF:])

        def ours_dn():
            gemm_grouped(1, h, wd, None, H, o, rs, rc, H, tile_m=256)

        def cub_dn():
            torch.mm(h, wd.t(), out=o)
        t = timed([ours_gu, cub_gu, cub_gu_swiglu], a.reps)
        fl = 4.0 * T * H * SF
        out.append(dict(case=f"{a.config} dense GateUp {T}x{H} -> 2x{SF}", ours_ms=t[0], cublas_ms=t[1],
                        cublas_plus_swiglu_ms=t[2], ours_tflops=fl / t[0] / 1e9, cublas_tflops=fl / t[1] / 1e9))
        t = timed([ours_dn, cub_dn], a.reps)
        fl = 2.0 * T * H * SF
        out.append(dict(case=f"{a.config} dense Down {T}x{SF} -> {H}", ours_ms=t[0], cublas_ms=t[1],
                        ours_tflops=fl / t[0] / 1e9, cublas_tflops=fl / t[1] / 1e9))
        del x, wg, wu, wgu, wd, h, o, hc
        torch.cuda.empty_cache()
    # ---- grouped: the routed experts (multinomial rows per expert, EP = 1)
    rows = T * k
    rng = np.random.default_rng(0)
    counts = rng.multinomial(rows, np.ones(E) / E).astype(np.int32)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int32)
    A = gen((rows, H), 1, 1.0)
    Wg, Wu = gen((E * F, H), 3, unif_scale(H)), gen((E * F, H), 4, unif_scale(H))
    Wd = gen((E * H, F), 5, unif_scale(F))
    Wgu = torch.cat([Wg.view(E, F, H), Wu.view(E, F, H)], dim=1)          # [E, 2F, H]
    h = torch.empty(rows, F, dtype=torch.bfloat16, device="cuda")
    o = torch.empty(rows, H, dtype=torch.bfloat16, device="cuda")
    hc = torch.empty(rows, 2 * F, dtype=torch.bfloat16, device="cuda")
    rs, rc = torch.from_numpy(starts).cuda(), torch.from_numpy(counts).cuda()
    segs = [(int(s), int(n)) for s, n in zip(starts, counts)]

    def ours_gu():
        gemm_grouped(0, A, Wg, Wu, F, h, rs, rc, F, tile_m=256)

    def dense_gu():
        for e, (s, n) in enumerate(segs):
            if n:
                torch.mm(A[s:s + n], Wgu[e].t(), out=hc[s:s + n])

    def ours_dn():
        gemm_grouped(1, h, Wd, None, H, o, rs, rc, H, tile_m=256)

    def dense_dn():
        Wd3 = Wd.view(E, H, F)
        for e, (s, n) in enumerate(segs):
            if n:
                torch.mm(h[s:s + n], Wd3[e].t(), out=o[s:s + n])
    offs = torch.from_numpy(np.cumsum(counts).astype(np.int32)).cuda()
    grouped = None
    try:
        torch._grouped_mm(A, Wgu.transpose(-2, -1), offs=offs)
        torch.cuda.synchronize()

        def grouped():
            torch._grouped_mm(A, Wgu.transpose(-2, -1), offs=offs)
    except Exception as ex:  # not available for this dtype / arch
        grouped_err = repr(ex)[:200]
    fns = [ours_gu, dense_gu] + ([grouped] if grouped else [])
    t = timed(fns, a.reps)
    fl = 4.0 * rows * H * F
    rec = dict(case=f"{a.config} grouped GateUp {E} experts, {rows} rows, {H} -> 2x{F}", ours_ms=t[0],
               cublas_per_expert_ms=t[1], ours_tflops=fl / t[0] / 1e9, cublas_per_expert_tflops=fl / t[1] / 1e9)
    if grouped:
        rec.update(torch_grouped_mm_ms=t[2], torch_grouped_mm_tflops=fl / t[2] / 1e9)
    else:
        rec.update(torch_grouped_mm=f"unavailable: {grouped_err}")
    out.append(rec)
    Wd3t = Wd.view(E, H, F)
    grouped_dn = None
    try:
        torch._grouped_mm(h, Wd3t.transpose(-2, -1), offs=offs)
        torch.cuda.synchronize()

        def grouped_dn():
            torch._grouped_mm(h, Wd3t.transpose(-2, -1), offs=offs)
    except Exception:
        pass
    fns = [ours_dn, dense_dn] + ([grouped_dn] if grouped_dn else [])
    t = timed(fns, a.reps)
    fl = 2.0 * rows * H * F
    rec = dict(case=f"{a.config} grouped Down {E} experts, {rows} rows, {F} -> {H}", ours_ms=t[0],
               cublas_per_expert_ms=t[1], ours_tflops=fl / t[0] / 1e9, cublas_per_expert_tflops=fl / t[1] / 1e9)
    if grouped_dn:
        rec.update(torch_grouped_mm_ms=t[2], torch_grouped_mm_tflops=fl / t[2] / 1e9)
    out.append(rec)
    for r in out:
        print(json.dumps({kk: (round(v, 4) if isinstance(v, float) else v) for kk, v in r.items()}), flush=True)


if __name__ == "__main__":
    main()
