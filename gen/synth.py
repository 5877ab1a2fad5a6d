"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the MoE method (SURVEY.md §8(d) "Synthetic
inputs"): it only turns (seed, tensor_id, global element index) into bf16 bit
patterns with a counter hash, so that

  * the oracle (``oracle/``) and the GPU path see identical inputs without
    either producing them for the other, and
  * tokens are indexed GLOBALLY and experts by GLOBAL expert id, so a rank's
    shard of x or of the expert weights does not depend on the EP degree D.

The device twin is ``gen/gen.cu`` (``libepsgen.so``); ``tests/test_gen.py``
checks the two are bit-identical.

Element value, for ``h = mix64(key(seed, tid) + (i + 1) * GOLDEN)``:

  * mode "unif" (scale s, an fp32):  f = float32(h >> 40) * 2^-23 - 1   (exact,
    in [-1, 1)), v = fp32(f * s) (one IEEE round-to-nearest multiply),
    result = bf16_rne(v).   U(-sqrt3, sqrt3)/sqrt(fan_in) is s = sqrt(3/fan_in).
  * mode "grid" (denominator d):     n = ((h >> 32) mod 17) - 8, result = n / d,
    exact in bf16 for d in {8, 64} (the exact-logit grid).
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
TID_MUL = np.uint64(0xD1B54A32D192ED03)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# tensor ids (SURVEY.md §8(d) "Seeds")
BASE_SEED = 20241016
TID_X, TID_WR, TID_WGATE, TID_WUP, TID_WDOWN = 1, 2, 3, 4, 5
TID_WS_GATE, TID_WS_UP, TID_WS_DOWN, TID_BIAS = 6, 7, 8, 9

MODE_UNIF, MODE_GRID = 0, 1


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * M1
    z = z ^ (z >> np.uint64(27))
    z = z * M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tid: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(tid + 1) * TID_MUL)],
                     dtype=np.uint64)
        return _mix64(z)[0]


def hash_u64(seed: int, tid: int, index: np.ndarray) -> np.ndarray:
    """h(seed, tid, i) for an array of global element indices i (uint64)."""
    key = stream_key(seed, tid)
    with np.errstate(over="ignore"):
        z = key + (index.astype(np.uint64) + np.uint64(1)) * GOLDEN
        return _mix64(z)


def f32_to_bf16_bits(v: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (no NaNs are generated)."""
    b = v.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def unif_scale(fan_in: int, amp2: float = 3.0) -> np.float32:
    """fp32 scale s with U(-sqrt(amp2), sqrt(amp2))/sqrt(fan_in) (fan_in=1: plain)."""
    return np.float32(math.sqrt(amp2 / fan_in))


def fill_bf16(n: int, seed: int, tid: int, index_base: int = 0, mode: int = MODE_UNIF,
              param: float = 1.0, chunk: int = 1 << 24) -> np.ndarray:
    """n bf16 bit patterns (uint16) for global indices index_base .. index_base+n-1."""
    out = np.empty(n, dtype=np.uint16)
    p32 = np.float32(param)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = np.arange(index_base + s, index_base + e, dtype=np.uint64)
        h = hash_u64(seed, tid, idx)
        if mode == MODE_UNIF:
            f = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)
            v = (f * p32).astype(np.float32)
            out[s:e] = f32_to_bf16_bits(v)
        elif mode == MODE_GRID:
            nn = ((h >> np.uint64(32)) % np.uint64(17)).astype(np.int64) - 8
            v = (nn.astype(np.float32) / p32).astype(np.float32)
            out[s:e] = f32_to_bf16_bits(v)
        else:
            raise ValueError(f"unknown mode {mode}")
    return out


def router_skew_bias(num_experts: int, s: float, seed: int = BASE_SEED,
                     identity: bool = False) -> np.ndarray:
    """Synthetic skew hook: beta_e = -s * ln(1 + pi(e)) in fp32.

    pi is a seeded permutation of the experts (hot experts scattered over ranks)
    or the identity (hot experts all on rank 0).  Computed once on the host and
    handed, as the same fp32 array, to both the oracle and the GPU.
    """
    if identity:
        perm = np.arange(num_experts)
    else:
        keys = hash_u64(seed, TID_BIAS, np.arange(num_experts, dtype=np.uint64))
        perm = np.argsort(keys, kind="stable")
        inv = np.empty_like(perm)
        inv[perm] = np.arange(num_experts)
        perm = inv
    return (-s * np.log1p(perm.astype(np.float64))).astype(np.float32)


# ----------------------------------------------------------------------------
# Workload configs (BASELINE.json "configs"); shapes only, no method arithmetic.
# ----------------------------------------------------------------------------
CONFIGS = {
    # name: (E, k, H, F, S, F_s, T_global, norm_topk)
    "tiny": dict(E=8, k=2, H=64, F=128, S=0, Fs=0, T=256, norm_topk=1),
    "mixtral": dict(E=8, k=2, H=4096, F=14336, S=0, Fs=0, T=16384, norm_topk=1),
    "dsv2_lite": dict(E=64, k=6, H=2048, F=1408, S=2, Fs=1408, T=32768, norm_topk=0),
    "dsv2": dict(E=160, k=6, H=5120, F=1536, S=2, Fs=1536, T=65536, norm_topk=0),
    # decode-regime batch (A22, NEXT-4; Table I's bs=256): weight-streaming, HBM-bound
    "dsv2_decode": dict(E=160, k=6, H=5120, F=1536, S=2, Fs=1536, T=256, norm_topk=0),
    "mixtral_decode": dict(E=8, k=2, H=4096, F=14336, S=0, Fs=0, T=256, norm_topk=1),
}


class Inputs:
    """Host (numpy, bf16 bit patterns) inputs of one MoE layer.

    Expert weights are generated only for the global expert ids in ``experts``
    (default all).  ``grid=True`` draws x and W_r from the exact-logit grid.
    """

    def __init__(self, E, k, H, F, S=0, Fs=0, T=256, seed=BASE_SEED, grid=False,
                 experts=None, skew=0.0, skew_identity=False, tokens=None, **_):
        self.E, self.k, self.H, self.F, self.S, self.Fs, self.T = E, k, H, F, S, Fs, T
        self.seed, self.grid = seed, grid
        tok = np.arange(T) if tokens is None else np.asarray(tokens)
        self.tokens = tok
        if grid:
            self.x = np.stack([fill_bf16(H, seed, TID_X, int(t) * H, MODE_GRID, 8.0) for t in tok]) \
                if tokens is not None else fill_bf16(T * H, seed, TID_X, 0, MODE_GRID, 8.0).reshape(T, H)
            self.w_router = fill_bf16(E * H, seed, TID_WR, 0, MODE_GRID, 64.0).reshape(E, H)
        else:
            sx = unif_scale(1)
            self.x = np.stack([fill_bf16(H, seed, TID_X, int(t) * H, MODE_UNIF, sx) for t in tok]) \
                if tokens is not None else fill_bf16(T * H, seed, TID_X, 0, MODE_UNIF, sx).reshape(T, H)
            self.w_router = fill_bf16(E * H, seed, TID_WR, 0, MODE_UNIF, unif_scale(H)).reshape(E, H)
        self.experts = np.arange(E) if experts is None else np.asarray(experts, dtype=np.int64)
        sH, sF = unif_scale(H), unif_scale(F)
        if len(self.experts) == 0:
            self.w_gate = self.w_up = self.w_down = None
        else:
            self._gen_experts(seed, sH, sF)
        self._gen_shared(seed, sH)
        self.router_bias = router_skew_bias(E, skew, seed, skew_identity) if skew else None

    def _gen_experts(self, seed, sH, sF):
        E, H, F = self.E, self.H, self.F
        self.w_gate = np.stack([fill_bf16(F * H, seed, TID_WGATE, int(e) * F * H, MODE_UNIF, sH)
                                for e in self.experts]).reshape(len(self.experts), F, H)
        self.w_up = np.stack([fill_bf16(F * H, seed, TID_WUP, int(e) * F * H, MODE_UNIF, sH)
                              for e in self.experts]).reshape(len(self.experts), F, H)
        self.w_down = np.stack([fill_bf16(H * F, seed, TID_WDOWN, int(e) * H * F, MODE_UNIF, sF)
                                for e in self.experts]).reshape(len(self.experts), H, F)

    def _gen_shared(self, seed, sH):
        H, SF = self.H, self.S * self.Fs
        if SF:
            sS = unif_scale(SF)
            self.ws_gate = fill_bf16(SF * H, seed, TID_WS_GATE, 0, MODE_UNIF, sH).reshape(SF, H)
            self.ws_up = fill_bf16(SF * H, seed, TID_WS_UP, 0, MODE_UNIF, sH).reshape(SF, H)
            self.ws_down = fill_bf16(H * SF, seed, TID_WS_DOWN, 0, MODE_UNIF, sS).reshape(H, SF)
        else:
            self.ws_gate = self.ws_up = self.ws_down = None

    def duplicate_router_rows(self, e_src: int, e_dst: int) -> None:
        """Tie fixture: W_r[e_dst] := W_r[e_src], so the pair always ties."""
        self.w_router[e_dst] = self.w_router[e_src]
