"""Seeded synthetic input generators (host numpy + device CUDA twin).

Shared by the oracle and the GPU path; holds none of the method's arithmetic.
"""
from .synth import (BASE_SEED, CONFIGS, Inputs, MODE_GRID, MODE_UNIF, TID_BIAS, TID_WDOWN, TID_WGATE,  # noqa: F401
                    TID_WR, TID_WS_DOWN, TID_WS_GATE, TID_WS_UP, TID_WUP, TID_X, bf16_bits_to_f32,
                    f32_to_bf16_bits, fill_bf16, hash_u64, router_skew_bias, unif_scale)
from .device import device_fill_bf16, load_device_gen  # noqa: F401
