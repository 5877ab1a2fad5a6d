"""CPU oracle for the EPS-MoE layer hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.  The product path
(paper_2410_12247_b200/) never imports it and fails loudly without its CUDA
library; the two share no code (only gen/, the seeded input generator).

Every function cites the passage of the paper (PAPER.md line numbers, P:n) it
follows; DESIGN.md §3 lists the readings taken where the paper is silent.
Pinned by tests/test_oracle_pins.py (no function is "parity unpinned").
"""
from .moe import (bf16_bits_to_f64, bf16_value_to_bits, chunk_groups, chunk_send_counts,  # noqa: F401
                  combine, dispatch_layout, expert_ffn, fmaf, fp8_block_exponent, fp8_dispatch_roundtrip,
                  local_reduce_combine, lr_group_ids, lr_layout, moe_layer, moe_tokens, round_bf16, slice_ranges,
                  router_logits, silu_f32, token_shards, topk_gating)
from .planner import activated_experts, pn_gain, pn_optimum_closed_form, pn_optimum_grid  # noqa: F401
