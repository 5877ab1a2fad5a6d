// Expert pipeline scheduler — pure host code, no CUDA calls.
//
//   pipeline number: argmax_{1<=N<=E} L(theta;N) - R(N),
//       L(theta;N) = min{T_comm/N, T_comp/N} (N-1),  R(N) = kN + b
//   kernel choice:   GroupGemm vs DenseGemm by per-expert load        (A8)
//   chunks:          horizontal split, weights split by expert, each chunk a
//                    balanced contiguous group of local experts       (R8);
//                    beyond N = E_loc, every expert group is split further
//                    into S token slices (N = E_loc * S, R8 extension)
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/epsmoe.h"
#include "internal.h"

namespace epsmoe {

// GEMM time (ms) of one expert with m rows, linear interpolation in the table
// (linear extrapolation beyond the last point, proportional below the first).
double cost_gemm_ms(const moe_cost_model_t& c, int kind, double m) {
  if (m <= 0) return 0.0;
  const int n = c.n_points;
  const float* xs = c.m_points;
  const float* ys = c.gemm_ms[kind];
  if (n <= 0) return 0.0;
  if (m <= xs[0]) return ys[0] * (m / xs[0]);
  for (int i = 1; i < n; ++i)
    if (m <= xs[i]) {
      double f = (m - xs[i - 1]) / (xs[i] - xs[i - 1]);
      return ys[i - 1] + f * (ys[i] - ys[i - 1]);
    }
  if (n == 1) return ys[0] * (m / xs[0]);
  double slope = (ys[n - 1] - ys[n - 2]) / (xs[n - 1] - xs[n - 2]);
  return ys[n - 1] + slope * (m - xs[n - 1]);
}

// Analytic stand-in used until moe_layer_calibrate measures the device:
// tensor-core time at a fraction of the sustained bf16 peak that saturates with
// rows per expert (Conclusion 1), plus a fixed per-launch cost.
void default_cost_model(const moe_config_t& cfg, moe_cost_model_t* c) {
  std::memset(c, 0, sizeof(*c));
  const double peak = 1.4e15;                     // sustained bf16 FLOP/s (B200_PROFILING.md)
  const double flop_per_row = 6.0 * cfg.hidden * (double)cfg.ffn;
  const float pts[MOE_COST_POINTS] = {16, 64, 128, 256, 512, 1024, 2048, 3072, 4096, 6144, 8192, 16384};
  c->n_points = MOE_COST_POINTS;
  for (int i = 0; i < MOE_COST_POINTS; ++i) {
    double m = pts[i];
    double tiles = std::ceil(m / 128.0);
    double eff_g = std::min(1.0, m / (tiles * 128.0)) * 0.85;   // grouped: M-tile padding only
    double eff_d = eff_g * (m / (m + 256.0));                   // dense: one launch per expert
    c->m_points[i] = (float)m;
    c->gemm_ms[0][i] = (float)(flop_per_row * m / (peak * eff_g) * 1e3);
    c->gemm_ms[1][i] = (float)(flop_per_row * m / (peak * eff_d) * 1e3 + 0.004);
  }
  c->a2a_fixed_ms = 0.02f;
  c->a2a_gbps = 700.0f;   // measured peer copy ~770 GB/s per direction (B200_PROFILING.md)
  c->k_ms = 0.015f;       // per-chunk fixed overhead (two NCCL groups + events)
  c->b_ms = 0.0f;
}

static void balanced_groups(int e_loc, int n, int32_t* begin) {
  int base = e_loc / n, rem = e_loc % n, acc = 0;
  begin[0] = 0;
  for (int c = 0; c < n; ++c) {
    acc += base + (c < rem ? 1 : 0);
    begin[c + 1] = acc;
  }
}

// Largest token-slice count the planner considers: chunks stay <= 64, slices
// <= 8 and >= 256 source tokens each (smaller slices re-read the group's
// weights for too few rows).
int plan_slice_max(int e_loc, int64_t t_loc) {
  int s = std::min<int64_t>(8, std::min<int64_t>(MOE_MAX_CHUNKS / e_loc, t_loc / 256));
  return std::max(1, s);
}

int plan_compute(const moe_config_t& cfg, const moe_cost_model_t& cost, int64_t global_tokens,
                 const int32_t* ghist, moe_plan_t* out) {
  const int E = cfg.num_experts, D = cfg.ep, k = cfg.top_k;
  if (D < 1 || E % D || E > MOE_MAX_EXPERTS || k < 1 || k > E) return MOE_ERR_INVALID;
  const int E_loc = E / D;
  std::memset(out, 0, sizeof(*out));
  out->token_slices = 1;

  // rows each expert receives (global), from the histogram or uniform (CalcPN mm)
  std::vector<double> rows(E, 0.0);
  std::vector<double> send_rows(D, 0.0), recv_rows(D, 0.0);
  if (ghist) {
    for (int r = 0; r < D; ++r)
      for (int e = 0; e < E; ++e) {
        double v = ghist[(int64_t)r * E + e];
        rows[e] += v;
        int owner = e / E_loc;
        if (owner != r) { send_rows[r] += v; recv_rows[owner] += v; }
      }
  } else {
    double mm = (double)global_tokens * k / E;   // mm = m * topk / EN
    for (int e = 0; e < E; ++e) rows[e] = mm;
    double cross = (double)global_tokens * k * (D - 1) / D / D;
    for (int r = 0; r < D; ++r) { send_rows[r] = cross; recv_rows[r] = cross; }
  }

  // per-expert kind (A8) and per-rank modelled compute; the plan follows the
  // max-loaded rank so every rank derives the same plan from the same input.
  double t_comp = 0.0;
  for (int d = 0; d < D; ++d) {
    double t = 0.0;
    for (int el = 0; el < E_loc; ++el) {
      int e = d * E_loc + el;
      double tg = cost_gemm_ms(cost, 0, rows[e]);
      double td = cost_gemm_ms(cost, 1, rows[e]);
      t += std::min(tg, td);
      if (d == cfg.rank) out->expert_kind[el] = (uint8_t)(td < tg ? MOE_GEMM_DENSE : MOE_GEMM_GROUPED);
    }
    t_comp = std::max(t_comp, t);
  }
  double t_comm = 0.0;
  if (D > 1) {
    double bytes = 0.0;
    for (int d = 0; d < D; ++d) bytes = std::max(bytes, std::max(send_rows[d], recv_rows[d]));
    bytes *= 2.0 * cfg.hidden;                           // bf16 rows, one direction
    double one = cost.a2a_fixed_ms + bytes / (cost.a2a_gbps * 1e9) * 1e3;
    t_comm = 2.0 * one;                                   // dispatch + combine
  }

  // pipeline number over N = 1..E_loc, then N = E_loc * S token-
  // sliced chunks (S = 2..slice_max, R8 extension); ties -> smaller N
  const double C = std::min(t_comm, t_comp);
  const int n_max = std::min(E_loc, MOE_MAX_CHUNKS);
  int best_n = 1;
  double best_v = -(cost.k_ms * 1 + cost.b_ms);
  auto consider = [&](int n) {
    double v = C / n * (n - 1) - (cost.k_ms * n + cost.b_ms);
    if (v > best_v) { best_v = v; best_n = n; }
  };
  for (int n = 2; n <= n_max; ++n) consider(n);
  const int s_max = (D > 1 && !cfg.local_reduce) ? plan_slice_max(E_loc, global_tokens / D) : 1;
  for (int s = 2; s <= s_max; ++s) consider(E_loc * s);
  out->num_chunks = best_n;
  out->token_slices = best_n > E_loc ? best_n / E_loc : 1;
  balanced_groups(E_loc, best_n / out->token_slices, out->group_begin);
  out->gemm_kind = MOE_GEMM_AUTO;
  out->sm_gemm = 0;
  out->comm_ctas = 0;
  out->pred_comm_ms = (float)t_comm;
  out->pred_comp_ms = (float)t_comp;
  out->pred_k_ms = cost.k_ms;
  out->pred_b_ms = cost.b_ms;
  out->pred_gain_ms = (float)(C - cost.b_ms - (C / best_n + cost.k_ms * best_n));
  return MOE_OK;
}

// Validate / complete a caller-supplied plan (group bounds filled in when the
// caller only set num_chunks).
int plan_normalise(const moe_config_t& cfg, moe_plan_t* p) {
  const int E_loc = cfg.num_experts / cfg.ep;
  if (p->token_slices < 1) p->token_slices = 1;
  const int S = p->token_slices;
  if (p->num_chunks < 1 || p->num_chunks > MOE_MAX_CHUNKS || p->num_chunks % S) return MOE_ERR_INVALID;
  const int NG = p->num_chunks / S;  // expert groups; chunk c = group c / S, slice c % S (R8)
  if (NG > E_loc) return MOE_ERR_INVALID;
  if (S > 1 && (cfg.ep == 1 || cfg.local_reduce)) {
    // ep == 1 has no all2all to pipeline; R16's groups assume expert-only chunks
    if (cfg.local_reduce && cfg.ep > 1) return MOE_ERR_UNSUPPORTED;
    p->token_slices = 1;
    p->num_chunks = NG;
  }
  bool ok = p->group_begin[0] == 0 && p->group_begin[NG] == E_loc;
  for (int c = 0; ok && c < NG; ++c) ok = p->group_begin[c + 1] > p->group_begin[c];
  if (!ok) balanced_groups(E_loc, NG, p->group_begin);
  if (p->gemm_kind != MOE_GEMM_AUTO)
    for (int e = 0; e < E_loc; ++e) p->expert_kind[e] = (uint8_t)p->gemm_kind;
  else
    for (int e = 0; e < E_loc; ++e)
      if (p->expert_kind[e] != MOE_GEMM_GROUPED && p->expert_kind[e] != MOE_GEMM_DENSE)
        p->expert_kind[e] = MOE_GEMM_GROUPED;
  return MOE_OK;
}

}  // namespace epsmoe
