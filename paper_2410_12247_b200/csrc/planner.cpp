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
#include <cstdlib>
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
  // one comm budget (the layer's default; EPSMOE_COMM_CTAS) at a2a_gbps, the
  // GEMMs slowed in proportion to the SMs they give up
  c->num_sms = 148;
  c->n_comm = 1;
  c->comm_ctas[0] = default_comm_ctas();
  c->a2a_gbps_at[0] = c->a2a_gbps;
  c->gemm_scale_at[0] = (float)(148.0 / (148.0 - 2.0 * c->comm_ctas[0]));
}

int default_comm_ctas() {
  const char* cv = std::getenv("EPSMOE_COMM_CTAS");
  return std::max(1, std::min(32, cv ? std::atoi(cv) : 8));
}

// Expected all2all rows per routed pair under expert-side LocalReduce (R16)
// with N chunks: a token sends one row per distinct (rank, chunk) group among
// its k experts.  With G = N * D groups of E / G experts and k distinct experts
// drawn uniformly, a group is missed with probability
// q = C(E - E/G, k) / C(E, k), so the token's remote groups number
// (G - N)(1 - q) on average (its own rank's N groups need no transfer), against
// k (D - 1) / D remote pairs.  (N = 1: D(1 - q) rows, the closed form of R16.)
double lr_rows_per_pair(int E, int D, int k, int N) {
  if (D <= 1) return 1.0;
  const double G = (double)N * D, s = (double)E / G;
  double q = 1.0;
  for (int i = 0; i < k; ++i) q *= std::max(0.0, (E - s - i) / (double)(E - i));
  const double remote_pairs = k * (D - 1.0) / D;
  return (G - N) * (1.0 - q) / remote_pairs;
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

  // per-expert kind (A8) and per-rank modelled compute on all SMs; the plan
  // follows the max-loaded rank so every rank derives the same plan.
  double t_comp_all = 0.0;
  for (int d = 0; d < D; ++d) {
    double t = 0.0;
    for (int el = 0; el < E_loc; ++el) {
      int e = d * E_loc + el;
      double tg = cost_gemm_ms(cost, 0, rows[e]);
      double td = cost_gemm_ms(cost, 1, rows[e]);
      t += std::min(tg, td);
      if (d == cfg.rank) out->expert_kind[el] = (uint8_t)(td < tg ? MOE_GEMM_DENSE : MOE_GEMM_GROUPED);
    }
    t_comp_all = std::max(t_comp_all, t);
  }
  // wire rows of the max-loaded rank in one direction, and the bytes per row:
  // dispatch FP8 rows (H + H/128 e4m3 + exponents, padded to 16 B; R15) or bf16,
  // combine always bf16 rows
  double pairs = 0.0;
  for (int d = 0; d < D; ++d) pairs = std::max(pairs, std::max(send_rows[d], recv_rows[d]));
  const double disp_row = cfg.dispatch_fp8 ? (double)(((cfg.hidden + cfg.hidden / 128) + 15) & ~15)
                                           : 2.0 * cfg.hidden;
  const double comb_row = 2.0 * cfg.hidden;
  // comm budgets: NCCL / put planes give up 2 * comm_ctas SMs; the copy-engine
  // plane none (its rows move without SMs)
  const int nsm = cost.num_sms > 0 ? cost.num_sms : 148;
  int ncand = (D > 1) ? std::max(1, std::min(cost.n_comm, (int)MOE_COMM_POINTS)) : 1;
  const bool ce = cfg.a2a_p2p == 2;
  if (ce) ncand = 1;
  // pipeline number over N = 1..E_loc, then N = E_loc * S token-
  // sliced chunks (S = 2..slice_max, R8 extension), for every comm budget;
  // the pair with the smallest modelled layer time T_comp + T_comm - G(N)
  // wins (ties -> smaller N, then the first budget).  For one budget and a
  // wire size independent of N this is the paper's argmax of G(N).
  const int n_max = std::min(E_loc, MOE_MAX_CHUNKS);
  const int s_max = (D > 1 && !cfg.local_reduce) ? plan_slice_max(E_loc, global_tokens / D) : 1;
  std::vector<int> cands;
  for (int n = 1; n <= n_max; ++n) cands.push_back(n);
  for (int s = 2; s <= s_max; ++s) cands.push_back(E_loc * s);
  int best_n = 1, best_i = 0;
  double best_t = 1e300, best_comm = 0.0, best_comp = t_comp_all, best_g = 0.0;
  for (int i = 0; i < ncand; ++i) {
    const bool have = cost.n_comm > 0 && i < cost.n_comm;
    const int cc = (D > 1 && !ce) ? (have ? cost.comm_ctas[i] : default_comm_ctas()) : 0;
    const double gbps = have && cost.a2a_gbps_at[i] > 0 ? cost.a2a_gbps_at[i] : cost.a2a_gbps;
    double scale = 1.0;
    if (cc > 0) scale = (have && cost.gemm_scale_at[i] > 0) ? cost.gemm_scale_at[i] : nsm / (double)(nsm - 2 * cc);
    const double t_comp = t_comp_all * scale;
    for (int n : cands) {
      double t_comm = 0.0;
      if (D > 1) {
        const double f = cfg.local_reduce ? lr_rows_per_pair(E, D, k, n) : 1.0;
        const double bytes = pairs * f * (disp_row + comb_row);
        t_comm = 2.0 * cost.a2a_fixed_ms + bytes / (gbps * 1e9) * 1e3;  // dispatch + combine
      }
      const double C = std::min(t_comm, t_comp);
      const double g = C / n * (n - 1) - (cost.k_ms * n + cost.b_ms);   // L(theta;N) - R(N)
      const double t = t_comp + t_comm - g;
      if (t < best_t - 1e-12) {
        best_t = t; best_n = n; best_i = i; best_comm = t_comm; best_comp = t_comp; best_g = g;
      }
    }
  }
  out->num_chunks = best_n;
  out->token_slices = best_n > E_loc ? best_n / E_loc : 1;
  balanced_groups(E_loc, best_n / out->token_slices, out->group_begin);
  out->gemm_kind = MOE_GEMM_AUTO;
  if (D > 1 && !ce) {
    const bool have = cost.n_comm > 0 && best_i < cost.n_comm;
    out->comm_ctas = have ? cost.comm_ctas[best_i] : default_comm_ctas();
    out->sm_gemm = nsm - 2 * out->comm_ctas;
  } else {
    out->comm_ctas = 0;
    out->sm_gemm = (D > 1) ? nsm : 0;
  }
  out->pred_comm_ms = (float)best_comm;
  out->pred_comp_ms = (float)best_comp;
  out->pred_k_ms = cost.k_ms;
  out->pred_b_ms = cost.b_ms;
  out->pred_gain_ms = (float)best_g;
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
